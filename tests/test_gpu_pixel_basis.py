"""GPU-vs-oracle parity of the pixel basis (eq:d_fwd_model's exact intersection
lengths d_{m,n,k}; reading R-pb), alone and with the response of reading R-N3, on
configs 2-5 (full size) and small edge geometries at the north star's tolerances, through the C ABI.
Expected values come from the oracle's O14 only.  The configs contain rays that run exactly along a
pixel edge (odd J, axis-aligned angles): the kernel's fp64 traversal repeats the oracle's operations,
so it picks the same pixel there."""
import numpy as np
import pytest

import oracle as O
import pget_data as P
from tests.metrics import rel_l2
from tests.test_gpu_parity import TOL_L2, assert_parity, dev, host, inputs, rho_tol

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PB = dict(pixel_basis=1)
VAR = dict(det_radius=1.6, c_slope=0.05, r_slope=0.35)

EDGE = [
    dict(n_px=17, n_angles=7, n_banks=2, n_det=13, n_subrays=3, subray_sigma=0.4, step_px=0.5, bank1_shift=0.0,
         batch=3),
    dict(n_px=40, n_angles=12, n_banks=1, n_det=64, n_subrays=1, subray_sigma=0.4, step_px=0.5, bank1_shift=0.0,
         batch=1),
    dict(n_px=9, n_angles=4, n_banks=2, n_det=5, n_subrays=5, subray_sigma=0.3, step_px=0.5, bank1_shift=0.37,
         batch=2),
]


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_26745_b200 as m
    return m


def _fwd_jvp_vjp(pg, gd, lam, mu, dl, dm, w, what):
    g = pg.Geometry(gd)
    assert g.info["angle_banks_merged"] == 0
    y_o, dy_o = O.jvp(gd, lam, mu, dl, dm, with_y=True)
    assert_parity(host(pg.forward(g, dev(lam), dev(mu))), y_o, f"{what} forward")
    yj, dy = pg.jvp(g, dev(lam), dev(mu), dev(dl), dev(dm), want_y=True)
    assert_parity(host(yj), y_o, f"{what} jvp.y")
    assert_parity(host(dy), dy_o, f"{what} jvp")
    if w is None:
        w = (0.1 * y_o).astype(np.float32)
    gl, gm = pg.vjp(g, dev(lam), dev(mu), dev(w))
    gl_o, gm_o = O.vjp(gd, lam, mu, w)
    assert_parity(host(gl), gl_o, f"{what} vjp.lam")
    assert_parity(host(gm), gm_o, f"{what} vjp.mu")
    return g, w


@pytest.mark.parametrize("cid", [2, 3, 4])
def test_pixel_basis_fwd_jvp_vjp(pg, cid):
    gd = dict(P.geometry_desc(cid), **PB)
    lam, mu, dl, dm, lp, mp = inputs(cid)
    w = (O.forward(gd, lp, mp) - O.forward(gd, lam, mu)).astype(np.float32)
    _fwd_jvp_vjp(pg, gd, lam, mu, dl, dm, w, f"pb cfg{cid}")


@pytest.mark.parametrize("cid", [2, 4])
def test_pixel_basis_with_response_fwd_jvp_vjp(pg, cid):
    gd = dict(P.geometry_desc(cid), **PB, **VAR)
    lam, mu, dl, dm, lp, mp = inputs(cid)
    w = (O.forward(gd, lp, mp) - O.forward(gd, lam, mu)).astype(np.float32)
    _fwd_jvp_vjp(pg, gd, lam, mu, dl, dm, w, f"pb+var cfg{cid}")


def test_pixel_basis_config5_batched(pg):
    """All 64 config-5 members in one launch (forward, JVP, VJP), each against the oracle."""
    gd = dict(P.geometry_desc(5), **PB)
    lam, mu, dl, dm, lp, mp = inputs(5)
    w = (O.forward(gd, lp, mp) - O.forward(gd, lam, mu)).astype(np.float32)
    _fwd_jvp_vjp(pg, gd, lam, mu, dl, dm, w, "pb cfg5")


@pytest.mark.parametrize("k", range(len(EDGE)))
def test_pixel_basis_edge_geometries(pg, k):
    gd = dict(EDGE[k], **PB)
    rng = np.random.default_rng(90 + k)
    shp = O.img_shape(gd)
    lam, mu = rng.uniform(0.0, 1.5, shp), rng.uniform(0.0, 0.8, shp)
    dl, dm = rng.uniform(-1, 1, shp), rng.uniform(-0.2, 0.2, shp)
    w = rng.standard_normal(O.sino_shape(gd)).astype(np.float32)
    _fwd_jvp_vjp(pg, gd, lam, mu, dl, dm, w, f"pb edge {k}")


def test_pixel_basis_differs_from_sampled_model(pg):
    gd = P.geometry_desc(2)
    lam, mu, *_ = inputs(2)
    y0 = host(pg.forward(pg.Geometry(gd), dev(lam), dev(mu)))
    y1 = host(pg.forward(pg.Geometry(dict(gd, **PB)), dev(lam), dev(mu)))
    assert rel_l2(y1, y0) > 1e-3


def test_pixel_basis_vjp_bitwise_deterministic(pg):
    gd = dict(P.geometry_desc(2), **PB)
    lam, mu, *_ = inputs(2)
    g = pg.Geometry(gd)
    w = np.random.default_rng(5).standard_normal(O.sino_shape(gd)).astype(np.float32)
    a = [tuple(host(t) for t in pg.vjp(g, dev(lam), dev(mu), dev(w))) for _ in range(3)]
    for x in a[1:]:
        assert np.array_equal(x[0], a[0][0]) and np.array_equal(x[1], a[0][1])


@pytest.mark.parametrize("cid,var", [(2, False), (4, False), (2, True)])
def test_pixel_basis_gn_operator(pg, cid, var):
    gd = dict(P.geometry_desc(cid), **PB, **(VAR if var else {}))
    cfg = P.CONFIGS[cid]
    g = pg.Geometry(gd)
    lam, mu = P.initial_guess(gd["n_px"])
    pl, pm = P.rod_directions(cid)
    ql, qm = pg.gn_apply(g, dev(lam), dev(mu), dev(pl), dev(pm), cfg.alpha, 0.25)
    ql_o, qm_o = O.apply_H(gd, lam, mu, cfg.alpha, 0.25, pl, pm)
    x = np.concatenate([host(ql).ravel(), host(qm).ravel()])
    o = np.concatenate([ql_o.ravel(), qm_o.ravel()])
    assert rel_l2(x, o) <= TOL_L2


@pytest.mark.parametrize("cid", [2, 3])
def test_pixel_basis_lm_iteration(pg, cid):
    """One LM iteration in the pixel basis, R-LM tolerances as test_lm_iteration."""
    cfg = P.CONFIGS[cid]
    gd = dict(P.geometry_desc(cid), **PB)
    g = pg.Geometry(gd)
    lt, mt = P.make_phantom(cid)
    y = P.poisson_noise(O.forward(gd, lt, mt), cfg.noise_peak, cfg.seed)
    l0, m0 = P.initial_guess(gd["n_px"])
    sl, sm, st = pg.gn_cg_step(g, dev(l0), dev(m0), dev(y), cfg.alpha, 0.0, cfg.n_cg)
    torch.cuda.synchronize()
    S = pg.read_stats(st, 1, cfg.n_cg)[0]
    sl_o, sm_o, So = O.gn_cg_step(gd, l0, m0, y, cfg.alpha, 0.0, cfg.n_cg)
    for k in ("f", "misfit", "reg", "grad_norm"):
        assert abs(S[k] - So[k]) <= 1e-5 * abs(So[k]), k
    assert abs(S["cg_res"][1] - So["cg_res"][1]) <= 1e-4 * So["cg_res"][1]
    assert abs(S["pred"] - So["pred"]) <= 1e-3 * abs(So["pred"])
    assert abs(S["rho"] - So["rho"]) <= rho_tol(So)
    assert S["accepted"] == So["accepted"]
    s = np.concatenate([host(sl).ravel(), host(sm).ravel()])
    assert rel_l2(s, np.concatenate([sl_o.ravel(), sm_o.ravel()])) <= 0.1
