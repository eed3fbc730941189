"""GPU-vs-oracle parity of the model variant (eq:d_fwd_model, PAPER.md:137-141;
reading R-N3): the collimator response r and the vertical correction c as functions of the distance to
the detector, on configs 2-4 (full size) at the north star's tolerances, through the C ABI.  Expected
values come from the oracle's O13 only."""
import numpy as np
import pytest

import oracle as O
import pget_data as P
from tests.metrics import rel_l2
from tests.test_gpu_parity import TOL_L2, assert_parity, dev, host, inputs, rho_tol

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VAR = dict(det_radius=1.6, c_slope=0.05, r_slope=0.35)


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_26745_b200 as m
    return m


@pytest.mark.parametrize("cid", [2, 3, 4])
def test_variant_fwd_jvp_vjp(pg, cid):
    gd = dict(P.geometry_desc(cid), **VAR)
    lam, mu, dl, dm, lp, mp = inputs(cid)
    g = pg.Geometry(gd)
    assert not g.info["angle_banks_merged"] or g.info["n_samples_traced"] * 2 == g.info["n_samples_nominal"]
    y_o, dy_o = O.jvp(gd, lam, mu, dl, dm, with_y=True)
    assert_parity(host(pg.forward(g, dev(lam), dev(mu))), y_o, f"var cfg{cid} forward")
    yj, dy = pg.jvp(g, dev(lam), dev(mu), dev(dl), dev(dm), want_y=True)
    assert_parity(host(yj), y_o, f"var cfg{cid} jvp.y")
    assert_parity(host(dy), dy_o, f"var cfg{cid} jvp")
    w = (O.forward(gd, lp, mp) - y_o).astype(np.float32)
    gl, gm = pg.vjp(g, dev(lam), dev(mu), dev(w))
    gl_o, gm_o = O.vjp(gd, lam, mu, w)
    assert_parity(host(gl), gl_o, f"var cfg{cid} vjp.lam")
    assert_parity(host(gm), gm_o, f"var cfg{cid} vjp.mu")


def test_variant_changes_the_model(pg):
    """The variant is not the base model: at config 2 the readings differ by far more than the parity
    tolerance (c lengthens every path, r redistributes between sub-rays)."""
    gd = P.geometry_desc(2)
    lam, mu, *_ = inputs(2)
    y0 = host(pg.forward(pg.Geometry(gd), dev(lam), dev(mu)))
    y1 = host(pg.forward(pg.Geometry(dict(gd, **VAR)), dev(lam), dev(mu)))
    assert rel_l2(y1, y0) > 1e-3


@pytest.mark.parametrize("cid", [2, 4])
def test_variant_gn_operator(pg, cid):
    gd = dict(P.geometry_desc(cid), **VAR)
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
def test_variant_lm_iteration(pg, cid):
    """One LM iteration with the variant, R-LM tolerances as test_lm_iteration."""
    cfg = P.CONFIGS[cid]
    gd = dict(P.geometry_desc(cid), **VAR)
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
