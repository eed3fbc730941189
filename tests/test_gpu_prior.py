"""GPU-vs-oracle parity of the geometry priors P1, P2 (pget_set_prior; SURVEY.md §8(f) N1;
PAPER.md:146-148 eq:lma_objective, continued with alpha at PAPER.md:288; oracle O10, pins P15).

Masks from pget_data.prior_masks (0 around every lattice position, 1 elsewhere).  Tolerances are
those of the prior-free tests (reading R-LM): the operator at the north star's 1e-5 rel-L2;
quantities before the CG loop at 1e-5; pred at 1e-3; rho by rho_tol; accept decisions where clear;
later LM iterations at 10 %, the final iterate at 5 %; the safeguard by its cancellation bound."""
import numpy as np
import pytest

import oracle as O
import pget_data as P
from tests.metrics import rel_l2
from tests.test_gpu_parity import rho_tol

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

A1, A2 = 0.5, 2.0


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_26745_b200 as m
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def _cfg2():
    cid = 2
    cfg = P.CONFIGS[cid]
    gd = P.geometry_desc(cid)
    lt, mt = P.make_phantom(cid)
    y = P.poisson_noise(O.forward(gd, lt, mt), cfg.noise_peak, cfg.seed)
    l0, m0 = P.initial_guess(gd["n_px"])
    m1, m2 = P.prior_masks(cid)
    return cid, cfg, gd, y, (l0, m0), (m1, m2)


@pytest.mark.parametrize("cached", [False, True])
def test_gn_apply_with_prior(pg, cached, monkeypatch):
    monkeypatch.setenv("PGET_GN_APPLY_CACHED", "1" if cached else "0")
    cid, cfg, gd, y, (l0, m0), (m1, m2) = _cfg2()
    g = pg.Geometry(gd)
    M1, M2 = dev(m1), dev(m2)
    g.set_prior(M1, M2, A1, A2)
    # rod directions (zero where the masks are 1) plus white noise everywhere
    pl, pm = P.rod_directions(cid)
    wl, wm = P.white_directions(pl.shape, 3)
    pl, pm = pl + 0.1 * wl, pm + 0.1 * wm
    ql, qm = pg.gn_apply(g, dev(l0), dev(m0), dev(pl), dev(pm), cfg.alpha, 0.25)
    ol, om = O.apply_H(gd, l0, m0, cfg.alpha, 0.25, pl, pm, prior=(m1, m2, A1, A2))
    x = np.concatenate([host(ql).ravel(), host(qm).ravel()])
    o = np.concatenate([ol.ravel(), om.ravel()])
    assert rel_l2(x, o) <= 1e-5
    # the prior's share is not negligible at these weights, and clearing it restores H
    o0 = np.concatenate([a.ravel() for a in O.apply_H(gd, l0, m0, cfg.alpha, 0.25, pl, pm)])
    assert rel_l2(o, o0) > 1e-3
    g.set_prior()
    ql, qm = pg.gn_apply(g, dev(l0), dev(m0), dev(pl), dev(pm), cfg.alpha, 0.25)
    assert rel_l2(np.concatenate([host(ql).ravel(), host(qm).ravel()]), o0) <= 1e-5


def test_lm_iteration_with_prior_cfg2(pg):
    cid, cfg, gd, y, (l0, m0), (m1, m2) = _cfg2()
    g = pg.Geometry(gd)
    M1, M2 = dev(m1), dev(m2)
    g.set_prior(M1, M2, A1, A2)
    sl, sm, st = pg.gn_cg_step(g, dev(l0), dev(m0), dev(y), cfg.alpha, 0.0, cfg.n_cg)
    torch.cuda.synchronize()
    S = pg.read_stats(st, 1, cfg.n_cg)[0]
    sl_o, sm_o, So = O.gn_cg_step(gd, l0, m0, y, cfg.alpha, 0.0, cfg.n_cg, prior=(m1, m2, A1, A2))
    So0 = O.gn_cg_step(gd, l0, m0, y, cfg.alpha, 0.0, 0)[2]
    assert So["reg"] - So0["reg"] > 1e-3 * So["f"]          # the prior is a visible part of f
    for k in ("f", "misfit", "reg", "grad_norm"):
        assert abs(S[k] - So[k]) <= 1e-5 * abs(So[k]), k
    assert abs(S["cg_res"][1] - So["cg_res"][1]) <= 1e-4 * So["cg_res"][1]
    assert abs(S["pred"] - So["pred"]) <= 1e-3 * abs(So["pred"])
    assert abs(S["rho"] - So["rho"]) <= rho_tol(So)
    assert S["accepted"] == So["accepted"]
    s = np.concatenate([host(sl).ravel(), host(sm).ravel()])
    assert rel_l2(s, np.concatenate([sl_o.ravel(), sm_o.ravel()])) <= 0.1


def test_lm_solve_with_prior(pg):
    """Batched LM solve with alpha continuation: the priors follow alpha."""
    B, n = 2, 32
    gd = dict(n_px=n, n_angles=16, n_banks=2, n_det=21, n_subrays=3, subray_sigma=0.4, step_px=0.5,
              bank1_shift=0.0, batch=B)
    lt, mt = P.make_phantom(2, n_px=n)
    g1 = dict(gd, batch=1)
    y = np.concatenate([P.poisson_noise(O.forward(g1, lt * (1 + 0.1 * b), mt), 1e4, 20 + b)
                        for b in range(B)]).astype(np.float32)
    l0, m0 = P.initial_guess(n, B)
    m1, m2 = P.prior_masks(2, n_px=n)
    m1, m2 = np.concatenate([m1] * B), np.concatenate([m2] * B)
    kw = dict(n_iter=4, n_cg=8, alpha0=1e-2, alpha_decay=5.0, k_freeze=2, beta0=0.1)
    g = pg.Geometry(gd)
    M1, M2 = dev(m1), dev(m2)
    g.set_prior(M1, M2, A1, A2)
    lam, mu = dev(l0), dev(m0)
    S = pg.lm_solve(g, lam, mu, dev(y), **kw)
    torch.cuda.synchronize()
    (lo, mo), So = O.lm_solve(gd, l0, m0, y, kw["n_iter"], kw["n_cg"], kw["alpha0"], kw["alpha_decay"],
                              kw["k_freeze"], kw["beta0"], prior=(m1, m2, A1, A2))
    lam, mu = host(lam), host(mu)
    for m in range(B):
        for key in ("f", "misfit", "reg", "grad_norm"):
            assert abs(S[0][m][key] - So[m][0][key]) <= 1e-5 * abs(So[m][0][key]), key
        for k in range(kw["n_iter"]):
            a, o = S[k][m], So[m][k]
            assert abs(a["f"] - o["f"]) <= (1e-5 if k == 0 else 0.1) * abs(o["f"]), (m, k)
            if abs(o["rho"] - 0.1) > 0.02:
                assert a["accepted"] == o["accepted"], (m, k)
        assert rel_l2(lam[m].astype(np.float64), lo[m]) <= 5e-2
        assert rel_l2(mu[m].astype(np.float64), mo[m]) <= 5e-2


def test_safeguard_with_prior(pg):
    from tests.test_gpu_safeguard import _check
    cid, cfg, gd, y, (l0, m0), (m1, m2) = _cfg2()
    g = pg.Geometry(gd)
    M1, M2 = dev(m1), dev(m2)
    g.set_prior(M1, M2, A1, A2)
    lt, mt = P.make_phantom(cid)
    sl, sm, _ = pg.gn_cg_step(g, dev(l0), dev(m0), dev(y), cfg.alpha, 0.0, cfg.n_cg)
    torch.cuda.synchronize()
    decided = _check(pg, gd, g, l0, m0, y, host(sl), host(sm), lt, mt, cfg.alpha, prior=(m1, m2, A1, A2))
    assert {"identity", "wild"} <= {d[0] for d in decided}, decided


def test_set_prior_errors(pg):
    gd = dict(n_px=16, n_angles=8, n_banks=2, n_det=9, n_subrays=1, subray_sigma=0.4, step_px=0.5,
              bank1_shift=0.0, batch=1)
    g = pg.Geometry(gd)
    z = torch.zeros(g.img_shape, device="cuda")
    with pytest.raises(RuntimeError, match="alpha1"):
        g.set_prior(z, z, -1.0, 0.0)
    with pytest.raises(RuntimeError, match="alpha1"):
        g.set_prior(z, None, float("nan"), 0.0)
    with pytest.raises(TypeError):
        g.set_prior(z.double(), None, 1.0, 0.0)
