"""GPU-vs-oracle parity of the full LM solve (pget_lm_solve; PAPER.md:144-182,
288) through the C ABI: alpha continuation, per-member beta schedule, box projection,
accept/reject, on a small batched geometry.

Tolerances (reading R-LM): everything before the first CG step is pinned at 1e-5; the accept
decisions must agree wherever rho is clear of eta = 0.1 by 0.02; the objective values of later
iterations at 10 % and the final iterate at 5 % relative L2 (each 20-step CG solve amplifies
fp32-level perturbations to 2-3 % in s and up to ~9 % in f(u + s): profiles/cg_sensitivity_r01*.txt);
the objective must decrease and the box is checked exactly."""
import numpy as np
import pytest

import oracle as O
import pget_data as P
from tests.metrics import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_26745_b200 as m
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _problem(batch=2, n_px=32):
    gd = dict(n_px=n_px, n_angles=16, n_banks=2, n_det=21, n_subrays=3, subray_sigma=0.4, step_px=0.5,
              bank1_shift=0.0, batch=batch)
    lt, mt = P.make_phantom(2, n_px=n_px)
    lts = np.concatenate([lt * (1.0 + 0.1 * b) for b in range(batch)])
    mts = np.concatenate([mt * (1.0 - 0.05 * b) for b in range(batch)])
    g1 = dict(gd, batch=1)
    y = np.concatenate([P.poisson_noise(O.forward(g1, lts[b:b + 1], mts[b:b + 1]), 1e4, 10 + b)
                        for b in range(batch)]).astype(np.float32)
    l0, m0 = P.initial_guess(n_px, batch)
    return gd, y, l0, m0


@pytest.mark.parametrize("box", [None, (0.0, 1.5, 0.0, 0.6)])
def test_lm_solve_parity(pg, box):
    gd, y, l0, m0 = _problem()
    kw = dict(n_iter=4, n_cg=8, alpha0=1e-2, alpha_decay=5.0, k_freeze=2, beta0=0.1)
    g = pg.Geometry(gd)
    lam, mu = dev(l0), dev(m0)
    S = pg.lm_solve(g, lam, mu, dev(y), box=box, **kw)
    torch.cuda.synchronize()
    (lo, mo), So = O.lm_solve(gd, l0, m0, y, kw["n_iter"], kw["n_cg"], kw["alpha0"], kw["alpha_decay"],
                              kw["k_freeze"], kw["beta0"], box=box)
    lam, mu = lam.cpu().numpy(), mu.cpu().numpy()
    for m in range(gd["batch"]):
        for key in ("f", "misfit", "reg", "grad_norm"):
            assert abs(S[0][m][key] - So[m][0][key]) <= 1e-5 * abs(So[m][0][key]), key
        for k in range(kw["n_iter"]):
            a, o = S[k][m], So[m][k]
            # f(u_k) for k >= 1 depends on k CG solves: each moves f(u + s) by up to ~9 % under fp32-level
            # perturbations (profiles/cg_sensitivity_r01*.txt), hence 10 % (R-LM)
            assert abs(a["f"] - o["f"]) <= (1e-5 if k == 0 else 0.1) * abs(o["f"]), (m, k)
            if abs(o["rho"] - 0.1) > 0.02:
                assert a["accepted"] == o["accepted"], (m, k, a["rho"], o["rho"])
        assert rel_l2(lam[m].astype(np.float64), lo[m]) <= 5e-2   # steps differ by 2-3 % each (R-LM)
        assert rel_l2(mu[m].astype(np.float64), mo[m]) <= 5e-2
        assert S[-1][m]["f_trial"] < S[0][m]["f"]
    if box is not None:
        assert lam.min() >= box[0] and lam.max() <= box[1] and mu.min() >= box[2] and mu.max() <= box[3]


def test_lm_solve_errors(pg):
    gd, y, l0, m0 = _problem(batch=1, n_px=16)
    g = pg.Geometry(gd)
    lam, mu, yd = dev(l0), dev(m0), dev(y)
    with pytest.raises(RuntimeError, match="empty box"):
        pg.lm_solve(g, lam, mu, yd, 1, 4, box=(1.0, 0.0, 0.0, 1.0))
    with pytest.raises(RuntimeError, match="alpha_decay"):
        pg.lm_solve(g, lam, mu, yd, 1, 4, alpha_decay=0.5)
    with pytest.raises(RuntimeError, match="n_cg"):
        pg.lm_solve(g, lam, mu, yd, 1, 10_000)


def test_lm_solve_sgp_parity(pg):
    """PGET_LM_SGP (O11): the box-constrained steps by gradient projection with
    Barzilai-Borwein lengths.  Same pins as the CG solve (reading R-LM: the inner iterations amplify
    fp32-level differences), plus the SGP-specific ones: every iterate inside the box, the first
    projected-gradient step ||d_0|| at 1e-5 (it precedes any GN product)."""
    gd, y, l0, m0 = _problem()
    box = (0.0, 1.5, 0.0, 0.6)
    kw = dict(n_iter=4, n_cg=8, alpha0=1e-2, alpha_decay=5.0, k_freeze=2, beta0=0.1)
    g = pg.Geometry(gd)
    lam, mu = dev(l0), dev(m0)
    S = pg.lm_solve(g, lam, mu, dev(y), box=box, sgp=True, **kw)
    torch.cuda.synchronize()
    (lo, mo), So = O.lm_solve(gd, l0, m0, y, kw["n_iter"], kw["n_cg"], kw["alpha0"], kw["alpha_decay"],
                              kw["k_freeze"], kw["beta0"], box=box, inner="sgp")
    lam, mu = lam.cpu().numpy(), mu.cpu().numpy()
    for m in range(gd["batch"]):
        for key in ("f", "misfit", "reg", "grad_norm"):
            assert abs(S[0][m][key] - So[m][0][key]) <= 1e-5 * abs(So[m][0][key]), key
        assert abs(S[0][m]["cg_res"][0] - So[m][0]["cg_res"][0]) <= 1e-5 * So[m][0]["cg_res"][0]
        for k in range(kw["n_iter"]):
            a, o = S[k][m], So[m][k]
            assert abs(a["f"] - o["f"]) <= (1e-5 if k == 0 else 0.1) * abs(o["f"]), (m, k)
            if abs(o["rho"] - 0.1) > 0.02:
                assert a["accepted"] == o["accepted"], (m, k, a["rho"], o["rho"])
        assert rel_l2(lam[m].astype(np.float64), lo[m]) <= 5e-2
        assert rel_l2(mu[m].astype(np.float64), mo[m]) <= 5e-2
        assert S[-1][m]["f_trial"] < S[0][m]["f"]
    assert lam.min() >= box[0] and lam.max() <= box[1] and mu.min() >= box[2] and mu.max() <= box[3]


def test_lm_solve_sgp_needs_box(pg):
    gd, y, l0, m0 = _problem(batch=1, n_px=16)
    g = pg.Geometry(gd)
    with pytest.raises(RuntimeError, match="PGET_LM_SGP"):
        pg.lm_solve(g, dev(l0), dev(m0), dev(y), 1, 4, sgp=True)


@pytest.mark.parametrize("sgp", [False, True])
def test_lm_solve_linear_constraint(pg, sgp):
    """lam <= c mu in every projection (O12, reading R-lin), with CG + projection and with
    SGP: parity pins as above, and every final iterate inside the feasible set."""
    gd, y, l0, m0 = _problem()
    box, c = (0.0, 1.5, 0.0, 0.6), 3.0
    kw = dict(n_iter=4, n_cg=8, alpha0=1e-2, alpha_decay=5.0, k_freeze=2, beta0=0.1)
    g = pg.Geometry(gd)
    lam, mu = dev(l0), dev(m0)
    S = pg.lm_solve(g, lam, mu, dev(y), box=box, sgp=sgp, lam_per_mu=c, **kw)
    torch.cuda.synchronize()
    (lo, mo), So = O.lm_solve(gd, l0, m0, y, kw["n_iter"], kw["n_cg"], kw["alpha0"], kw["alpha_decay"],
                              kw["k_freeze"], kw["beta0"], box=box + (c,), inner="sgp" if sgp else "cg")
    lam, mu = lam.cpu().numpy(), mu.cpu().numpy()
    for m in range(gd["batch"]):
        for key in ("f", "misfit", "reg", "grad_norm"):
            assert abs(S[0][m][key] - So[m][0][key]) <= 1e-5 * abs(So[m][0][key]), key
        for k in range(kw["n_iter"]):
            a, o = S[k][m], So[m][k]
            assert abs(a["f"] - o["f"]) <= (1e-5 if k == 0 else 0.1) * abs(o["f"]), (m, k)
            if abs(o["rho"] - 0.1) > 0.02:
                assert a["accepted"] == o["accepted"], (m, k)
        assert rel_l2(lam[m].astype(np.float64), lo[m]) <= 5e-2
        assert rel_l2(mu[m].astype(np.float64), mo[m]) <= 5e-2
    assert np.all(lam <= c * mu + 1e-6 * c) and lam.min() >= box[0] and mu.max() <= box[3]
    assert np.any(np.isclose(lam, c * mu, rtol=1e-5, atol=0) & (lam > 0))   # the constraint binds
    with pytest.raises(RuntimeError, match="lam_per_mu"):
        pg.lm_solve(g, dev(l0), dev(m0), dev(y), 1, 4, lam_per_mu=3.0)
