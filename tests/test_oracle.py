"""Pins of the fp64 oracle against what the paper and the mathematics fix
(SURVEY.md §8(c.4) P1-P12).  CPU only.  None of these re-types an oracle formula:
each compares it with a closed form, a symmetry, brute force, finite differences,
a library routine or an algebraic identity of a different function.
"""
import math

import numpy as np
import pytest

import oracle as O
import pget_data as P
from tests.metrics import max_rel, rel_l2


def small(n_px=16, n_angles=8, n_det=9, J=3, batch=1, **kw):
    d = dict(n_px=n_px, n_angles=n_angles, n_banks=2, n_det=n_det, n_subrays=J,
             subray_sigma=0.4, step_px=0.5, bank1_shift=0.0, batch=batch)
    d.update(kw)
    return d


def rand_img(g, seed, lo=0.0, hi=1.0):
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=O.img_shape(g))


# ----------------------------------------------------------------------------- P1 geometry
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_p1_tables_closed_form(cid):
    g = P.geometry_desc(cid)
    t = O.tables(g)
    N, nA, nd, J = g["n_px"], g["n_angles"], g["n_det"], g["n_subrays"]
    h = 2.0 / N
    # angles 2*pi*a/n_A, cos/sin of theta (+pi for bank 1)
    assert np.allclose(t["angles"], 2 * np.pi * np.arange(nA) / nA, rtol=0, atol=1e-15)
    assert np.allclose(t["dirs"][:, 0, 0], np.cos(t["angles"]), atol=1e-15)
    assert np.allclose(t["dirs"][:, 1, 0], -np.cos(t["angles"]), atol=1e-15)
    assert np.allclose(t["dirs"][:, 1, 1], -np.sin(t["angles"]), atol=1e-15)
    # offsets: endpoints +-1 at the outer sub-ray centres, mirror symmetry bitwise
    off = t["offsets"]
    for b in range(2):
        assert np.array_equal(off[b, ::-1, ::-1], -off[b])
    assert np.array_equal(off[0], off[1])
    pitch = 2.0 / (nd - 1)
    assert np.allclose(np.diff(off[0].ravel()), pitch / J, atol=1e-14)   # uniform sub-ray lattice
    # weights: normalised Gaussian, sigma = 0.4 pitch
    w = t["weights"]
    assert abs(w.sum() - 1.0) <= 2 ** -52 * J
    dj = (np.arange(J) + 0.5) / J - 0.5
    ref = np.exp(-dj ** 2 / (2 * 0.4 ** 2))
    assert np.allclose(w, ref / ref.sum(), rtol=1e-14, atol=0)
    # t-lattice
    hh, delta, T = t["tlat"]
    assert hh == h and delta == 0.5 * h
    m = math.ceil((math.sqrt(2) + h) / delta)
    assert T == delta * m and t["n_t"] == 2 * m


@pytest.mark.parametrize("gd", [small(), small(n_px=33, n_angles=12, J=2, n_det=7),
                                P.geometry_desc(1)])
def test_p1_clip_is_exact_support(gd):
    """Brute force: sample i lies in [i_lo, i_hi] iff its position is inside the
    support box |x|,|y| <= 1 + h/2 of the zero-padded bilinear interpolant."""
    t = O.tables(gd)
    h, delta, T = t["tlat"]
    i = np.arange(t["n_t"])
    tt = -T + (i + 0.5) * delta
    bb = 1 + h / 2
    for a in range(gd["n_angles"]):
        for b in range(2):
            c, s = t["dirs"][a, b]
            for d in range(gd["n_det"]):
                for j in range(gd["n_subrays"]):
                    sig = t["offsets"][b, d, j]
                    x = sig * (-s) + tt * c
                    y = sig * c + tt * s
                    inside = (np.abs(x) <= bb * (1 + 1e-12)) & (np.abs(y) <= bb * (1 + 1e-12))
                    strict = (np.abs(x) <= bb * (1 - 1e-12)) & (np.abs(y) <= bb * (1 - 1e-12))
                    lo, hi = t["clip"][a, b, d, j]
                    sel = (i >= lo) & (i <= hi)
                    assert np.all(inside[sel]) and np.all(sel[strict])


# ----------------------------------------------------------------------------- P2 / P4 closed forms
def _disk_geom(N, nA=4):
    return dict(n_px=N, n_angles=nA, n_banks=2, n_det=91, n_subrays=1, subray_sigma=0.4,
                step_px=0.5, bank1_shift=0.0, batch=1)


def _disk_errors(N, mu0):
    g = _disk_geom(N)
    lam, mu = P.disk_phantom(N, 0.5, 1.0, mu0)
    y = O.forward(g, lam, mu)[0]                    # [nA][2][91]
    s = O.tables(g)["offsets"][0, :, 0]
    R = 0.5
    sel = np.abs(s) <= 0.9 * R
    chord = 2 * np.sqrt(np.maximum(R * R - s ** 2, 0))
    ref = chord if mu0 == 0 else (1 - np.exp(-mu0 * chord)) / mu0
    err = np.abs(y[:, 0, sel] - ref[sel]) / ref[sel]
    return err, y


def test_p2_radon_disk():
    """mu = 0: the plain Radon transform, g(s) = 2 lam0 sqrt(R^2 - s^2) (north star)."""
    err, y = _disk_errors(128, 0.0)
    assert err.max() <= 1e-2
    # bank duality at mu = 0: bank 1 sees the same lines reversed
    assert np.abs(y[:, 1, :] - y[:, 0, ::-1]).max() <= 1e-13 * np.abs(y).max()


def test_p4_attenuated_disk_closed_form_and_convergence():
    """Uniform disk lam0 = 1, mu0 = 0.5, R = 0.5: g(s) = (1 - e^{-mu0 2 sqrt(R^2-s^2)})/mu0
    (north star; PAPER.md:48-54 eq:fwd_model); first-order convergence in h."""
    means = []
    for N in (128, 256):
        err, _ = _disk_errors(N, 0.5)
        assert err.max() <= 1.5e-2
        assert err.mean() <= 0.15 * (2.0 / N)
        means.append(err.mean())
    assert means[0] / means[1] >= 1.5


# ----------------------------------------------------------------------------- P3 quadrature closed form
@pytest.mark.parametrize("n,lam0,mu0,delta", [(1, 1.0, 0.5, 0.01), (37, 0.8, 0.5, 0.015625),
                                              (400, 1.3, 2.0, 0.0078125), (730, 1.0, 0.05, 0.00390625)])
def test_p3_geometric_series(n, lam0, mu0, delta):
    g = O.ray_quadrature(np.full(n, lam0), np.full(n, mu0), delta)
    x = mu0 * delta
    ref = lam0 * delta * math.exp(-x / 2) * math.expm1(-n * x) / math.expm1(-x)
    assert abs(g - ref) <= 1e-14 * ref


def test_p3_recurrence_equals_double_loop():
    """Brute force: the O(n) suffix recurrence equals the O(n^2) double loop of the definition."""
    g = small(n_px=12, n_angles=6, J=2, n_det=7)
    lam, mu = rand_img(g, 1), rand_img(g, 2, 0, 2.0)
    a = O.forward(g, lam, mu)
    b = O.forward(g, lam, mu, naive=True)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()


# ----------------------------------------------------------------------------- P5 invariants
def test_p5_invariants():
    g = small(n_px=20, n_angles=8)
    lam, mu = rand_img(g, 3), rand_img(g, 4, 0, 0.6)
    lam2 = rand_img(g, 5)
    y1 = O.forward(g, lam, mu)
    y2 = O.forward(g, lam2, mu)
    y12 = O.forward(g, 2.0 * lam - 0.5 * lam2, mu)
    assert rel_l2(y12, 2 * y1 - 0.5 * y2) <= 1e-13                 # linear in lambda
    assert np.all(O.forward(g, np.zeros_like(lam), mu) == 0.0)      # lambda = 0 -> y = 0
    for k in range(5):                                              # monotone in every mu pixel
        mu_up = mu.copy()
        j, i = np.random.default_rng(k).integers(0, 20, size=2)
        mu_up[0, j, i] += 0.3
        assert np.all(O.forward(g, lam, mu_up) <= y1 + 1e-15)
    # bank identity: y[a][1][d] = y[(a + nA/2) mod nA][0][d]
    nA = g["n_angles"]
    sh = np.roll(y1[0, :, 0, :], -nA // 2, axis=0)
    assert np.abs(y1[0, :, 1, :] - sh).max() <= 1e-13 * np.abs(y1).max()


# ----------------------------------------------------------------------------- P6 rotation
@pytest.mark.parametrize("cid", [1, 2])
def test_p6_rotation_invariance(cid):
    cfg = P.CONFIGS[cid]
    lam, mu = P.make_phantom(cid)
    lam, mu = lam.astype(np.float64), mu.astype(np.float64)
    g = P.geometry_desc(cid, n_angles=40 if cid == 2 else cfg.n_angles)
    nA = g["n_angles"]
    y = O.forward(g, lam, mu)
    # 180 degrees: lam'[iy][ix] = lam[N-1-iy][N-1-ix]  ->  y'[a] = y[a - nA/2]
    y180 = O.forward(g, lam[:, ::-1, ::-1], mu[:, ::-1, ::-1])
    assert rel_l2(y180, np.roll(y, nA // 2, axis=1)) <= 1e-12
    if nA % 4 == 0:
        # +90 degrees: lam'[iy][ix] = lam[N-1-ix][iy]  ->  y'[a] = y[a - nA/4]
        r90 = lambda im: np.transpose(im, (0, 2, 1))[:, :, ::-1]
        y90 = O.forward(g, r90(lam), r90(mu))
        assert rel_l2(y90, np.roll(y, nA // 4, axis=1)) <= 1e-12
        # the wrong sign must fail (confirms the orientation once)
        assert rel_l2(y90, np.roll(y, -nA // 4, axis=1)) > 1e-3


def test_p6_single_pixel_orientation():
    g = small(n_px=16, n_angles=4, J=1, n_det=31)
    lam = np.zeros((1, 16, 16))
    lam[0, 3, 12] = 1.0                     # x = -1 + 12.5h > 0, y = -1 + 3.5h < 0
    mu = np.zeros_like(lam)
    y = O.forward(g, lam, mu)[0]
    s = O.tables(g)["offsets"][0, :, 0]
    h = 2 / 16
    x0, y0 = -1 + 12.5 * h, -1 + 3.5 * h
    # theta = 0: omega = (1, 0), omega_perp = (0, 1) -> the pixel projects to s = y0
    assert abs(s[np.argmax(y[0, 0])] - y0) <= 2 / 30
    # theta = pi/2: omega_perp = (-1, 0) -> s = -x0
    assert abs(s[np.argmax(y[1, 0])] + x0) <= 2 / 30


# ----------------------------------------------------------------------------- P7 JVP
def test_p7_jvp_central_differences():
    g = small(n_px=24, n_angles=10, J=3, n_det=11)
    lam, mu = rand_img(g, 10, 0, 1.5), rand_img(g, 11, 0, 0.6)
    un = math.sqrt(np.sum(lam ** 2) + np.sum(mu ** 2))
    for k in range(20):
        rng = np.random.default_rng(100 + k)
        dl = rng.uniform(-1, 1, lam.shape)
        dm = rng.uniform(-0.1, 0.1, mu.shape)
        eps = 1e-6 * un / math.sqrt(np.sum(dl ** 2) + np.sum(dm ** 2))
        fd = (O.forward(g, lam + eps * dl, mu + eps * dm) - O.forward(g, lam - eps * dl, mu - eps * dm)) / (2 * eps)
        jv = O.jvp(g, lam, mu, dl, dm)
        assert rel_l2(jv, fd) <= 1e-7


def test_p7_jvp_lambda_part_is_forward():
    """D_lam F[dlam] = F(dlam, mu) (PAPER.md:56 eq:frechet) and lam = 0, dlam = 0 -> 0."""
    g = small(n_px=20)
    lam, mu, dl = rand_img(g, 1), rand_img(g, 2, 0, 0.6), rand_img(g, 3, -1, 1)
    jv = O.jvp(g, lam, mu, dl, np.zeros_like(mu))
    assert rel_l2(jv, O.forward(g, dl, mu)) <= 1e-14
    assert np.all(O.jvp(g, np.zeros_like(lam), mu, np.zeros_like(lam), rand_img(g, 4)) == 0)


# ----------------------------------------------------------------------------- P8 adjoint
def test_p8_adjoint_identity_100_triples():
    g = small(n_px=12, n_angles=6, J=2, n_det=9)
    for k in range(100):
        rng = np.random.default_rng(1000 + k)
        lam = rng.uniform(0, 1.5, O.img_shape(g))
        mu = rng.uniform(0, 0.6, O.img_shape(g))
        vl = rng.standard_normal(O.img_shape(g))
        vm = rng.standard_normal(O.img_shape(g))
        w = rng.standard_normal(O.sino_shape(g))
        jv = O.jvp(g, lam, mu, vl, vm)
        gl, gm = O.vjp(g, lam, mu, w)
        lhs = np.sum(jv * w)
        rhs = np.sum(vl * gl) + np.sum(vm * gm)
        assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(jv) * np.linalg.norm(w)


def test_p8_dense_jacobian_transpose():
    g = dict(n_px=8, n_angles=4, n_banks=2, n_det=5, n_subrays=2, subray_sigma=0.4, step_px=0.5,
             bank1_shift=0.0, batch=1)
    rng = np.random.default_rng(5)
    lam = rng.uniform(0.2, 1.5, (1, 8, 8))
    mu = rng.uniform(0.1, 0.6, (1, 8, 8))
    npx = 64
    cols = []
    for k in range(2 * npx):
        e = np.zeros(2 * npx)
        e[k] = 1.0
        cols.append(O.jvp(g, lam, mu, e[:npx].reshape(1, 8, 8), e[npx:].reshape(1, 8, 8)).ravel())
    Jd = np.stack(cols, axis=1)                       # [n_sino, 2 npx]
    ns = Jd.shape[0]
    rows = []
    for r in range(ns):
        w = np.zeros(ns)
        w[r] = 1.0
        gl, gm = O.vjp(g, lam, mu, w.reshape(O.sino_shape(g)))
        rows.append(np.concatenate([gl.ravel(), gm.ravel()]))
    JT = np.stack(rows, axis=0)                       # [n_sino, 2 npx] should equal Jd
    assert np.abs(JT - Jd).max() <= 1e-12 * np.abs(Jd).max()


def test_p8_vjp_zero_weights():
    g = small()
    gl, gm = O.vjp(g, rand_img(g, 1), rand_img(g, 2), np.zeros(O.sino_shape(g)))
    assert np.all(gl == 0) and np.all(gm == 0)


# ----------------------------------------------------------------------------- P9 per-ray adjoint
def test_p9_per_ray_adjoint_fd():
    rng = np.random.default_rng(9)
    n, delta = 60, 0.01
    ls, ms = rng.uniform(0, 1.5, n), rng.uniform(0, 3, n)
    dl, dm = O.ray_adjoint(ls, ms, delta)
    eps = 1e-3          # g is linear in lam and smooth in mu: truncation O(eps^2 delta^2) << roundoff
    for i in range(0, n, 7):
        e = np.zeros(n)
        e[i] = eps
        fl = (O.ray_quadrature(ls + e, ms, delta) - O.ray_quadrature(ls - e, ms, delta)) / (2 * eps)
        fm = (O.ray_quadrature(ls, ms + e, delta) - O.ray_quadrature(ls, ms - e, delta)) / (2 * eps)
        assert abs(fl - dl[i]) <= 1e-8 * abs(dl[i])
        assert abs(fm - dm[i]) <= 1e-8 * abs(dm[i])


# ----------------------------------------------------------------------------- P10 regulariser
def test_p10_laplacian():
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal((1, 11, 11)), rng.standard_normal((1, 11, 11))
    LLx = O.laplacian(O.laplacian(x))
    LLy = O.laplacian(O.laplacian(y))
    assert abs(np.sum(x * LLy) - np.sum(LLx * y)) <= 1e-12 * np.abs(LLx).max()
    assert np.sum(x * LLx) >= 0
    c = O.laplacian(np.full((1, 11, 11), 2.5))[0]
    assert np.all(c[1:-1, 1:-1] == 0) and c[0, 5] == 2.5 and c[0, 0] == 5.0
    d = np.zeros((1, 7, 7))
    d[0, 3, 3] = 1.0
    Ld = O.laplacian(d)[0]
    ref = np.zeros((7, 7))
    ref[3, 3] = 4
    ref[2, 3] = ref[4, 3] = ref[3, 2] = ref[3, 4] = -1
    assert np.array_equal(Ld, ref)


# ----------------------------------------------------------------------------- P11 / P12 GN-CG and LM
def _dense_H(g, lam, mu, alpha, beta):
    npx = g["n_px"] ** 2
    N = g["n_px"]
    Jc, Lc = [], []
    for k in range(2 * npx):
        e = np.zeros(2 * npx)
        e[k] = 1.0
        Jc.append(O.jvp(g, lam, mu, e[:npx].reshape(1, N, N), e[npx:].reshape(1, N, N)).ravel())
        Lc.append(np.concatenate([O.laplacian(e[:npx].reshape(1, N, N)).ravel(),
                                  O.laplacian(e[npx:].reshape(1, N, N)).ravel()]))
    Jd, Ld = np.stack(Jc, 1), np.stack(Lc, 1)
    return Jd, Ld, Jd.T @ Jd + alpha * Ld.T @ Ld + beta * np.eye(2 * npx)


def test_p11_cg_equals_dense_solve():
    N = 6
    g = dict(n_px=N, n_angles=6, n_banks=2, n_det=9, n_subrays=2, subray_sigma=0.4, step_px=0.5,
             bank1_shift=0.0, batch=1)
    rng = np.random.default_rng(2)
    lam, mu = rng.uniform(0.3, 1.2, (1, N, N)), rng.uniform(0.1, 0.5, (1, N, N))
    y = O.forward(g, rng.uniform(0.3, 1.2, (1, N, N)), rng.uniform(0.1, 0.5, (1, N, N)))
    alpha, beta = 1e-2, 0.05
    Jd, Ld, H = _dense_H(g, lam, mu, alpha, beta)
    r = (O.forward(g, lam, mu) - y).ravel()
    u = np.concatenate([lam.ravel(), mu.ravel()])
    b = -(Jd.T @ r + alpha * Ld.T @ (Ld @ u))
    s_ref = np.linalg.solve(H, b)
    sl, sm, st = O.gn_cg_step(g, lam, mu, y, alpha, beta, 200)
    s = np.concatenate([sl.ravel(), sm.ravel()])
    assert rel_l2(s, s_ref) <= 1e-8
    assert abs(st["grad_norm"] - np.linalg.norm(b)) <= 1e-10 * np.linalg.norm(b)
    # operator level: oracle H p (J^T via the VJP) equals the dense H built from JVP columns
    p = rng.standard_normal(2 * N * N)
    hl, hm = O.apply_H(g, lam, mu, alpha, beta, p[:N * N].reshape(1, N, N), p[N * N:].reshape(1, N, N))
    assert rel_l2(np.concatenate([hl.ravel(), hm.ravel()]), H @ p) <= 1e-12
    # model: pred = m(0) - m(s) with m(s) = 1/2||r + Js||^2 + alpha/2 ||L(u+s)||^2 (eq:m-function)
    def m(sv):
        return 0.5 * np.sum((r + Jd @ sv) ** 2) + 0.5 * alpha * np.sum((Ld @ (u + sv)) ** 2)
    assert abs(st["f"] - m(np.zeros_like(s))) <= 1e-12 * st["f"]          # m(0) = f(u)
    assert abs(st["pred"] - (m(np.zeros_like(s)) - m(s))) <= 1e-9 * abs(st["pred"])


def test_p11_cg_equals_dense_solve_with_priors():
    """With the O10 priors (diagonal masks m1, m2, weights a1, a2) the LM step solves
    (J^T J + alpha L^T L + diag(a1 m1^2, a2 m2^2) + beta I) s = b with b = -(J^T r + alpha L^T L u +
    (a1 m1^2 lam, a2 m2^2 mu)), and pred = m(0) - m(s) for the model with the prior rows
    sqrt(a1) m1 lam, sqrt(a2) m2 mu of F~ (eq:m-function).  Every matrix
    here is built in numpy from JVP columns and the masks; a dropped or doubled prior term in the
    oracle's b, H, or pred (its ps2 = 2 prior_value(s)) fails one of the three checks."""
    N = 6
    g = dict(n_px=N, n_angles=6, n_banks=2, n_det=9, n_subrays=2, subray_sigma=0.4, step_px=0.5,
             bank1_shift=0.0, batch=1)
    rng = np.random.default_rng(7)
    lam, mu = rng.uniform(0.3, 1.2, (1, N, N)), rng.uniform(0.1, 0.5, (1, N, N))
    y = O.forward(g, rng.uniform(0.3, 1.2, (1, N, N)), rng.uniform(0.1, 0.5, (1, N, N)))
    m1 = (rng.uniform(size=(1, N, N)) < 0.5).astype(np.float64)
    m2 = (rng.uniform(size=(1, N, N)) < 0.5).astype(np.float64)
    a1, a2 = 0.7, 3.0
    alpha, beta = 1e-2, 0.05
    Jd, Ld, H = _dense_H(g, lam, mu, alpha, beta)
    D = np.concatenate([a1 * m1.ravel() ** 2, a2 * m2.ravel() ** 2])
    H = H + np.diag(D)
    r = (O.forward(g, lam, mu) - y).ravel()
    u = np.concatenate([lam.ravel(), mu.ravel()])
    b = -(Jd.T @ r + alpha * Ld.T @ (Ld @ u) + D * u)
    s_ref = np.linalg.solve(H, b)
    pr = (m1, m2, a1, a2)
    sl, sm, st = O.gn_cg_step(g, lam, mu, y, alpha, beta, 200, prior=pr)
    s = np.concatenate([sl.ravel(), sm.ravel()])
    assert rel_l2(s, s_ref) <= 1e-8
    assert abs(st["grad_norm"] - np.linalg.norm(b)) <= 1e-10 * np.linalg.norm(b)

    def m(sv):
        return (0.5 * np.sum((r + Jd @ sv) ** 2) + 0.5 * alpha * np.sum((Ld @ (u + sv)) ** 2)
                + 0.5 * np.sum(D * (u + sv) ** 2))
    s0 = np.zeros_like(s)
    assert abs(st["f"] - m(s0)) <= 1e-12 * st["f"]
    assert abs(st["pred"] - (m(s0) - m(s))) <= 1e-9 * abs(st["pred"])
    # the same at a truncated CG iterate (s not the minimiser, so pred's quadratic term is tested
    # separately from <b, s>): 3 CG steps
    sl, sm, st = O.gn_cg_step(g, lam, mu, y, alpha, beta, 3, prior=pr)
    s = np.concatenate([sl.ravel(), sm.ravel()])
    assert abs(st["pred"] - (m(s0) - m(s))) <= 1e-9 * abs(st["pred"])
    assert abs(st["als2"] - (alpha * np.sum((Ld @ s) ** 2) + np.sum(D * s ** 2))) <= 1e-9 * st["als2"]


def test_p12_reject_when_pred_not_positive():
    """Reading R-accept: rho = (f(u) - f(u+s)) / pred is the ratio of the actual to the predicted
    decrease (eq:rho_agreement); a box that clips the CG step hard makes pred < 0, and
    a step that then raises f has rho > eta although it is no decrease.  Such a step is rejected."""
    g, _, y, (l0, m0) = _tiny_lm()
    sl, sm, st = O.lm_step_box(g, l0, m0, y, 1e-3, 0.0, 8, (0.7, 0.9, 0.28, 0.31), inner="cg")
    assert st["pred"] < 0 and st["f_trial"] > st["f"] and st["rho"] > 0.1   # the old rule accepted it
    assert not st["accepted"]
    assert st["beta_next"] == max(0.0, st["beta_min"])


def test_p11_cg_recurrence_residuals():
    N = 8
    g = dict(n_px=N, n_angles=8, n_banks=2, n_det=11, n_subrays=2, subray_sigma=0.4, step_px=0.5,
             bank1_shift=0.0, batch=1)
    rng = np.random.default_rng(4)
    lam, mu = rng.uniform(0.3, 1.2, (1, N, N)), rng.uniform(0.1, 0.5, (1, N, N))
    y = O.forward(g, *P.disk_phantom(N, 0.6, 1.0, 0.4))
    alpha, beta = 1e-3, 0.0
    preds = []
    for k in (1, 3, 6):
        sl, sm, st = O.gn_cg_step(g, lam, mu, y, alpha, beta, k)
        hl, hm = O.apply_H(g, lam, mu, alpha, beta, sl, sm)
        # b = -(J^T r + alpha L^T L u): rebuild from the first CG residual norm and H s
        _, _, st0 = O.gn_cg_step(g, lam, mu, y, alpha, beta, 0)
        r = O.forward(g, lam, mu) - y
        gl, gm = O.vjp(g, lam, mu, r)
        bl = -(gl + alpha * O.laplacian(O.laplacian(lam)))
        bm = -(gm + alpha * O.laplacian(O.laplacian(mu)))
        res = np.sqrt(np.sum((bl - hl) ** 2) + np.sum((bm - hm) ** 2))
        assert abs(res - st["cg_res"][k]) <= 1e-8 * st["cg_res"][0]
        preds.append(st["pred"])
        assert st["pred"] > 0
    assert preds[0] < preds[1] < preds[2]           # quadratic model decreases monotonically


def test_p11_linear_case_rho_one():
    """lam = 0, alpha = 0: J_mu = 0 so s_mu = 0, and F is linear in lam -> rho = 1."""
    N = 10
    g = dict(n_px=N, n_angles=8, n_banks=2, n_det=11, n_subrays=1, subray_sigma=0.4, step_px=0.5,
             bank1_shift=0.0, batch=1)
    lt, mt = P.disk_phantom(N, 0.6, 1.0, 0.4)
    y = O.forward(g, lt, mt)
    lam = np.zeros((1, N, N))
    sl, sm, st = O.gn_cg_step(g, lam, mt, y, 0.0, 0.0, 15)
    assert np.all(sm == 0)
    assert abs(st["rho"] - 1.0) <= 1e-10
    assert st["accepted"]


def test_p12_lm_wrap():
    cfg = P.CONFIGS[2]
    g = P.geometry_desc(2, n_px=32, n_angles=24)
    lt, mt = P.make_phantom(2, n_px=32)
    y = P.poisson_noise(O.forward(g, lt, mt), 1e4, 2)
    l0, m0 = P.initial_guess(32)
    sl, sm, st = O.gn_cg_step(g, l0, m0, y, cfg.alpha, 0.0, 8)
    assert st["pred"] > 0
    r = O.forward(g, l0, m0) - y
    reg = 0.5 * cfg.alpha * (np.sum(O.laplacian(l0) ** 2) + np.sum(O.laplacian(m0) ** 2))
    assert abs(st["f"] - (0.5 * np.sum(r ** 2) + reg)) <= 1e-12 * st["f"]
    assert np.all(np.diff(st["cg_res"]) != 0)
    if st["accepted"]:
        assert st["f_trial"] < st["f"]


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_p1_sample_counts_golden(cid):
    import json, os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sample_counts.json")))[str(cid)]
    g = P.geometry_desc(cid)
    t = O.tables(g)
    cl = t["clip"]
    assert int(np.clip(cl[..., 1] - cl[..., 0] + 1, 0, None).sum()) * g["batch"] == gold["samples"]
    assert cl[..., 0].size * g["batch"] == gold["rays"]
    assert t["n_t"] == gold["n_t"]


# ----------------------------------------------------------------------------- P13 safeguard (O8, N2)
def _lm_case(n_px=24, n_angles=16, n_cg=6):
    cfg = P.CONFIGS[2]
    g = P.geometry_desc(2, n_px=n_px, n_angles=n_angles)
    lt, mt = P.make_phantom(2, n_px=n_px)
    y = P.poisson_noise(O.forward(g, lt, mt), 1e4, 2)
    l0, m0 = P.initial_guess(n_px)
    sl, sm, st = O.gn_cg_step(g, l0, m0, y, cfg.alpha, 0.0, n_cg)
    return cfg, g, (lt, mt), y, (l0, m0), (sl, sm), st


def test_p13_candidate_equal_to_lm_step_matches_vjp_route():
    """u~ = u_k + s_k: m_k(s~) = m_k(s_k), and pred / rho equal the LM wrap's values, which that
    route computes as <b,s> - 1/2(...) with b from the VJP (adjoint of the JVP used here)."""
    cfg, g, _, y, (l0, m0), (sl, sm), st = _lm_case()
    (nl, nm), [r] = O.safeguard(g, l0, m0, y, sl, sm, l0 + sl, m0 + sm, cfg.alpha, 0.1)
    assert abs(r["m0"] - st["f"]) <= 1e-12 * st["f"]            # m_k(0) = f(u_k)
    assert abs(r["m_cand"] - r["m_lm"]) <= 1e-12 * st["f"]
    assert abs(r["pred_lm"] - st["pred"]) <= 1e-8 * st["pred"]
    assert abs(r["f_cand"] - st["f_trial"]) <= 1e-12 * st["f"]
    assert abs(r["rho_cand"] - st["rho"]) <= 1e-7 * abs(st["rho"])
    assert r["accepted"] == st["accepted"]
    np.testing.assert_array_equal(nl, l0 + sl)


def test_p13_model_exact_for_lambda_only_steps():
    """F is linear in lam (eq:frechet: D_lam F[dlam] = F(dlam, mu)) and the penalty is quadratic,
    so for s = (s_lam, 0) the model is exact: m_k(s) = f(u_k + s) for any s_lam."""
    cfg, g, _, y, (l0, m0), _, _ = _lm_case(n_px=16, n_angles=8)
    rng = np.random.default_rng(5)
    z = np.zeros_like(l0)
    for scale in (1e-2, 1.0, 30.0):
        dl = scale * rng.standard_normal(l0.shape)
        _, [r] = O.safeguard(g, l0, m0, y, z, z, l0 + dl, m0, cfg.alpha, 0.1)
        assert abs(r["m_cand"] - r["f_cand"]) <= 1e-10 * max(r["f_cand"], r["f"])


def test_p13_model_slope_and_curvature():
    """d/dt m_k(t s)|0 = d/dt f(u_k + t s)|0 (central differences of f); m_k(t s) is a quadratic in t
    (third differences vanish); and for a CG step from 0 with beta = 0, t = 1 minimises m_k(t s_k)
    (Galerkin condition <s, H s> = <b, s>)."""
    cfg, g, _, y, (l0, m0), (sl, sm), _ = _lm_case()
    rng = np.random.default_rng(9)
    dl, dm = 0.05 * rng.standard_normal(l0.shape), 0.01 * rng.standard_normal(m0.shape)
    z = np.zeros_like(l0)

    def m_of(t, al=dl, am=dm):
        _, [r] = O.safeguard(g, l0, m0, y, z, z, l0 + t * al, m0 + t * am, cfg.alpha, 0.1)
        return r["m_cand"], r["f_cand"], r["f"]

    h = 1e-4
    mp, fp, f0 = m_of(h)
    mn, fn, _ = m_of(-h)
    assert abs((mp - mn) - (fp - fn)) <= 1e-5 * abs(fp - fn)
    vals = [m_of(t)[0] for t in (0.0, 1.0, 2.0, 3.0)]
    third = vals[3] - 3 * vals[2] + 3 * vals[1] - vals[0]
    assert abs(third) <= 1e-9 * max(abs(v) for v in vals)
    ms = [m_of(t, sl, sm)[0] for t in (0.9, 1.0, 1.1)]
    assert ms[1] < ms[0] and ms[1] < ms[2]


def test_p13_decision_rule_cases():
    """Each condition of eq:uk+1_condition rejects on its own: u~ = u_k (no model decrease),
    u~ = u_k + 1.5 s_k (m_k(s~) > m_k(s_k) by the Galerkin property), a wild candidate (model rises);
    u~ = u_k + s_k is accepted exactly when the LM step is."""
    cfg, g, _, y, (l0, m0), (sl, sm), st = _lm_case()
    rng = np.random.default_rng(3)
    cases = {
        "identity": (l0, m0),
        "overshoot": (l0 + 1.5 * sl, m0 + 1.5 * sm),
        "wild": (l0 + 5.0 * rng.standard_normal(l0.shape), m0 + rng.standard_normal(m0.shape)),
        "lm": (l0 + sl, m0 + sm),
    }
    out = {k: O.safeguard(g, l0, m0, y, sl, sm, cl, cm, cfg.alpha, 0.1) for k, (cl, cm) in cases.items()}
    r = out["identity"][1][0]
    assert r["pred_cand"] == 0.0 and r["rho_cand"] == 0.0 and not r["accepted"]
    np.testing.assert_array_equal(out["identity"][0][0], l0 + sl)
    r = out["overshoot"][1][0]
    assert r["m_cand"] > r["m_lm"] and not r["accepted"]
    r = out["wild"][1][0]
    # f rises and the model rises more: rho > kappa although the candidate is worse; the model tests
    # (m_k(s~) <= m_k(s_k), pred > 0) reject it
    assert r["f_cand"] > r["f"] and r["pred_cand"] < 0 and r["m_cand"] > r["m_lm"] and not r["accepted"]
    assert out["lm"][1][0]["accepted"] == st["accepted"]


def test_p13_ground_truth_candidate_noise_free():
    """Noise-free data y = F(u†) and u~ = u†: f(u~) is the penalty alone, (alpha/2)||L u†||^2."""
    cfg = P.CONFIGS[2]
    n = 16
    g = P.geometry_desc(2, n_px=n, n_angles=8)
    lt, mt = P.make_phantom(2, n_px=n)
    y = O.forward(g, lt, mt)
    l0, m0 = P.initial_guess(n)
    sl, sm, _ = O.gn_cg_step(g, l0, m0, y, cfg.alpha, 0.0, 4)
    _, [r] = O.safeguard(g, l0, m0, y, sl, sm, lt, mt, cfg.alpha, 0.1)
    reg = 0.5 * cfg.alpha * (np.sum(O.laplacian(lt) ** 2) + np.sum(O.laplacian(mt) ** 2))
    assert abs(r["f_cand"] - reg) <= 1e-12 * max(reg, 1e-300) + 1e-14 * r["f"]


# ----------------------------------------------------------------------------- P14 LM solve (O9, N1)
def _tiny_lm(n_px=16, n_angles=8, noise=True):
    g = P.geometry_desc(2, n_px=n_px, n_angles=n_angles)
    lt, mt = P.make_phantom(2, n_px=n_px)
    yc = O.forward(g, lt, mt)
    y = P.poisson_noise(yc, 1e4, 3) if noise else yc
    l0, m0 = P.initial_guess(n_px)
    return g, (lt, mt), y, (l0, m0)


def test_p14_one_iteration_is_the_lm_wrap():
    g, _, y, (l0, m0) = _tiny_lm()
    (l1, m1), [sts] = O.lm_solve(g, l0, m0, y, 1, 6, 1e-3, beta0=0.05)
    sl, sm, st = O.gn_cg_step(g, l0, m0, y, 1e-3, 0.05, 6)
    for k in ("f", "pred", "f_trial", "rho", "beta_next"):
        assert sts[0][k] == st[k], k
    if st["accepted"]:
        np.testing.assert_allclose(l1, l0 + sl, rtol=0, atol=0)
    else:
        np.testing.assert_array_equal(l1, l0)


def test_p14_objective_chain_and_beta_rules():
    """Constant alpha: f_{k+1} = f(u_k + s_k) when iteration k is accepted, else f_k; the LM parameter
    follows the x10 (reject, >= beta_min) / x0.2 (rho > 0.75) rules from beta0."""
    g, _, y, (l0, m0) = _tiny_lm()
    _, [sts] = O.lm_solve(g, l0, m0, y, 6, 6, 1e-3, k_freeze=0, beta0=1.0)
    beta = 1.0
    for k in range(6):
        s = sts[k]
        if k + 1 < 6:
            want = s["f_trial"] if s["accepted"] else s["f"]
            assert abs(sts[k + 1]["f"] - want) <= 1e-12 * want
        if s["accepted"]:
            assert s["beta_next"] in (beta, 0.2 * beta)
            assert (s["beta_next"] == 0.2 * beta) == (s["rho"] > 0.75)
        else:
            assert s["beta_next"] == max(10.0 * beta, s["beta_min"])
        beta = s["beta_next"]
    assert sts[-1]["f_trial"] < sts[0]["f"]


def test_p14_alpha_continuation():
    """alpha_k = alpha0 / 5^min(k, k_freeze): R(u_k) / (||L lam_k||^2 + ||L mu_k||^2) = alpha_k / 2."""
    g, _, y, (l0, m0) = _tiny_lm()
    n, kf = 5, 2
    _, [sts] = O.lm_solve(g, l0, m0, y, n, 4, 1e-2, alpha_decay=5.0, k_freeze=kf, beta0=0.1)
    for k in range(n):
        (lk, mk), _ = O.lm_solve(g, l0, m0, y, k, 4, 1e-2, alpha_decay=5.0, k_freeze=kf, beta0=0.1)   # u_k
        q = np.sum(O.laplacian(lk) ** 2) + np.sum(O.laplacian(mk) ** 2)
        ak = 1e-2 / 5.0 ** min(k, kf)
        assert abs(sts[k]["reg"] - 0.5 * ak * q) <= 1e-12 * sts[k]["reg"]


def test_p14_box_projection():
    """Every iterate lies in the box; a box that never binds reproduces the unconstrained solve; a
    binding box changes the trajectory."""
    g, _, y, (l0, m0) = _tiny_lm()
    big = (-1e9, 1e9, -1e9, 1e9)
    (la, ma), sa = O.lm_solve(g, l0, m0, y, 3, 6, 1e-3, beta0=0.1)
    (lb, mb), sb = O.lm_solve(g, l0, m0, y, 3, 6, 1e-3, beta0=0.1, box=big)
    np.testing.assert_array_equal(la, lb)
    np.testing.assert_array_equal(ma, mb)
    box = (0.0, 1.2, 0.0, 0.4)
    (lc, mc), sc = O.lm_solve(g, l0, m0, y, 4, 6, 1e-3, beta0=0.1, box=box)
    assert lc.min() >= 0.0 and lc.max() <= 1.2 and mc.min() >= 0.0 and mc.max() <= 0.4
    (ld, md), _ = O.lm_solve(g, l0, m0, y, 4, 6, 1e-3, beta0=0.1)
    assert ld.min() < 0.0 or ld.max() > 1.2 or md.min() < 0.0 or md.max() > 0.4   # the box binds
    assert not np.array_equal(lc, ld)


def test_p14_converges_on_noise_free_data():
    """Noise-free data, alpha continuation 1e-2 / 5^k frozen at k = 4: the data misfit falls by more
    than two orders of magnitude in 8 iterations and the iterate approaches the phantom."""
    g, (lt, mt), y, (l0, m0) = _tiny_lm(noise=False)
    (l8, m8), [sts] = O.lm_solve(g, l0, m0, y, 8, 12, 1e-2, alpha_decay=5.0, k_freeze=4, beta0=0.0)
    assert sts[-1]["misfit"] < 1e-2 * sts[0]["misfit"]
    e0 = np.linalg.norm(np.concatenate([(l0 - lt).ravel(), (m0 - mt).ravel()]))
    e8 = np.linalg.norm(np.concatenate([(l8 - lt).ravel(), (m8 - mt).ravel()]))
    assert e8 < 0.5 * e0


# ----------------------------------------------------------------------------- P15 geometry priors (O10, N1)
def _prior_case(a1=0.3, a2=2.0):
    # N = 48: a one-pixel margin around the 0.2-pitch lattice leaves the diagonal gaps and the ring
    # outside the lattice unmasked (at N = 16 the margin covers everything)
    g, (lt, mt), y, (l0, m0) = _tiny_lm(n_px=48, n_angles=12)
    m1, m2 = (m.astype(np.float64) for m in P.prior_masks(2, n_px=g["n_px"]))
    return g, y, (l0, m0), (m1, m2, a1, a2)


def test_p15_masks_geometry():
    """The masks are 0 on (a margin around) every lattice position and 1 elsewhere: the phantom's
    emission lies entirely where the mask is 0, the background where it is 1."""
    for cid in (2, 3, 4):
        lt, mt = P.make_phantom(cid)
        m1, m2 = P.prior_masks(cid)
        assert set(np.unique(m1)) <= {0.0, 1.0} and np.array_equal(m1, m2)
        assert np.all(lt[m1 == 1.0] == 0.0)           # no rod pixel is penalised
        assert 0.2 < m1.mean() < 0.9


def test_p15_zero_weight_or_zero_mask_is_no_prior():
    g, y, (l0, m0), (m1, m2, a1, a2) = _prior_case()
    base = O.gn_cg_step(g, l0, m0, y, 1e-3, 0.05, 6)[2]
    for pr in ((m1, m2, 0.0, 0.0), (0 * m1, 0 * m2, a1, a2), (None, None, a1, a2)):
        st = O.gn_cg_step(g, l0, m0, y, 1e-3, 0.05, 6, prior=pr)[2]
        for k in ("f", "reg", "grad_norm", "pred", "f_trial"):
            assert st[k] == base[k], (k, pr[2])


def test_p15_objective_and_operator_closed_form():
    """f and H change by exactly the diagonal terms: f_P - f = a1/2 ||m1 lam||^2 + a2/2 ||m2 mu||^2
    and H_P p - H p = (a1 m1^2 p_lam, a2 m2^2 p_mu) (numpy, not the oracle's code)."""
    g, y, (l0, m0), (m1, m2, a1, a2) = _prior_case()
    st0 = O.gn_cg_step(g, l0, m0, y, 1e-3, 0.0, 0)[2]
    st1 = O.gn_cg_step(g, l0, m0, y, 1e-3, 0.0, 0, prior=(m1, m2, a1, a2))[2]
    want = 0.5 * a1 * np.sum((m1 * l0.astype(np.float64)) ** 2) + 0.5 * a2 * np.sum((m2 * m0.astype(np.float64)) ** 2)
    assert want > 1e-3 * st0["f"]
    assert abs((st1["f"] - st0["f"]) - want) <= 1e-12 * st1["f"]
    rng = np.random.default_rng(5)
    pl, pm = rng.standard_normal(l0.shape), rng.standard_normal(m0.shape)
    h0 = O.apply_H(g, l0, m0, 1e-3, 0.1, pl, pm)
    h1 = O.apply_H(g, l0, m0, 1e-3, 0.1, pl, pm, prior=(m1, m2, a1, a2))
    # (the threaded VJP's partial sums are added in a scheduling-dependent order: ~1e-11 relative)
    np.testing.assert_allclose(h1[0] - h0[0], a1 * m1 ** 2 * pl, rtol=0, atol=1e-9 * np.abs(h0[0]).max())
    np.testing.assert_allclose(h1[1] - h0[1], a2 * m2 ** 2 * pm, rtol=0, atol=1e-9 * np.abs(h0[1]).max())
    assert np.abs(a1 * m1 ** 2 * pl).max() > 1e-3 * np.abs(h0[0]).max()


def test_p15_gradient_is_finite_difference_of_f():
    """b = -grad f with the priors: <b, d> = -(f(u + h d) - f(u - h d)) / 2h (central differences of the
    objective, evaluated through the safeguard's f(u~))."""
    g, y, (l0, m0), pr = _prior_case()
    l0 = l0.astype(np.float64) + 0.05
    m0 = m0.astype(np.float64) + 0.02
    rng = np.random.default_rng(11)
    dl, dm = rng.standard_normal(l0.shape), 0.2 * rng.standard_normal(m0.shape)
    st = O.gn_cg_step(g, l0, m0, y, 1e-3, 0.0, 1, prior=pr)[2]
    # one CG step from 0: s = a b with a = <b,b>/<b,Hb> > 0, so <b, d> follows from s; use the pred
    # identity instead: with n_cg = 0, s = 0; recover b through the step of a 1-step solve
    sl, sm, st1 = O.gn_cg_step(g, l0, m0, y, 1e-3, 0.0, 1, prior=pr)
    bnorm = st1["grad_norm"]
    a = np.sqrt(np.sum(sl ** 2) + np.sum(sm ** 2)) / bnorm          # s = a b
    bl, bm = sl / a, sm / a
    z = np.zeros_like(l0)
    h = 1e-4

    def f_at(t):
        _, [r] = O.safeguard(g, l0, m0, y, z, z, l0 + t * dl, m0 + t * dm, 1e-3, 0.1, prior=pr)
        return r["f_cand"]
    fd = (f_at(h) - f_at(-h)) / (2 * h)
    assert abs(-(np.sum(bl * dl) + np.sum(bm * dm)) - fd) <= 1e-5 * abs(fd)
    assert st["grad_norm"] == bnorm


def test_p15_model_matches_f_to_first_order():
    """m_k with the prior rows of F~: d/dt m_k(t s)|0 = d/dt f(u + t s)|0, and m_k(t s) is quadratic."""
    g, y, (l0, m0), pr = _prior_case()
    rng = np.random.default_rng(13)
    dl, dm = 0.05 * rng.standard_normal(l0.shape), 0.01 * rng.standard_normal(m0.shape)
    z = np.zeros_like(l0)

    def m_of(t):
        _, [r] = O.safeguard(g, l0, m0, y, z, z, l0 + t * dl, m0 + t * dm, 1e-3, 0.1, prior=pr)
        return r["m_cand"], r["f_cand"]
    h = 1e-4
    (mp, fp), (mn, fn) = m_of(h), m_of(-h)
    assert abs((mp - mn) - (fp - fn)) <= 1e-5 * abs(fp - fn)
    vals = [m_of(t)[0] for t in (0.0, 1.0, 2.0, 3.0)]
    assert abs(vals[3] - 3 * vals[2] + 3 * vals[1] - vals[0]) <= 1e-9 * max(abs(v) for v in vals)


def test_p15_prior_continues_with_alpha():
    """alpha^(k) = (alpha1, alpha2) / 5^k: the regulariser of iteration k is
    alpha_k/2 ||L u_k||^2 + (alpha1_k/2) ||m1 lam_k||^2 + (alpha2_k/2) ||m2 mu_k||^2."""
    g, y, (l0, m0), (m1, m2, a1, a2) = _prior_case()
    n, kf = 4, 2
    pr = (m1, m2, a1, a2)
    _, [sts] = O.lm_solve(g, l0, m0, y, n, 4, 1e-2, alpha_decay=5.0, k_freeze=kf, beta0=0.1, prior=pr)
    for k in range(n):
        (lk, mk), _ = O.lm_solve(g, l0, m0, y, k, 4, 1e-2, alpha_decay=5.0, k_freeze=kf, beta0=0.1, prior=pr)
        c = 1.0 / 5.0 ** min(k, kf)
        q = np.sum(O.laplacian(lk) ** 2) + np.sum(O.laplacian(mk) ** 2)
        want = 0.5 * 1e-2 * c * q + 0.5 * a1 * c * np.sum((m1 * lk) ** 2) + 0.5 * a2 * c * np.sum((m2 * mk) ** 2)
        assert abs(sts[k]["reg"] - want) <= 1e-12 * want, k


def test_p15_prior_pulls_masked_emission_down():
    """On noise-free data a strong emission prior lowers the emission outside the lattice positions
    relative to the unpenalised solve (the prior does what the paper uses it for)."""
    g, y, (l0, m0), (m1, m2, a1, a2) = _prior_case()
    (l_a, _), _ = O.lm_solve(g, l0, m0, y, 4, 8, 1e-3, beta0=0.01)
    (l_b, _), _ = O.lm_solve(g, l0, m0, y, 4, 8, 1e-3, beta0=0.01, prior=(m1, m2, 50.0, 0.0))
    out = m1 == 1.0
    assert np.sum(l_b[out] ** 2) < 0.5 * np.sum(l_a[out] ** 2)


# ----------------------------------------------------------------------------- P16 SGP inner solver (O11, N1)
def _sgp_case(n_px=8, n_angles=6):
    g = P.geometry_desc(2, n_px=n_px, n_angles=n_angles)
    lt, mt = P.make_phantom(2, n_px=n_px)
    y = O.forward(g, lt, mt)
    l0, m0 = P.initial_guess(n_px)
    return g, y, (l0.astype(np.float64), m0.astype(np.float64))


def _grad_b(g, l0, m0, y, alpha):
    """b = -grad f(u) from a one-step CG solve (s = a b with a = <b,b>/<b,Hb>), independent of SGP."""
    sl, sm, st = O.gn_cg_step(g, l0, m0, y, alpha, 0.0, 1)
    a = np.sqrt(np.sum(sl ** 2) + np.sum(sm ** 2)) / st["grad_norm"]
    return sl / a, sm / a


def test_p16_sgp_iterates_feasible_and_monotone():
    """u + s stays in the box; with beta = 0, pred = -q(s) and the exact line search makes q decrease
    at every iteration."""
    g, y, (l0, m0) = _sgp_case()
    box = (0.0, 0.9, 0.0, 0.35)
    preds = []
    for n in range(1, 8):
        sl, sm, st = O.lm_step_box(g, l0, m0, y, 1e-3, 0.0, n, box)
        assert np.all(l0 + sl >= box[0] - 1e-15) and np.all(l0 + sl <= box[1] + 1e-15)
        assert np.all(m0 + sm >= box[2] - 1e-15) and np.all(m0 + sm <= box[3] + 1e-15)
        preds.append(st["pred"])
    assert all(b >= a - 1e-12 * abs(a) for a, b in zip(preds, preds[1:])), preds
    assert preds[-1] > preds[0] > 0


def test_p16_sgp_matches_lbfgsb_on_the_box_qp():
    """Converged SGP = the minimiser of q(s) = 1/2 s^T H s - b^T s over the box from scipy's L-BFGS-B
    (H p through O.apply_H, b from an independent CG step)."""
    from scipy.optimize import minimize
    g, y, (l0, m0) = _sgp_case()
    alpha = 1e-3
    box = (0.0, 0.9, 0.0, 0.35)
    bl, bm = _grad_b(g, l0, m0, y, alpha)
    b = np.concatenate([bl.ravel(), bm.ravel()])
    n = bl.size

    def q_and_grad(x):
        hl, hm = O.apply_H(g, l0, m0, alpha, 0.0, x[:n].reshape(bl.shape), x[n:].reshape(bl.shape))
        hx = np.concatenate([hl.ravel(), hm.ravel()])
        return 0.5 * x @ hx - b @ x, hx - b
    lo = np.concatenate([box[0] - l0.ravel(), box[2] - m0.ravel()])
    hi = np.concatenate([box[1] - l0.ravel(), box[3] - m0.ravel()])
    ref = minimize(q_and_grad, np.zeros(2 * n), jac=True, method="L-BFGS-B", bounds=list(zip(lo, hi)),
                   options=dict(maxiter=5000, ftol=1e-15, gtol=1e-12))
    # alpha = 1e-3 leaves H ill-conditioned: gradient projection needs ~3000 iterations here
    sl, sm, st = O.lm_step_box(g, l0, m0, y, alpha, 0.0, 3000, box)
    x = np.concatenate([sl.ravel(), sm.ravel()])
    assert q_and_grad(x)[0] <= ref.fun + 1e-10 * abs(ref.fun)
    assert np.linalg.norm(x - ref.x) <= 1e-4 * np.linalg.norm(ref.x)
    assert np.any(np.isclose(x, lo)) or np.any(np.isclose(x, hi))      # the box binds


def test_p16_sgp_without_binding_box_is_the_newton_step():
    """A box far away: SGP converges to the unconstrained minimiser H^{-1} b, as CG does."""
    g, y, (l0, m0) = _sgp_case()
    box = (-1e3, 1e3, -1e3, 1e3)
    sl, sm, _ = O.lm_step_box(g, l0, m0, y, 1e-3, 0.0, 3000, box)
    cl, cm, _ = O.gn_cg_step(g, l0, m0, y, 1e-3, 0.0, 400)
    x, c = np.concatenate([sl.ravel(), sm.ravel()]), np.concatenate([cl.ravel(), cm.ravel()])
    assert np.linalg.norm(x - c) <= 1e-4 * np.linalg.norm(c)


def test_p16_lm_solve_with_sgp_decreases_f_inside_the_box():
    g, y, (l0, m0) = _sgp_case(n_px=16, n_angles=8)
    box = (0.0, 1.6, 0.0, 0.6)
    (lk, mk), [sts] = O.lm_solve(g, l0, m0, y, 5, 10, 1e-3, beta0=0.01, box=box, inner="sgp")
    assert sts[-1]["f_trial"] < 0.2 * sts[0]["f"]
    assert lk.min() >= box[0] and lk.max() <= box[1] and mk.min() >= box[2] and mk.max() <= box[3]


# ----------------------------------------------------------------------------- P17 linear constraint lam <= c mu (O12, N1)
def test_p17_projection_is_the_euclidean_projection():
    """Variational inequality <x - P x, z - P x> <= 0 for every feasible z (which characterises the
    projection onto a convex set), feasibility, idempotence; c = 0 is the plain box clamp."""
    rng = np.random.default_rng(17)
    box = (0.0, 2.0, 0.0, 1.0, 2.5)
    x = rng.uniform(-1.0, 3.0, size=4000)
    y = rng.uniform(-0.5, 1.5, size=4000)
    pl, pm = O.project(x, y, box)
    assert np.all((pl >= 0) & (pl <= 2) & (pm >= 0) & (pm <= 1) & (pl <= 2.5 * pm + 1e-12))
    zl = rng.uniform(0, 2, size=20000)
    zm = rng.uniform(0, 1, size=20000)
    ok = zl <= 2.5 * zm
    zl, zm = zl[ok][:3000], zm[ok][:3000]
    vi = (x - pl)[:, None] * (zl[None, :] - pl[:, None]) + (y - pm)[:, None] * (zm[None, :] - pm[:, None])
    assert vi.max() <= 1e-12
    ql, qm = O.project(pl, pm, box)
    np.testing.assert_allclose(ql, pl, rtol=0, atol=1e-15)
    np.testing.assert_allclose(qm, pm, rtol=0, atol=1e-15)
    cl, cm = O.project(x, y, box[:4])
    np.testing.assert_array_equal(cl, np.clip(x, 0, 2))
    np.testing.assert_array_equal(cm, np.clip(y, 0, 1))
    assert np.any(pl == 2.5 * pm) and np.any(pl < 2.5 * pm)        # the constraint binds somewhere


def test_p17_lm_solve_respects_the_constraint():
    """Every LM iterate (CG + projection, and SGP) satisfies lam <= c mu; a non-binding c changes
    nothing (bitwise)."""
    g, y, (l0, m0) = _sgp_case(n_px=16, n_angles=8)
    for inner in ("cg", "sgp"):
        (lk, mk), [sts] = O.lm_solve(g, l0, m0, y, 4, 8, 1e-3, beta0=0.01, box=(0.0, 1.6, 0.0, 0.6, 3.0),
                                     inner=inner)
        assert np.all(lk <= 3.0 * mk + 1e-12) and sts[-1]["f_trial"] < sts[0]["f"]
        assert np.any(np.isclose(lk, 3.0 * mk) & (lk > 0))
        # mu >= 0.01 in the box, so lam <= 1e6 mu never binds
        (la, ma), [sa] = O.lm_solve(g, l0, m0, y, 3, 6, 1e-3, beta0=0.01, box=(0.0, 1.6, 0.01, 0.6), inner=inner)
        (lb, mb), [sb] = O.lm_solve(g, l0, m0, y, 3, 6, 1e-3, beta0=0.01, box=(0.0, 1.6, 0.01, 0.6, 1e6),
                                    inner=inner)
        np.testing.assert_array_equal(la, lb)
        assert [s["f"] for s in sa] == [s["f"] for s in sb]


# ----------------------------------------------------------------------------- P18 model variant (O13, N3)
# the collimator response r and the vertical correction c of eq:d_fwd_model as
# functions of the emission point's distance to the detector (reading R-N3)
VAR = dict(det_radius=1.6, c_slope=0.05, r_slope=0.35)


def test_p18_tables():
    """c_i = 1 + c_slope d_i >= 1 grows with the distance d_i = det_radius - t_i to the detector (PAPER.md:141:
    'c >= 1 ... far-away emissions'); the response W_j(d) sums to 1 over the sub-rays at every distance
    (a probability split over the detector's sub-rays), is symmetric in j, and widens with d."""
    g = small(n_px=32, J=5, **VAR)
    t = O.tables(g)
    h, delta, T = t["tlat"]
    v = O.variant_tables(g)
    n_t = v["c"].size
    ti = -T + (np.arange(n_t) + 0.5) * delta
    d = VAR["det_radius"] - ti
    assert np.all(d > 0)
    np.testing.assert_allclose(v["c"], 1 + VAR["c_slope"] * d, rtol=1e-15)
    assert np.all(np.diff(v["c"]) < 0) and v["c"].min() >= 1.0
    W = v["w"]
    assert np.abs(W.sum(0) - 1).max() <= 4e-16
    assert np.array_equal(W, W[::-1])
    assert np.all(np.diff(W[2]) > 0)            # the centre sub-ray's share shrinks with distance (i up = nearer)
    # the centre share at distance 0 is the base model's weight at sigma0
    g0 = small(n_px=32, J=5, det_radius=1.6, c_slope=0.0, r_slope=0.0)
    np.testing.assert_allclose(O.variant_tables(g0)["w"][:, 0], t["weights"], rtol=1e-15)


def test_p18_reduces_to_base_model():
    """Slopes 0: the variant's code path reproduces the base model (the response moves inside the ray
    sum: 1e-13 rel); mu = 0: c drops out exactly (exp(-c 0) = 1), whatever its slope."""
    g = small(n_px=20, J=3)
    lam, mu = rand_img(g, 1, 0, 1.5), rand_img(g, 2, 0, 0.6)
    dl, dm = rand_img(g, 3, -1, 1), rand_img(g, 4, -0.1, 0.1)
    g0 = dict(g, det_radius=1.6, c_slope=0.0, r_slope=0.0)
    y, dy = O.jvp(g, lam, mu, dl, dm, with_y=True)
    y0, dy0 = O.jvp(g0, lam, mu, dl, dm, with_y=True)
    assert rel_l2(y0, y) <= 1e-13 and rel_l2(dy0, dy) <= 1e-13
    w = np.random.default_rng(5).standard_normal(O.sino_shape(g))
    gl, gm = O.vjp(g, lam, mu, w)
    gl0, gm0 = O.vjp(g0, lam, mu, w)
    assert rel_l2(gl0, gl) <= 1e-13 and rel_l2(gm0, gm) <= 1e-13
    z = np.zeros_like(mu)
    ya = O.forward(dict(g, det_radius=1.6, c_slope=0.0, r_slope=0.3), lam, z)
    yb = O.forward(dict(g, det_radius=1.6, c_slope=0.4, r_slope=0.3), lam, z)
    assert np.array_equal(ya, yb)


def test_p18_c_attenuated_disk_closed_form():
    """c alone (J = 1, so W = 1): uniform disk lam0 = 1, mu0 = 0.5, R = 0.5, chord [-l, l] along the ray,
    g(s) = int_{-l}^{l} exp(-c(t) mu0 (l - t)) dt with c(t) = 1 + c_slope (det_radius - t): the correction
    multiplies the whole path from the emission point to the detector (eq:d_fwd_model).  Quadrature by
    scipy; first-order convergence in h as P4."""
    from scipy.integrate import quad
    D, kc, mu0, R = 1.6, 0.2, 0.5, 0.5
    means = []
    for N in (128, 256):
        g = dict(_disk_geom(N), det_radius=D, c_slope=kc, r_slope=0.0)
        lam, mu = P.disk_phantom(N, R, 1.0, mu0)
        y = O.forward(g, lam, mu)[0]
        s = O.tables(g)["offsets"][0, :, 0]
        sel = np.abs(s) <= 0.9 * R
        ref = []
        for sv in s[sel]:
            l = math.sqrt(R * R - sv * sv)
            ref.append(quad(lambda t: math.exp(-(1 + kc * (D - t)) * mu0 * (l - t)), -l, l, epsabs=1e-13)[0])
        ref = np.array(ref)
        err = np.abs(y[:, 0, sel] - ref) / ref
        assert err.max() <= 1.5e-2
        means.append(err.mean())
        # the wrong reading c(t) = 1 + c_slope (det_radius + t) (distance from the far side) is far off
        wrong = np.array([quad(lambda t: math.exp(-(1 + kc * (D + t)) * mu0 * (l - t)), -l, l)[0]
                          for l in np.sqrt(R * R - s[sel] ** 2)])
        assert (np.abs(y[:, 0, sel] - wrong) / wrong).mean() > 5 * err.mean()
    assert means[0] / means[1] >= 1.5


def test_p18_r_uniform_disk_closed_form():
    """r alone (mu = 0, J = 5): a uniform emitting disk gives y_d = sum_j int_{chord_j} W_j(det_radius - t) dt
    with the sub-ray offsets of O1 (scipy quadrature over each sub-ray's chord; first-order convergence)."""
    from scipy.integrate import quad
    D, kr, R, J = 1.6, 0.6, 0.5, 5
    p = 2.0 / 90
    s0 = 0.4 * p
    dj = np.array([(2 * j + 1 - J) / (2 * J) * p for j in range(J)])

    def Wj(j, d):
        q = np.exp(-dj ** 2 / (2 * (s0 * (1 + kr * d)) ** 2))
        return q[j] / q.sum()
    means = []
    for N in (128, 256):
        g = dict(_disk_geom(N), n_subrays=J, det_radius=D, c_slope=0.0, r_slope=kr)
        lam, mu = P.disk_phantom(N, R, 1.0, 0.0)
        y = O.forward(g, lam, mu)[0]
        s = O.tables(g)["offsets"][0, :, J // 2]
        sel = np.abs(s) <= 0.85 * R
        ref = []
        for sv in s[sel]:
            tot = 0.0
            for j in range(J):
                l = math.sqrt(max(R * R - (sv + dj[j]) ** 2, 0.0))
                tot += quad(lambda t: Wj(j, D - t), -l, l, epsabs=1e-14)[0]
            ref.append(tot)
        ref = np.array(ref)
        err = np.abs(y[:, 0, sel] - ref) / ref
        assert err.max() <= 1.5e-2
        means.append(err.mean())
    assert means[0] / means[1] >= 1.5


def test_p18_r_invariant_for_fields_constant_across_rays():
    """theta = 0 rays run along x; an emission field that depends on x only is seen identically by every
    sub-ray of a detector, so sum_j W_j(d) = 1 makes the detector reading independent of r_slope
    (catches a response that is not normalised per distance, or applied per ray instead of per sample)."""
    N = 32
    g = dict(n_px=N, n_angles=4, n_banks=2, n_det=9, n_subrays=5, subray_sigma=0.4, step_px=0.5,
             bank1_shift=0.0, batch=1, det_radius=1.6, c_slope=0.0)
    x = np.random.default_rng(3).uniform(0.2, 1.5, N)
    lam = np.tile(x, (N, 1))[None]              # lam[j][i] = x[i]: constant along y
    mu = np.zeros_like(lam)
    ya = O.forward(dict(g, r_slope=0.0), lam, mu)[0]
    yb = O.forward(dict(g, r_slope=0.8), lam, mu)[0]
    inner = slice(1, 8)                         # detectors whose sub-rays all lie inside the grid
    assert np.abs(ya[0, 0, inner] - yb[0, 0, inner]).max() <= 1e-13 * np.abs(ya).max()
    assert np.abs(ya[1, 0] - yb[1, 0]).max() > 1e-4 * np.abs(ya).max()   # at 90 deg the field varies across rays


def test_p18_c_lowers_every_reading():
    """mu > 0 everywhere: a larger vertical correction lengthens every path, so every reading falls."""
    g = small(n_px=20, J=3)
    lam, mu = rand_img(g, 1, 0.2, 1.5), rand_img(g, 2, 0.1, 0.6)
    ya = O.forward(dict(g, det_radius=1.6, c_slope=0.02, r_slope=0.2), lam, mu)
    yb = O.forward(dict(g, det_radius=1.6, c_slope=0.08, r_slope=0.2), lam, mu)
    assert np.all(yb < ya)


def test_p18_jvp_central_differences():
    g = small(n_px=24, n_angles=10, J=3, n_det=11, **VAR)
    lam, mu = rand_img(g, 10, 0, 1.5), rand_img(g, 11, 0, 0.6)
    un = math.sqrt(np.sum(lam ** 2) + np.sum(mu ** 2))
    for k in range(20):
        rng = np.random.default_rng(200 + k)
        dl = rng.uniform(-1, 1, lam.shape)
        dm = rng.uniform(-0.1, 0.1, mu.shape)
        eps = 1e-6 * un / math.sqrt(np.sum(dl ** 2) + np.sum(dm ** 2))
        fd = (O.forward(g, lam + eps * dl, mu + eps * dm) - O.forward(g, lam - eps * dl, mu - eps * dm)) / (2 * eps)
        assert rel_l2(O.jvp(g, lam, mu, dl, dm), fd) <= 1e-7


def test_p18_adjoint_identity_and_dense_transpose():
    g = small(n_px=12, n_angles=6, J=2, n_det=9, **VAR)
    for k in range(100):
        rng = np.random.default_rng(3000 + k)
        lam = rng.uniform(0, 1.5, O.img_shape(g))
        mu = rng.uniform(0, 0.6, O.img_shape(g))
        vl, vm = rng.standard_normal(O.img_shape(g)), rng.standard_normal(O.img_shape(g))
        w = rng.standard_normal(O.sino_shape(g))
        jv = O.jvp(g, lam, mu, vl, vm)
        gl, gm = O.vjp(g, lam, mu, w)
        assert abs(np.sum(jv * w) - np.sum(vl * gl) - np.sum(vm * gm)) <= 1e-10 * np.linalg.norm(jv) * np.linalg.norm(w)
    g = dict(n_px=8, n_angles=4, n_banks=2, n_det=5, n_subrays=3, subray_sigma=0.4, step_px=0.5,
             bank1_shift=0.0, batch=1, **dict(VAR, det_radius=2.0))   # det_radius >= T = 1.75 at N = 8
    rng = np.random.default_rng(6)
    lam, mu = rng.uniform(0.2, 1.5, (1, 8, 8)), rng.uniform(0.1, 0.6, (1, 8, 8))
    npx = 64
    Jd = np.stack([O.jvp(g, lam, mu, e[:npx].reshape(1, 8, 8), e[npx:].reshape(1, 8, 8)).ravel()
                   for e in np.eye(2 * npx)], axis=1)
    ns = Jd.shape[0]
    JT = np.stack([np.concatenate([x.ravel() for x in O.vjp(g, lam, mu, e.reshape(O.sino_shape(g)))])
                   for e in np.eye(ns)], axis=0)
    assert np.abs(JT - Jd).max() <= 1e-12 * np.abs(Jd).max()


# ----------------------------------------------------------------------------- P19 pixel basis (O14, R-pb)
PB = dict(pixel_basis=1)


def _clip_len(x0, x1, y0, y1, p0, om):
    """length of the line p0 + t om inside the closed box [x0,x1] x [y0,y1] (slab clipping)"""
    tin, tout = -np.inf, np.inf
    for k, (a, b) in enumerate(((x0, x1), (y0, y1))):
        if om[k] == 0.0:
            if not (a <= p0[k] <= b):
                return 0.0
            continue
        t1, t2 = (a - p0[k]) / om[k], (b - p0[k]) / om[k]
        tin, tout = max(tin, min(t1, t2)), min(tout, max(t1, t2))
    return max(0.0, tout - tin)


@pytest.mark.parametrize("N", [7, 8, 13])
def test_p19_crossings_match_per_pixel_clipping(N):
    """The traversal's pixels and lengths equal, pixel by pixel, the clipped length of the line in each
    pixel box (brute force over all N^2 pixels, eq:d_fwd_model's d_{m,n,k} as 'the distances a ray
    covers within pixel k'); the pixels come in order of t and each is an edge or corner
    neighbour of the previous one; the lengths sum to the chord of the square."""
    h = 2.0 / N
    rng = np.random.default_rng(N)
    for k in range(60):
        phi = rng.uniform(0, 2 * np.pi) if k > 3 else k * np.pi / 2 + 0.1
        c, s = math.cos(phi), math.sin(phi)
        sigma = rng.uniform(-1.3, 1.3)
        pix, ln, tm = O.pb_crossings(N, c, s, sigma)
        p0, om = (-sigma * s, sigma * c), (c, s)
        ref = np.zeros(N * N)
        for r in range(N):
            for q in range(N):
                ref[r * N + q] = _clip_len(-1 + q * h, -1 + (q + 1) * h, -1 + r * h, -1 + (r + 1) * h, p0, om)
        got = np.zeros(N * N)
        np.add.at(got, pix, ln)
        assert len(set(pix.tolist())) == len(pix)
        assert np.abs(got - ref).max() <= 1e-12
        assert np.all(np.diff(tm) > 0)
        rows, cols = pix // N, pix % N
        assert np.all(np.maximum(np.abs(np.diff(rows)), np.abs(np.diff(cols))) == 1)
        chord = _clip_len(-1, 1, -1, 1, p0, om)
        assert abs(ln.sum() - chord) <= 1e-12


def test_p19_uniform_square_is_the_chord():
    """mu = 0, lam = 1 on the whole grid: every ray reads the chord of the square [-1,1]^2, in closed
    form 2 at theta = 0, pi/2 (|s| < 1) and 2 sqrt2 - 2|s| at theta = pi/4 (|s| < sqrt2); y = sum_j w_j chord.
    (J = 2: no sub-ray runs exactly along the square's edge, a measure-zero case either reading allows.)"""
    g = small(n_px=16, n_angles=8, J=2, n_det=21, **PB)
    lam, mu = np.ones(O.img_shape(g)), np.zeros(O.img_shape(g))
    y = O.forward(g, lam, mu)[0]
    T = O.tables(g)
    w, off = T["weights"], T["offsets"]
    for a, chord in ((0, lambda s: np.where(np.abs(s) < 1, 2.0, 0.0)),
                     (2, lambda s: np.where(np.abs(s) < 1, 2.0, 0.0)),
                     (1, lambda s: np.maximum(2 * math.sqrt(2) - 2 * np.abs(s), 0.0))):
        for b in range(2):
            ref = (chord(off[b]) * w[None, :]).sum(axis=1)
            assert np.abs(y[a, b] - ref).max() <= 1e-12


def test_p19_mu0_is_the_line_integral_of_the_pixel_field():
    """mu = 0: the reading is the line integral of the piecewise-constant emission field, checked
    against brute-force sampling of that field along each sub-ray (step 2e-5: error <= 2N jumps x step
    x max), weighted by w_j.  (J = 2 and 5 angles: no ray runs along a pixel edge, where the two
    readings may pick either side.)"""
    g = small(n_px=10, n_angles=5, J=2, n_det=8, **PB)
    N = 10
    h = 2.0 / N
    lam = rand_img(g, 19, 0.2, 1.5)
    y = O.forward(g, lam, np.zeros_like(lam))[0]
    T = O.tables(g)
    dt = 2e-5
    t = np.arange(-1.5, 1.5, dt) + dt / 2
    for a in range(5):
        for b in range(2):
            c, s = T["dirs"][a, b]
            for d in range(8):
                ref = 0.0
                for j in range(2):
                    sig = T["offsets"][b, d, j]
                    x, yy = -sig * s + t * c, sig * c + t * s
                    ins = (np.abs(x) < 1) & (np.abs(yy) < 1)
                    col = np.clip(np.floor((x[ins] + 1) / h).astype(int), 0, N - 1)
                    row = np.clip(np.floor((yy[ins] + 1) / h).astype(int), 0, N - 1)
                    ref += T["weights"][j] * lam[0, row, col].sum() * dt
                assert abs(y[a, b, d] - ref) <= 2 * (2 * N + 2) * dt * lam.max()


@pytest.mark.parametrize("mu0", [0.7, 3.0])
def test_p19_attenuated_square_bracketed_by_the_exact_integral(mu0):
    """lam = 1 on the square, mu = mu0 on its left half (x < 0): the exact attenuated transform along
    theta = 0 (detector at +x) is 1 + (1 - e^{-mu0})/mu0 for |s| < 1, along theta = pi (detector at
    -x) e^{-mu0} + (1 - e^{-mu0})/mu0.  Per pixel the midpoint reading l e^{-mu (A + l/2)} and the exact
    e^{-mu A} (1 - e^{-mu l})/mu differ by the factor sinh(x/2)/(x/2), x = mu l, so
    y <= exact <= y sinh(x/2)/(x/2) at x = mu0 h (a dropped 1/2, a reversed direction or a missing term
    leaves the bracket); the readings also equal the geometric series of the midpoint terms."""
    N = 16
    h = 2.0 / N
    g = small(n_px=N, n_angles=2, J=1, n_det=15, **PB)
    lam = np.ones(O.img_shape(g))
    mu = np.zeros(O.img_shape(g))
    mu[0, :, : N // 2] = mu0
    y = O.forward(g, lam, mu)[0]
    s = O.tables(g)["offsets"][0, :, 0]
    sel = np.abs(s) < 1 - 1e-9
    x = mu0 * h
    fac = math.sinh(x / 2) / (x / 2)
    e0 = 1 + (1 - math.exp(-mu0)) / mu0
    e1 = math.exp(-mu0) + (1 - math.exp(-mu0)) / mu0
    assert abs(e0 - e1) > 0.05
    for a, b, ex in ((0, 0, e0), (0, 1, e1), (1, 0, e1), (1, 1, e0)):
        yy = y[a, b, sel]
        assert np.all(yy <= ex * (1 + 1e-12))
        assert np.all(ex <= yy * fac * (1 + 1e-12))
        # and exactly: the N/2 attenuating pixels of length h form a geometric series
        geo = h * math.exp(-x / 2) * math.expm1(-N // 2 * x) / math.expm1(-x)
        mid = (1.0 if ex == e0 else math.exp(-mu0)) + geo
        assert np.abs(yy - mid).max() <= 1e-13


def test_p19_rotation_invariance():
    """90 and 180 degree rotations of the images shift the sinogram by nA/4, nA/2 angles (J = 2: no ray
    on a pixel edge, where the midpoint rule picks the upper / right pixel and the symmetry is lost)."""
    g = small(n_px=14, n_angles=8, J=2, n_det=13, **PB)
    lam, mu = rand_img(g, 31), rand_img(g, 32, 0, 0.8)
    nA = 8
    y = O.forward(g, lam, mu)
    r90 = lambda im: np.transpose(im, (0, 2, 1))[:, :, ::-1]
    assert rel_l2(O.forward(g, r90(lam), r90(mu)), np.roll(y, nA // 4, axis=1)) <= 1e-12
    assert rel_l2(O.forward(g, lam[:, ::-1, ::-1], mu[:, ::-1, ::-1]), np.roll(y, nA // 2, axis=1)) <= 1e-12


@pytest.mark.parametrize("var", [False, True])
def test_p19_jvp_central_differences(var):
    g = small(n_px=20, n_angles=10, J=3, n_det=11, **PB, **(VAR if var else {}))
    lam, mu = rand_img(g, 40, 0, 1.5), rand_img(g, 41, 0, 0.6)
    un = math.sqrt(np.sum(lam ** 2) + np.sum(mu ** 2))
    for k in range(10):
        rng = np.random.default_rng(400 + k)
        dl = rng.uniform(-1, 1, lam.shape)
        dm = rng.uniform(-0.1, 0.1, mu.shape)
        eps = 1e-6 * un / math.sqrt(np.sum(dl ** 2) + np.sum(dm ** 2))
        fd = (O.forward(g, lam + eps * dl, mu + eps * dm) - O.forward(g, lam - eps * dl, mu - eps * dm)) / (2 * eps)
        assert rel_l2(O.jvp(g, lam, mu, dl, dm), fd) <= 1e-7
    # the lambda part of the JVP is the forward of dlam (linear in lambda)
    dl = rand_img(g, 42, -1, 1)
    assert rel_l2(O.jvp(g, lam, mu, dl, np.zeros_like(mu)), O.forward(g, dl, mu)) <= 1e-13


@pytest.mark.parametrize("var", [False, True])
def test_p19_adjoint_identity_and_dense_transpose(var):
    g = small(n_px=12, n_angles=6, J=2, n_det=9, **PB, **(VAR if var else {}))
    for k in range(50):
        rng = np.random.default_rng(5000 + k)
        lam = rng.uniform(0, 1.5, O.img_shape(g))
        mu = rng.uniform(0, 0.6, O.img_shape(g))
        vl, vm = rng.standard_normal(O.img_shape(g)), rng.standard_normal(O.img_shape(g))
        w = rng.standard_normal(O.sino_shape(g))
        jv = O.jvp(g, lam, mu, vl, vm)
        gl, gm = O.vjp(g, lam, mu, w)
        assert abs(np.sum(jv * w) - np.sum(vl * gl) - np.sum(vm * gm)) <= 1e-10 * np.linalg.norm(jv) * np.linalg.norm(w)
    g = dict(n_px=6, n_angles=4, n_banks=2, n_det=5, n_subrays=2, subray_sigma=0.4, step_px=0.5,
             bank1_shift=0.0, batch=1, **PB, **(dict(VAR, det_radius=2.5) if var else {}))
    rng = np.random.default_rng(7)
    lam, mu = rng.uniform(0.2, 1.5, (1, 6, 6)), rng.uniform(0.1, 0.6, (1, 6, 6))
    npx = 36
    Jd = np.stack([O.jvp(g, lam, mu, e[:npx].reshape(1, 6, 6), e[npx:].reshape(1, 6, 6)).ravel()
                   for e in np.eye(2 * npx)], axis=1)
    JT = np.stack([np.concatenate([x.ravel() for x in O.vjp(g, lam, mu, e.reshape(O.sino_shape(g)))])
                   for e in np.eye(Jd.shape[0])], axis=0)
    assert np.abs(JT - Jd).max() <= 1e-12 * np.abs(Jd).max()


def test_p19_variant_reduces_and_changes():
    """With the O13 response at zero slopes the pixel basis is unchanged (sum_j W_j = 1 and w_j = W_j(d)
    at r_slope 0, c = 1); the variant alone at nonzero c lowers every reading (c >= 1 in the exponent)."""
    g = small(n_px=16, n_angles=6, J=3, n_det=11, **PB)
    lam, mu = rand_img(g, 50, 0.1, 1.2), rand_img(g, 51, 0.05, 0.6)
    y0 = O.forward(g, lam, mu)
    y1 = O.forward(dict(g, det_radius=1.6, c_slope=0.0, r_slope=0.0), lam, mu)
    assert np.abs(y1 - y0).max() <= 1e-13 * np.abs(y0).max()
    yc = O.forward(dict(g, det_radius=1.6, c_slope=0.1, r_slope=0.0), lam, mu)
    assert np.all(yc[y0 > 0] < y0[y0 > 0])


def test_p19_attenuated_disk_converges():
    """The north star's disk closed form g(s) = (1 - e^{-mu0 2 sqrt(R^2 - s^2)})/mu0 for the pixelated
    (area-fraction) disk: the pixel-basis readings converge to it at first order in h."""
    means = []
    for N in (64, 128, 256):
        g = dict(_disk_geom(N), **PB)
        lam, mu = P.disk_phantom(N, 0.5, 1.0, 0.5)
        y = O.forward(g, lam, mu)[0]
        s = O.tables(g)["offsets"][0, :, 0]
        sel = np.abs(s) <= 0.9 * 0.5
        chord = 2 * np.sqrt(np.maximum(0.25 - s ** 2, 0))
        ref = (1 - np.exp(-0.5 * chord)) / 0.5
        err = np.abs(y[:, 0, sel] - ref[sel]) / ref[sel]
        assert err.max() <= 0.3 * 64 / N
        means.append(err.mean())
    assert means[0] / means[1] >= 1.5 and means[1] / means[2] >= 1.5


def test_p19_cg_equals_dense_solve():
    N = 6
    g = dict(n_px=N, n_angles=6, n_banks=2, n_det=9, n_subrays=2, subray_sigma=0.4, step_px=0.5,
             bank1_shift=0.0, batch=1, **PB)
    rng = np.random.default_rng(12)
    lam, mu = rng.uniform(0.3, 1.2, (1, N, N)), rng.uniform(0.1, 0.5, (1, N, N))
    y = O.forward(g, rng.uniform(0.3, 1.2, (1, N, N)), rng.uniform(0.1, 0.5, (1, N, N)))
    alpha, beta = 1e-2, 0.05
    Jd, Ld, H = _dense_H(g, lam, mu, alpha, beta)
    r = (O.forward(g, lam, mu) - y).ravel()
    u = np.concatenate([lam.ravel(), mu.ravel()])
    b = -(Jd.T @ r + alpha * Ld.T @ (Ld @ u))
    sl, sm, st = O.gn_cg_step(g, lam, mu, y, alpha, beta, 200)
    assert rel_l2(np.concatenate([sl.ravel(), sm.ravel()]), np.linalg.solve(H, b)) <= 1e-8
