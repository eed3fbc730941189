"""ctypes wrapper of the fp64 CPU oracle (oracle/pget_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
path (paper_2604_26745_b200) never imports it and shares no code with it.

Every function takes the geometry descriptor as a dict with the fields of
pget_geometry_desc and numpy arrays (any float dtype; widened to fp64 exactly).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pget_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

ST_CG = 16  # offset of the CG residual norms in the stats vector


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (fp64, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Desc(C.Structure):
    _fields_ = [("n_px", C.c_int), ("n_angles", C.c_int), ("n_banks", C.c_int),
                ("n_det", C.c_int), ("n_subrays", C.c_int), ("subray_sigma", C.c_double),
                ("step_px", C.c_double), ("bank1_shift", C.c_double), ("batch", C.c_int),
                ("det_radius", C.c_double), ("c_slope", C.c_double), ("r_slope", C.c_double),
                ("pixel_basis", C.c_int)]


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        P = C.c_void_p
        for name, args in [
            ("orc_tables", [P] * 8), ("orc_forward", [P] * 4), ("orc_forward_naive", [P] * 4),
            ("orc_jvp", [P] * 7), ("orc_vjp", [P] * 6), ("orc_n_t", [P]), ("orc_variant_tables", [P] * 3),
            ("orc_gn_cg_step", [P, P, P, P, C.c_double, C.c_double, C.c_int, P, P, P]),
            ("orc_apply_H", [P, P, P, C.c_double, C.c_double, P, P]),
            ("orc_lm_step_box", [P, P, P, P, C.c_double, C.c_double, C.c_int, P, C.c_int, P, P, P]),
            ("orc_safeguard", [P, P, P, P, P, P, P, P, C.c_double, C.c_double, P, P]),
            ("orc_lm_solve", [P, P, P, P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_double, P, C.c_int,
                              P]),
        ]:
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = C.c_int
        _lib.orc_laplacian.argtypes = [C.c_int, C.c_int, P, P]
        _lib.orc_laplacian.restype = None
        _lib.orc_ray_quadrature.argtypes = [C.c_int, P, P, C.c_double]
        _lib.orc_ray_quadrature.restype = C.c_double
        _lib.orc_ray_adjoint.argtypes = [C.c_int, P, P, C.c_double, P, P]
        _lib.orc_ray_adjoint.restype = None
        _lib.orc_threads.restype = C.c_int
        _lib.orc_pb_crossings.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, P, P, P]
        _lib.orc_pb_crossings.restype = C.c_int
        _lib.orc_set_prior.argtypes = [P, P, C.c_double, C.c_double]
        _lib.orc_project.argtypes = [P, P, C.c_size_t, P]
        _lib.orc_project.restype = None
        _lib.orc_set_prior.restype = None
    return _lib


class _Prior:
    """O10 geometry priors for the duration of one oracle call: prior = (mask_lam, mask_mu, alpha1,
    alpha2) with masks [B][N][N] (or None), member = the batch member of a per-member call."""

    def __init__(self, g, prior, member=None):
        self.lib, self.keep = _load(), []
        self.args = (None, None, 0.0, 0.0)
        if prior is not None:
            m1, m2, a1, a2 = prior
            shp = img_shape(g)

            def arr(m):
                if m is None:
                    return None
                a = _f64(m).reshape(shp)
                a = np.ascontiguousarray(a if member is None else a[member])
                self.keep.append(a)
                return _p(a)
            self.args = (arr(m1), arr(m2), float(a1), float(a2))

    def __enter__(self):
        self.lib.orc_set_prior(*self.args)
        return self

    def __exit__(self, *exc):
        self.lib.orc_set_prior(None, None, 0.0, 0.0)


def _desc(g: dict) -> _Desc:
    return _Desc(int(g["n_px"]), int(g["n_angles"]), int(g.get("n_banks", 2)), int(g.get("n_det", 91)),
                 int(g.get("n_subrays", 1)), float(g.get("subray_sigma", 0.4)),
                 float(g.get("step_px", 0.5)), float(g.get("bank1_shift", 0.0)), int(g.get("batch", 1)),
                 float(g.get("det_radius", 0.0)), float(g.get("c_slope", 0.0)), float(g.get("r_slope", 0.0)),
                 int(g.get("pixel_basis", 0)))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def variant_tables(g: dict) -> dict:
    """O13 tables of the model variant (N3): c_i [n_t] and W_j(d_i) [J][n_t]."""
    lib = _load()
    d = _desc(g)
    n_t = lib.orc_n_t(C.byref(d))
    Cv = np.zeros(n_t)
    W = np.zeros((int(g.get("n_subrays", 1)), n_t))
    rc = lib.orc_variant_tables(C.byref(d), _p(Cv), _p(W))
    assert rc == 0, rc
    return {"c": Cv, "w": W}


def pb_crossings(n_px, c, s, sigma):
    """O14: the pixels (row * N + col) the line sigma omega_perp + t omega, omega = (c, s), crosses in
    [-1,1]^2 in order of increasing t, with the intersection lengths and the chord midpoints' t."""
    lib = _load()
    n = 2 * int(n_px) + 4
    pix = np.zeros(n, np.int32)
    ln = np.zeros(n)
    tm = np.zeros(n)
    M = lib.orc_pb_crossings(int(n_px), float(c), float(s), float(sigma), _p(pix), _p(ln), _p(tm))
    if M < 0:
        raise MemoryError("orc_pb_crossings")
    return pix[:M].copy(), ln[:M].copy(), tm[:M].copy()


def threads() -> int:
    return _load().orc_threads()


def sino_shape(g):
    d = _desc(g)
    return (d.batch, d.n_angles, d.n_banks, d.n_det)


def img_shape(g):
    d = _desc(g)
    return (d.batch, d.n_px, d.n_px)


def tables(g: dict) -> dict:
    """All O1 tables: angles, dirs (cos,sin), offsets, weights, tlat (h, Delta, T), n_t, clip."""
    lib = _load()
    d = _desc(g)
    nA, nB, nd, J = d.n_angles, d.n_banks, d.n_det, d.n_subrays
    out = dict(angles=np.zeros(nA), dirs=np.zeros((nA, nB, 2)), offsets=np.zeros((nB, nd, J)),
               weights=np.zeros(J), tlat=np.zeros(3), clip=np.zeros((nA, nB, nd, J, 2), np.int32))
    nt = C.c_int(0)
    lib.orc_tables(C.byref(d), _p(out["angles"]), _p(out["dirs"]), _p(out["offsets"]),
                   _p(out["weights"]), _p(out["tlat"]), C.byref(nt), _p(out["clip"]))
    out["n_t"] = nt.value
    return out


def forward(g, lam, mu, naive=False):
    lib = _load()
    d = _desc(g)
    lam, mu = _f64(lam), _f64(mu)
    y = np.zeros(sino_shape(g))
    rc = (lib.orc_forward_naive if naive else lib.orc_forward)(C.byref(d), _p(lam), _p(mu), _p(y))
    assert rc == 0, rc
    return y


def jvp(g, lam, mu, dlam, dmu, with_y=False):
    lib = _load()
    d = _desc(g)
    a = [_f64(x) for x in (lam, mu, dlam, dmu)]
    y = np.zeros(sino_shape(g))
    dy = np.zeros(sino_shape(g))
    rc = lib.orc_jvp(C.byref(d), *[_p(x) for x in a], _p(y), _p(dy))
    assert rc == 0, rc
    return (y, dy) if with_y else dy


def vjp(g, lam, mu, w):
    lib = _load()
    d = _desc(g)
    lam, mu, w = _f64(lam), _f64(mu), _f64(w)
    gl = np.zeros(img_shape(g))
    gm = np.zeros(img_shape(g))
    rc = lib.orc_vjp(C.byref(d), _p(lam), _p(mu), _p(w), _p(gl), _p(gm))
    assert rc == 0, rc
    return gl, gm


def laplacian(u):
    lib = _load()
    u = _f64(u)
    if u.ndim == 2:
        u = u[None]
    out = np.zeros_like(u)
    lib.orc_laplacian(u.shape[-1], u.shape[0], _p(u), _p(out))
    return out


def apply_H(g, lam, mu, alpha, beta, p_lam, p_mu, prior=None):
    lib = _load()
    d = _desc(g)
    lam, mu = _f64(lam), _f64(mu)
    p = np.concatenate([_f64(p_lam).ravel(), _f64(p_mu).ravel()])
    out = np.zeros_like(p)
    with _Prior(g, prior):
        rc = lib.orc_apply_H(C.byref(d), _p(lam), _p(mu), alpha, beta, _p(p), _p(out))
    assert rc == 0
    n = p.size // 2
    return out[:n].reshape(img_shape(g)), out[n:].reshape(img_shape(g))


def gn_cg_step(g, lam, mu, y, alpha, beta, n_cg, prior=None):
    """One LM iteration (O7; with the O10 priors).  Returns (s_lam, s_mu, stats dict)."""
    lib = _load()
    d = _desc(g)
    lam, mu, y = _f64(lam), _f64(mu), _f64(y)
    sl = np.zeros(img_shape(g))
    sm = np.zeros(img_shape(g))
    st = np.zeros(ST_CG + n_cg + 1)
    with _Prior(g, prior):
        rc = lib.orc_gn_cg_step(C.byref(d), _p(lam), _p(mu), _p(y), float(alpha), float(beta), int(n_cg),
                                _p(sl), _p(sm), _p(st))
    assert rc == 0, rc
    return sl, sm, stats_dict(st, n_cg)


def lm_step_box(g, lam, mu, y, alpha, beta, n_it, box, inner="sgp", prior=None):
    """One LM iteration inside a box: CG + projection (inner="cg") or SGP (O11).  Returns (s_lam, s_mu,
    stats dict)."""
    lib = _load()
    d = _desc(g)
    lam, mu, y = _f64(lam), _f64(mu), _f64(y)
    bx = _box5(box)
    sl, sm = np.zeros(img_shape(g)), np.zeros(img_shape(g))
    st = np.zeros(ST_CG + n_it + 1)
    with _Prior(g, prior):
        rc = lib.orc_lm_step_box(C.byref(d), _p(lam), _p(mu), _p(y), float(alpha), float(beta), int(n_it), _p(bx),
                                 int(inner == "sgp"), _p(sl), _p(sm), _p(st))
    assert rc == 0, rc
    return sl, sm, stats_dict(st, n_it)


def _box5(box):
    """(lam_lo, lam_hi, mu_lo, mu_hi[, c]) -> the oracle's 5-vector; c > 0 adds lam <= c mu (O12)."""
    b = list(box) + [0.0] * (5 - len(box))
    return np.ascontiguousarray(b, dtype=np.float64)


def project(lam, mu, box):
    """O12: the per-pixel Euclidean projection of (lam, mu) onto the LM solve's feasible set."""
    lib = _load()
    l, m = _f64(lam).copy(), _f64(mu).copy()
    lib.orc_project(_p(l), _p(m), l.size, _p(_box5(box)))
    return l, m


def stats_dict(st, n_cg):
    return dict(f=st[0], misfit=st[1], reg=st[2], grad_norm=st[3], pred=st[4], f_trial=st[5],
                rho=st[6], accepted=bool(st[7]), beta_next=st[8], n_cg_done=int(st[9]),
                breakdown=int(st[10]), beta_min=st[11], js2=st[12], als2=st[13], bs=st[14],
                cg_res=np.array(st[ST_CG:ST_CG + n_cg + 1]))


def ray_quadrature(lam_s, mu_s, delta):
    lib = _load()
    l, m = _f64(lam_s), _f64(mu_s)
    return lib.orc_ray_quadrature(len(l), _p(l), _p(m), float(delta))


def ray_adjoint(lam_s, mu_s, delta):
    lib = _load()
    l, m = _f64(lam_s), _f64(mu_s)
    dl = np.zeros_like(l)
    dm = np.zeros_like(l)
    lib.orc_ray_adjoint(len(l), _p(l), _p(m), float(delta), _p(dl), _p(dm))
    return dl, dm


def safeguard(g, lam, mu, y, s_lam, s_mu, c_lam, c_mu, alpha, kappa=0.1, prior=None):
    """Prop. 1 safeguard (O8), per batch member.  Returns ((u_next_lam, u_next_mu), [dict per member])."""
    lib = _load()
    B = int(g.get("batch", 1))
    shp = img_shape(g)
    arrs = [_f64(a).reshape(shp) for a in (lam, mu, s_lam, s_mu, c_lam, c_mu)]
    ys = _f64(y).reshape(B, -1)
    g1 = dict(g, batch=1)
    d = _desc(g1)
    nl, nm, res = np.zeros(shp), np.zeros(shp), []
    for m in range(B):
        l, u, sl, sm, cl, cm = (np.ascontiguousarray(a[m]) for a in arrs)
        ym = np.ascontiguousarray(ys[m])
        un = np.zeros(2 * l.size)
        out = np.zeros(7)
        with _Prior(g, prior, m):
            rc = lib.orc_safeguard(C.byref(d), _p(l), _p(u), _p(ym), _p(sl), _p(sm), _p(cl), _p(cm), float(alpha),
                                   float(kappa), _p(un), _p(out))
        assert rc == 0, rc
        nl[m] = un[:l.size].reshape(l.shape)
        nm[m] = un[l.size:].reshape(l.shape)
        res.append(dict(f=out[0], f_cand=out[1], m0=out[2], m_cand=out[3], m_lm=out[4], rho_cand=out[5],
                        accepted=bool(out[6]), pred_cand=out[2] - out[3], pred_lm=out[2] - out[4]))
    return (nl, nm), res


def lm_solve(g, lam, mu, y, n_iter, n_cg, alpha0, alpha_decay=5.0, k_freeze=0, beta0=0.0, box=None, prior=None,
             inner="cg"):
    """O9: n_iter LM iterations per batch member (inner solver "cg", or "sgp" (O11) with a box).
    Returns ((lam, mu), [[stats dict per iteration] per member])."""
    assert inner in ("cg", "sgp") and (inner == "cg" or box is not None)
    lib = _load()
    B = int(g.get("batch", 1))
    shp = img_shape(g)
    lam_o, mu_o = _f64(lam).reshape(shp).copy(), _f64(mu).reshape(shp).copy()
    ys = _f64(y).reshape(B, -1)
    d = _desc(dict(g, batch=1))
    bx = None if box is None else _box5(box)
    out = []
    for m in range(B):
        l = np.ascontiguousarray(lam_o[m])
        u = np.ascontiguousarray(mu_o[m])
        st = np.zeros(n_iter * (ST_CG + n_cg + 1))
        with _Prior(g, prior, m):
            rc = lib.orc_lm_solve(C.byref(d), _p(l), _p(u), _p(np.ascontiguousarray(ys[m])), int(n_iter),
                                  int(n_cg), float(alpha0), float(alpha_decay), int(k_freeze), float(beta0),
                                  None if bx is None else _p(bx), int(inner == "sgp"), _p(st))
        assert rc == 0, rc
        lam_o[m], mu_o[m] = l, u
        row = ST_CG + n_cg + 1
        out.append([stats_dict(st[k * row:(k + 1) * row], n_cg) for k in range(n_iter)])
    return (lam_o, mu_o), out
