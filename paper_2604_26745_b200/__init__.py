"""Python binding of libpget (include/pget.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module
only checks tensor shapes/dtypes, passes device pointers and the current torch
stream through ctypes, and allocates outputs/workspaces with torch.  There is
no CPU fallback: if libpget.so is missing or fails to load, importing the
binding raises.

Names follow the C ABI: Geometry (pget_geometry_create/destroy/info/export),
forward, jvp, vjp, gn_apply, gn_cg_step.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._build import LIB, build as _build_lib, needs_build as _needs_build

__all__ = ["Geometry", "forward", "jvp", "vjp", "gn_apply", "gn_cg_step", "safeguard", "lm_solve", "GNStats", "SafeguardStats", "LMParams", "lib",
           "PGET_GN_EVAL_TRIAL", "TABLES", "OPS"]

PGET_GN_EVAL_TRIAL = 1
PGET_MAX_CG = 256
TABLES = {"angles": 0, "dirs": 1, "offsets": 2, "weights": 3, "tlat": 4, "clip": 5, "var_c": 6, "var_w": 7}
OPS = {"forward": 0, "jvp": 1, "vjp": 2, "gn_cg_step": 3, "gn_apply": 4, "safeguard": 5, "lm_solve": 6}
EXPORTED = ["pget_status_string", "pget_last_error_message", "pget_geometry_create", "pget_geometry_destroy",
            "pget_geometry_info", "pget_table_bytes", "pget_geometry_export", "pget_workspace_bytes",
            "pget_forward", "pget_jvp", "pget_vjp", "pget_gn_apply", "pget_gn_cg_step", "pget_safeguard", "pget_lm_solve", "pget_profile_begin",
            "pget_profile_end", "pget_set_prior", "pget_schedule_check"]
MODES = ("forward", "jvp", "vjp", "gn")


class _Desc(C.Structure):
    _fields_ = [("n_px", C.c_int32), ("n_angles", C.c_int32), ("n_banks", C.c_int32), ("n_det", C.c_int32),
                ("n_subrays", C.c_int32), ("subray_sigma", C.c_double), ("step_px", C.c_double),
                ("bank1_shift", C.c_double), ("batch", C.c_int32), ("det_radius", C.c_double),
                ("c_slope", C.c_double), ("r_slope", C.c_double), ("pixel_basis", C.c_int32),
                ("pad_", C.c_int32)]


class _Info(C.Structure):
    _fields_ = [("n_rays", C.c_int64), ("n_samples_nominal", C.c_int64), ("image_elems", C.c_int64),
                ("sino_elems", C.c_int64), ("n_t", C.c_int32), ("n_px", C.c_int32), ("n_angles", C.c_int32),
                ("n_banks", C.c_int32), ("n_det", C.c_int32), ("n_subrays", C.c_int32), ("batch", C.c_int32),
                ("h", C.c_double), ("delta", C.c_double), ("T", C.c_double), ("n_samples_traced", C.c_int64),
                ("angle_banks_merged", C.c_int32), ("pad_", C.c_int32), ("n_samples_traced_jvp", C.c_int64)]


class GNStats(C.Structure):
    _fields_ = [("f", C.c_double), ("misfit", C.c_double), ("reg", C.c_double), ("grad_norm", C.c_double),
                ("pred", C.c_double), ("f_trial", C.c_double), ("rho", C.c_double), ("beta_next", C.c_double),
                ("beta_min", C.c_double), ("js2", C.c_double), ("als2", C.c_double), ("bs", C.c_double),
                ("accepted", C.c_int32), ("n_cg_done", C.c_int32), ("breakdown", C.c_int32), ("pad_", C.c_int32),
                ("cg_res", C.c_double * (PGET_MAX_CG + 1))]

    def to_dict(self, n_cg=None):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("cg_res", "pad_")}
        d["accepted"] = bool(d["accepted"])
        n = self.n_cg_done if n_cg is None else n_cg
        d["cg_res"] = np.array(self.cg_res[: n + 1])
        return d


PGET_LM_BOX = 1
PGET_LM_SGP = 2


class LMParams(C.Structure):
    _fields_ = [("n_iter", C.c_int32), ("n_cg", C.c_int32), ("alpha0", C.c_float), ("alpha_decay", C.c_float),
                ("k_freeze", C.c_int32), ("beta0", C.c_float), ("lam_lo", C.c_float), ("lam_hi", C.c_float),
                ("mu_lo", C.c_float), ("mu_hi", C.c_float), ("flags", C.c_uint32), ("lam_per_mu", C.c_float)]


class Prior(C.Structure):
    _fields_ = [("mask_lam", C.c_void_p), ("mask_mu", C.c_void_p), ("alpha1", C.c_float), ("alpha2", C.c_float)]


class SafeguardStats(C.Structure):
    _fields_ = [("f", C.c_double), ("f_cand", C.c_double), ("m_cand", C.c_double), ("m_lm", C.c_double),
                ("pred_cand", C.c_double), ("pred_lm", C.c_double), ("rho_cand", C.c_double), ("kappa", C.c_double),
                ("accepted", C.c_int32), ("pad_", C.c_int32)]

    def to_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}
        d["accepted"] = bool(d["accepted"])
        return d


_lib = None


def lib():
    """Load libpget.so (building it first if the sources are newer); raise if impossible."""
    global _lib
    if _lib is None:
        if _needs_build():
            _build_lib()
        if not os.path.exists(LIB):
            raise ImportError(f"libpget.so not found at {LIB}")
        L = C.CDLL(LIB)
        P, S = C.c_void_p, C.c_size_t
        L.pget_status_string.restype = C.c_char_p
        L.pget_status_string.argtypes = [C.c_int]
        L.pget_last_error_message.restype = C.c_char_p
        L.pget_geometry_create.argtypes = [C.POINTER(_Desc), C.c_int, C.POINTER(P)]
        L.pget_geometry_destroy.argtypes = [P]
        L.pget_geometry_info.argtypes = [P, C.POINTER(_Info)]
        L.pget_table_bytes.argtypes = [P, C.c_int]
        L.pget_table_bytes.restype = S
        L.pget_geometry_export.argtypes = [P, C.c_int, P, S]
        L.pget_workspace_bytes.argtypes = [P, C.c_int]
        L.pget_workspace_bytes.restype = S
        L.pget_forward.argtypes = [P, P, P, P, P, S, P]
        L.pget_jvp.argtypes = [P, P, P, P, P, P, P, P, S, P]
        L.pget_vjp.argtypes = [P, P, P, P, P, P, P, S, P]
        L.pget_gn_apply.argtypes = [P, P, P, P, P, C.c_float, C.c_float, P, P, P, S, P]
        L.pget_gn_cg_step.argtypes = [P, P, P, P, C.c_float, C.c_float, C.c_int32, C.c_uint32, P, P, P, P, S, P]
        L.pget_safeguard.argtypes = [P, P, P, P, P, P, P, P, C.c_float, C.c_float, P, P, P, P, S, P]
        L.pget_lm_solve.argtypes = [P, P, P, P, C.POINTER(LMParams), P, P, S, P]
        L.pget_schedule_check.argtypes = [P]
        L.pget_workspace_region.argtypes = [P, C.c_int, C.c_int, C.POINTER(S), C.POINTER(S)]
        L.pget_set_prior.argtypes = [P, C.POINTER(Prior)]
        L.pget_check_finite.argtypes = [P, S, P, P]
        L.pget_profile_begin.argtypes = [C.c_int32]
        L.pget_profile_end.argtypes = [P, P, P]
        for n in ("pget_profile_begin", "pget_profile_end", "pget_geometry_create", "pget_geometry_destroy", "pget_geometry_info", "pget_geometry_export",
                  "pget_forward", "pget_jvp", "pget_vjp", "pget_gn_apply", "pget_gn_cg_step", "pget_safeguard", "pget_lm_solve", "pget_schedule_check", "pget_set_prior",
                  "pget_workspace_region", "pget_check_finite"):
            getattr(L, n).restype = C.c_int
        _lib = L
    return _lib


def _check(rc, what):
    if rc != 0:
        L = lib()
        raise RuntimeError(f"{what}: {L.pget_status_string(rc).decode()}: {L.pget_last_error_message().decode()}")


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


class Geometry:
    """pget_geometry handle.  desc: dict with the pget_geometry_desc fields."""

    def __init__(self, desc: dict, device: int | None = None):
        self.desc = dict(desc)
        if device is None:
            import torch
            device = torch.cuda.current_device()
        self.device = int(device)           # device < 0: host-only handle (tables/info only)
        d = _Desc(int(desc["n_px"]), int(desc["n_angles"]), int(desc.get("n_banks", 2)), int(desc.get("n_det", 91)),
                  int(desc.get("n_subrays", 1)), float(desc.get("subray_sigma", 0.4)),
                  float(desc.get("step_px", 0.5)), float(desc.get("bank1_shift", 0.0)), int(desc.get("batch", 1)),
                  float(desc.get("det_radius", 0.0)), float(desc.get("c_slope", 0.0)), float(desc.get("r_slope", 0.0)),
                  int(desc.get("pixel_basis", 0)), 0)
        h = C.c_void_p()
        _check(lib().pget_geometry_create(C.byref(d), self.device, C.byref(h)), "pget_geometry_create")
        self._h = h
        info = _Info()
        _check(lib().pget_geometry_info(h, C.byref(info)), "pget_geometry_info")
        self.info = {k: getattr(info, k) for k, _ in _Info._fields_}
        self._ws = {}

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().pget_geometry_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def img_shape(self):
        i = self.info
        return (i["batch"], i["n_px"], i["n_px"])

    @property
    def sino_shape(self):
        i = self.info
        return (i["batch"], i["n_angles"], i["n_banks"], i["n_det"])

    def export(self, name: str):
        tid = TABLES[name]
        nbytes = lib().pget_table_bytes(self._h, tid)
        dt = np.int32 if name == "clip" else np.float64
        out = np.zeros(nbytes // np.dtype(dt).itemsize, dtype=dt)
        _check(lib().pget_geometry_export(self._h, tid, out.ctypes.data_as(C.c_void_p), nbytes), "export")
        return out

    def set_prior(self, mask_lam=None, mask_mu=None, alpha1=0.0, alpha2=0.0):
        """Attach the geometry priors P1 = diag(mask_lam), P2 = diag(mask_mu) (pget_set_prior): later
        GN / LM / safeguard calls add alpha1/2 ||P1 lam||^2 + alpha2/2 ||P2 mu||^2 to f.  Masks are
        contiguous fp32 CUDA tensors of img_shape (kept referenced here); all None clears."""
        if mask_lam is None and mask_mu is None:
            _check(lib().pget_set_prior(self._h, None), "pget_set_prior")
            self._prior = None
            return
        for m in (mask_lam, mask_mu):
            if m is not None:
                _f32(m, self.img_shape, "mask")
        pr = Prior(mask_lam.data_ptr() if mask_lam is not None else None,
                   mask_mu.data_ptr() if mask_mu is not None else None, float(alpha1), float(alpha2))
        _check(lib().pget_set_prior(self._h, C.byref(pr)), "pget_set_prior")
        self._prior = (mask_lam, mask_mu)

    def workspace_region(self, op: str, region: int):
        """(offset, bytes) of a CG vector inside `op`'s workspace (pget_workspace_region; tests)."""
        off, n = C.c_size_t(), C.c_size_t()
        _check(lib().pget_workspace_region(self._h, OPS[op], int(region), C.byref(off), C.byref(n)),
               "pget_workspace_region")
        return off.value, n.value

    def schedule_check(self):
        """Host-side consistency check of the handle's static schedules (raises on a violation)."""
        _check(lib().pget_schedule_check(self._h), "pget_schedule_check")

    def workspace_bytes(self, op: str) -> int:
        return int(lib().pget_workspace_bytes(self._h, OPS[op]))

    def workspace(self, op: str):
        """A cached torch uint8 workspace for `op` on this geometry's device."""
        import torch
        n = self.workspace_bytes(op)
        ws = self._ws.get(op)
        if ws is None or ws.numel() < n:
            ws = torch.empty(max(n, 16), dtype=torch.uint8, device=f"cuda:{self.device}")
            self._ws[op] = ws
        return ws


def _f32(t, shape, what):
    """A contiguous float32 CUDA tensor of exactly `shape` ([B][N][N] images, [B][n_angles][n_banks][n_det]
    sinograms); with batch 1 the leading batch axis may be omitted.  Anything else raises: the C ABI
    reads raw pointers, so a tensor of the right size in another layout would be misread."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise TypeError(f"{what}: expected a contiguous float32 CUDA tensor")
    shape = tuple(shape)
    if tuple(t.shape) != shape and not (shape[0] == 1 and tuple(t.shape) == shape[1:]):
        raise ValueError(f"{what}: shape {tuple(t.shape)} != {shape}")
    return t


def forward(g: Geometry, lam, mu, y=None, ws=None, stream=None):
    import torch
    _f32(lam, g.img_shape, "lam"); _f32(mu, g.img_shape, "mu")
    if y is None:
        y = torch.empty(g.sino_shape, dtype=torch.float32, device=lam.device)
    _f32(y, g.sino_shape, "y")
    ws = g.workspace("forward") if ws is None else ws
    _check(lib().pget_forward(g.handle, _ptr(lam), _ptr(mu), _ptr(y), _ptr(ws), ws.numel(), _stream(stream)),
           "pget_forward")
    return y


def jvp(g: Geometry, lam, mu, dlam, dmu, want_y=False, y=None, dy=None, ws=None, stream=None):
    import torch
    for t, n in ((lam, "lam"), (mu, "mu"), (dlam, "dlam"), (dmu, "dmu")):
        _f32(t, g.img_shape, n)
    if dy is None:
        dy = torch.empty(g.sino_shape, dtype=torch.float32, device=lam.device)
    if want_y and y is None:
        y = torch.empty(g.sino_shape, dtype=torch.float32, device=lam.device)
    _f32(dy, g.sino_shape, "dy")
    if want_y:
        _f32(y, g.sino_shape, "y")
    ws = g.workspace("jvp") if ws is None else ws
    _check(lib().pget_jvp(g.handle, _ptr(lam), _ptr(mu), _ptr(dlam), _ptr(dmu), _ptr(y) if want_y else None,
                          _ptr(dy), _ptr(ws), ws.numel(), _stream(stream)), "pget_jvp")
    return (y, dy) if want_y else dy


def vjp(g: Geometry, lam, mu, w, g_lam=None, g_mu=None, ws=None, stream=None):
    import torch
    _f32(lam, g.img_shape, "lam"); _f32(mu, g.img_shape, "mu"); _f32(w, g.sino_shape, "w")
    if g_lam is None:
        g_lam = torch.empty(g.img_shape, dtype=torch.float32, device=lam.device)
        g_mu = torch.empty(g.img_shape, dtype=torch.float32, device=lam.device)
    _f32(g_lam, g.img_shape, "g_lam"); _f32(g_mu, g.img_shape, "g_mu")
    ws = g.workspace("vjp") if ws is None else ws
    _check(lib().pget_vjp(g.handle, _ptr(lam), _ptr(mu), _ptr(w), _ptr(g_lam), _ptr(g_mu), _ptr(ws), ws.numel(),
                          _stream(stream)), "pget_vjp")
    return g_lam, g_mu


def gn_apply(g: Geometry, lam, mu, p_lam, p_mu, alpha, beta, ws=None, stream=None):
    import torch
    for t, n in ((lam, "lam"), (mu, "mu"), (p_lam, "p_lam"), (p_mu, "p_mu")):
        _f32(t, g.img_shape, n)
    q_lam = torch.empty(g.img_shape, dtype=torch.float32, device=lam.device)
    q_mu = torch.empty_like(q_lam)
    ws = g.workspace("gn_apply") if ws is None else ws
    _check(lib().pget_gn_apply(g.handle, _ptr(lam), _ptr(mu), _ptr(p_lam), _ptr(p_mu), float(alpha), float(beta),
                               _ptr(q_lam), _ptr(q_mu), _ptr(ws), ws.numel(), _stream(stream)), "pget_gn_apply")
    return q_lam, q_mu


def stats_buffer(g: Geometry, device=None):
    import torch
    return torch.zeros(g.info["batch"] * C.sizeof(GNStats), dtype=torch.uint8,
                       device=device or f"cuda:{g.device}")


def read_stats(buf, batch: int, n_cg=None):
    host = buf.cpu().numpy().tobytes()
    out = []
    for m in range(batch):
        st = GNStats.from_buffer_copy(host[m * C.sizeof(GNStats):(m + 1) * C.sizeof(GNStats)])
        out.append(st.to_dict(n_cg))
    return out


def gn_cg_step(g: Geometry, lam, mu, y_meas, alpha, beta, n_cg, flags=PGET_GN_EVAL_TRIAL, s_lam=None, s_mu=None,
               stats=None, ws=None, stream=None):
    """One LM iteration (pget_gn_cg_step).  Returns (s_lam, s_mu, stats_device_buffer)."""
    import torch
    _f32(lam, g.img_shape, "lam"); _f32(mu, g.img_shape, "mu"); _f32(y_meas, g.sino_shape, "y_meas")
    if s_lam is None:
        s_lam = torch.empty(g.img_shape, dtype=torch.float32, device=lam.device)
        s_mu = torch.empty_like(s_lam)
    _f32(s_lam, g.img_shape, "s_lam"); _f32(s_mu, g.img_shape, "s_mu")
    if stats is None:
        stats = stats_buffer(g, lam.device)
    ws = g.workspace("gn_cg_step") if ws is None else ws
    _check(lib().pget_gn_cg_step(g.handle, _ptr(lam), _ptr(mu), _ptr(y_meas), float(alpha), float(beta), int(n_cg),
                                 int(flags), _ptr(s_lam), _ptr(s_mu), _ptr(stats), _ptr(ws), ws.numel(),
                                 _stream(stream)), "pget_gn_cg_step")
    return s_lam, s_mu, stats


def check_finite(t, stream=None):
    """Raise RuntimeError (PGET_ERR_NOT_FINITE) if the float32 CUDA tensor t holds a NaN or an infinity
    (pget_check_finite; synchronises the stream)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise TypeError("check_finite: expected a contiguous float32 CUDA tensor")
    flag = torch.empty(1, dtype=torch.int32, device=t.device)
    _check(lib().pget_check_finite(_ptr(t), t.numel(), _ptr(flag), _stream(stream)), "pget_check_finite")


def profile_begin(max_launches: int = 4096):
    """Start counting library kernel launches and timing projector launches (CUDA events)."""
    _check(lib().pget_profile_begin(int(max_launches)), "pget_profile_begin")


def profile_end():
    """Stop tracing; returns {'ms': {mode: ms}, 'launches': {mode: n}, 'total_launches': n}."""
    ms = (C.c_double * 4)()
    n = (C.c_int64 * 4)()
    tot = C.c_int64()
    _check(lib().pget_profile_end(ms, n, C.byref(tot)), "pget_profile_end")
    return {"ms": dict(zip(MODES, list(ms))), "launches": dict(zip(MODES, list(n))), "total_launches": tot.value}


def safeguard(g: Geometry, lam, mu, y_meas, s_lam, s_mu, cand_lam, cand_mu, alpha, kappa=0.1, u_next=None,
              ws=None, stream=None):
    """Prop. 1 safeguard (pget_safeguard).  Returns ((u_next_lam, u_next_mu), [stats dict per member])."""
    import torch
    for t, n in ((lam, "lam"), (mu, "mu"), (s_lam, "s_lam"), (s_mu, "s_mu"), (cand_lam, "cand_lam"),
                 (cand_mu, "cand_mu")):
        _f32(t, g.img_shape, n)
    _f32(y_meas, g.sino_shape, "y_meas")
    if u_next is None:
        u_next = (torch.empty(g.img_shape, dtype=torch.float32, device=lam.device),
                  torch.empty(g.img_shape, dtype=torch.float32, device=lam.device))
    B = g.info["batch"]
    buf = torch.zeros(B * C.sizeof(SafeguardStats), dtype=torch.uint8, device=lam.device)
    ws = g.workspace("safeguard") if ws is None else ws
    _check(lib().pget_safeguard(g.handle, _ptr(lam), _ptr(mu), _ptr(y_meas), _ptr(s_lam), _ptr(s_mu), _ptr(cand_lam),
                                _ptr(cand_mu), float(alpha), float(kappa), _ptr(u_next[0]), _ptr(u_next[1]),
                                _ptr(buf), _ptr(ws), ws.numel(), _stream(stream)), "pget_safeguard")
    host = buf.cpu().numpy().tobytes()
    n = C.sizeof(SafeguardStats)
    return u_next, [SafeguardStats.from_buffer_copy(host[m * n:(m + 1) * n]).to_dict() for m in range(B)]


def lm_solve(g: Geometry, lam, mu, y_meas, n_iter, n_cg=20, alpha0=1e-3, alpha_decay=5.0, k_freeze=0, beta0=0.0,
             box=None, sgp=False, lam_per_mu=0.0, ws=None, stream=None):
    """Full LM solve (pget_lm_solve): lam, mu are updated in place.  box = (lam_lo, lam_hi, mu_lo, mu_hi)
    or None; sgp: the box-constrained steps by SGP (PGET_LM_SGP); lam_per_mu > 0 adds lam <= lam_per_mu mu
    to the box.  Returns [[stats dict per member] per iteration]."""
    import torch
    _f32(lam, g.img_shape, "lam"); _f32(mu, g.img_shape, "mu"); _f32(y_meas, g.sino_shape, "y_meas")
    p = LMParams(int(n_iter), int(n_cg), float(alpha0), float(alpha_decay), int(k_freeze), float(beta0),
                 *(float(x) for x in (box if box is not None else (0.0, 0.0, 0.0, 0.0))),
                 (PGET_LM_BOX if box is not None else 0) | (PGET_LM_SGP if sgp else 0), float(lam_per_mu))
    B = g.info["batch"]
    buf = torch.zeros(max(1, n_iter) * B * C.sizeof(GNStats), dtype=torch.uint8, device=lam.device)
    ws = g.workspace("lm_solve") if ws is None else ws
    _check(lib().pget_lm_solve(g.handle, _ptr(lam), _ptr(mu), _ptr(y_meas), C.byref(p), _ptr(buf), _ptr(ws),
                               ws.numel(), _stream(stream)), "pget_lm_solve")
    host = buf.cpu().numpy().tobytes()
    n = C.sizeof(GNStats)
    return [[GNStats.from_buffer_copy(host[(k * B + m) * n:(k * B + m + 1) * n]).to_dict(n_cg) for m in range(B)]
            for k in range(n_iter)]
