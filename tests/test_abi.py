"""CPU tests of the C-ABI library: it loads, exports every symbol include/pget.h
declares, validates arguments, and its host geometry tables are bit-exact with
the oracle's (pin P1).  No compute call runs here (no GPU)."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2604_26745_b200 as pg
import pget_data as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "pget.h")).read()
    return sorted(set(re.findall(r"\b(pget_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = pg.lib()
    names = declared_functions()
    assert len(names) >= 13
    out = subprocess.run(["nm", "-D", "--defined-only", pg.LIB], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    for n in names:
        assert n in exported, n
        assert hasattr(lib, n)


def test_library_links_no_oracle():
    out = subprocess.run(["ldd", pg.LIB], capture_output=True, text=True).stdout
    assert "oracle" not in out
    out = subprocess.run(["nm", "-D", pg.LIB], capture_output=True, text=True).stdout
    assert "orc_" not in out


def _same_bits(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


GEOMS = [P.geometry_desc(c) for c in (1, 2, 3, 4, 5)] + [
    dict(n_px=33, n_angles=12, n_banks=2, n_det=7, n_subrays=2, subray_sigma=0.4, step_px=0.5, bank1_shift=0.0,
         batch=1),
    dict(n_px=16, n_angles=7, n_banks=1, n_det=5, n_subrays=9, subray_sigma=0.3, step_px=0.37, bank1_shift=0.0,
         batch=3),
    dict(n_px=24, n_angles=10, n_banks=2, n_det=11, n_subrays=3, subray_sigma=0.4, step_px=0.5, bank1_shift=6.5,
         batch=1),
]


@pytest.mark.parametrize("gd", GEOMS)
def test_tables_bit_exact_with_oracle(gd):
    g = pg.Geometry(gd, device=-1)
    t = O.tables(gd)
    assert _same_bits(g.export("angles"), t["angles"].ravel())
    assert _same_bits(g.export("dirs"), t["dirs"].ravel())
    assert _same_bits(g.export("offsets"), t["offsets"].ravel())
    assert _same_bits(g.export("weights"), t["weights"].ravel())
    assert _same_bits(g.export("tlat"), t["tlat"].ravel())
    assert _same_bits(g.export("clip"), t["clip"].ravel())
    assert g.info["n_t"] == t["n_t"]
    cl = t["clip"]
    assert g.info["n_samples_nominal"] == int(np.clip(cl[..., 1] - cl[..., 0] + 1, 0, None).sum()) * gd["batch"]


def test_shifted_bank_has_empty_rays():
    gd = GEOMS[-1]
    cl = pg.Geometry(gd, device=-1).export("clip").reshape(10, 2, 11, 3, 2)
    assert np.any(cl[..., 0] > cl[..., 1])


def test_invalid_desc_rejected():
    for bad in (dict(n_px=1), dict(n_det=1), dict(n_subrays=0), dict(n_subrays=65), dict(n_banks=3),
                dict(step_px=0.0), dict(subray_sigma=-1.0), dict(batch=0), dict(step_px=float("nan"))):
        gd = dict(GEOMS[0], **bad)
        with pytest.raises(RuntimeError, match="INVALID_ARGUMENT"):
            pg.Geometry(gd, device=-1)


def test_compute_on_host_only_handle_fails_cleanly():
    import ctypes as C
    g = pg.Geometry(GEOMS[5], device=-1)
    rc = pg.lib().pget_forward(g.handle, None, None, None, None, 0, None)
    assert rc == 1
    assert b"host-only" in pg.lib().pget_last_error_message()
    assert pg.lib().pget_workspace_bytes(g.handle, 99) == 0
    assert pg.lib().pget_table_bytes(g.handle, 42) == 0
    for op in pg.OPS:
        assert g.workspace_bytes(op) > 0
    pr = pg.Prior(None, None, 1.0, 1.0)
    assert pg.lib().pget_set_prior(g.handle, C.byref(pr)) == 1      # host-only handle
    assert pg.lib().pget_set_prior(None, None) == 1


def test_host_struct_layouts():
    """The C structs the binding mirrors keep their sizes (pget.h): the LM parameters (48 B, the last
    field lam_per_mu replaced a pad), the prior, the safeguard statistics."""
    import ctypes as C
    assert C.sizeof(pg.LMParams) == 48
    assert C.sizeof(pg.Prior) == 24
    assert C.sizeof(pg.SafeguardStats) == 72


@pytest.mark.parametrize("gd", [P.geometry_desc(c) for c in (1, 2, 3, 4)] + [
    dict(n_px=33, n_angles=12, n_banks=2, n_det=7, n_subrays=2, subray_sigma=0.4, step_px=0.5, bank1_shift=0.0,
         batch=3),
    dict(n_px=16, n_angles=7, n_banks=1, n_det=5, n_subrays=9, subray_sigma=0.3, step_px=0.37, bank1_shift=0.0,
         batch=1),
    dict(n_px=24, n_angles=10, n_banks=2, n_det=11, n_subrays=3, subray_sigma=0.4, step_px=0.5, bank1_shift=6.5,
         batch=2),
    dict(n_px=64, n_angles=90, n_banks=2, n_det=91, n_subrays=1, subray_sigma=0.4, step_px=0.5, bank1_shift=0.0,
         batch=7),
], ids=["cfg1", "cfg2", "cfg3", "cfg4", "odd33", "onebank", "shift", "batch7"])
def test_static_schedules_consistent(gd):
    """Host logic: the static schedules (fused forward/JVP task lists, the segmented adjoint's units,
    stages, slots, reduce lists, coefficient-cache layout, comb groups) pass pget_schedule_check."""
    g = pg.Geometry(gd, device=-1)
    g.schedule_check()


def test_workspace_regions_inside_and_disjoint():
    """pget_workspace_region: the CG vectors p, q of an LM iteration are four disjoint image-sized
    regions inside the workspace the call asks for."""
    gd = P.geometry_desc(2)
    g = pg.Geometry(gd, device=-1)
    total = g.workspace_bytes("gn_cg_step")
    spans = [g.workspace_region("gn_cg_step", r) for r in range(4)]
    img = int(np.prod(g.img_shape)) * 4
    for off, n in spans:
        assert n == img and off % 16 == 0 and off + n <= total
    spans.sort()
    for (a, n), (b, _) in zip(spans, spans[1:]):
        assert a + n <= b
    with pytest.raises(RuntimeError):
        g.workspace_region("forward", 0)
    with pytest.raises(RuntimeError):
        g.workspace_region("gn_cg_step", 7)


VAR_GEOMS = [dict(P.geometry_desc(c), det_radius=1.6, c_slope=0.05, r_slope=0.35) for c in (2, 4)] + [
    dict(n_px=16, n_angles=7, n_banks=1, n_det=5, n_subrays=9, subray_sigma=0.3, step_px=0.37, bank1_shift=0.0,
         batch=3, det_radius=2.0, c_slope=0.2, r_slope=1.0)]


@pytest.mark.parametrize("gd", VAR_GEOMS)
def test_variant_tables_bit_exact_with_oracle(gd):
    """Model variant (N3, reading R-N3): the library's c_i and W_j(d_i) equal the oracle's O13 tables bit
    for bit; the variant disables line pairing (its attenuation does not factor along a line)."""
    g = pg.Geometry(gd, device=-1)
    v = O.variant_tables(gd)
    assert _same_bits(g.export("var_c"), v["c"])
    assert _same_bits(g.export("var_w").reshape(v["w"].shape), v["w"])
    base = pg.Geometry(dict(gd, det_radius=0.0), device=-1)
    assert g.info["n_samples_traced"] >= base.info["n_samples_traced"]
    if base.info["angle_banks_merged"]:
        assert g.info["n_samples_traced"] == 2 * base.info["n_samples_traced"]   # unpaired
    assert g.export("var_c").size > 0 and base.export("var_c").size == 0


def test_variant_desc_validation():
    import ctypes as C
    bad = [dict(P.geometry_desc(2), det_radius=1.0, c_slope=0.1),          # det_radius < T
           dict(P.geometry_desc(2), det_radius=1.6, c_slope=-0.1),         # negative slope
           dict(P.geometry_desc(2), det_radius=1.6, r_slope=float("nan"))]
    for gd in bad:
        with pytest.raises(RuntimeError, match="INVALID_ARGUMENT"):
            pg.Geometry(gd, device=-1)


def test_pixel_basis_host_handle():
    """Pixel basis (N3, reading R-pb): the descriptor carries pixel_basis (88-byte struct), the handle
    traces every angle-bank (no merging), its sample count is the crossing count of the oracle's O14
    traversal up to corner coincidences (an edge pair crossed at one t counts once there), and values
    other than 0 / 1 are rejected."""
    import ctypes as C
    assert C.sizeof(pg._Desc) == 88
    gd = dict(n_px=12, n_angles=6, n_banks=2, n_det=9, n_subrays=3, subray_sigma=0.4, step_px=0.5,
              bank1_shift=0.0, batch=2, pixel_basis=1)
    g = pg.Geometry(gd, device=-1)
    assert g.info["angle_banks_merged"] == 0
    T = O.tables(gd)
    ref = 0
    for a in range(6):
        for b in range(2):
            c, s = T["dirs"][a, b]
            for d in range(9):
                for j in range(3):
                    ref += len(O.pb_crossings(12, c, s, T["offsets"][b, d, j])[0])
    n_rays = 6 * 2 * 9 * 3
    assert 2 * ref <= g.info["n_samples_nominal"] <= 2 * (ref + n_rays)
    assert g.info["n_samples_traced"] == g.info["n_samples_nominal"]
    for c in (2, 4):
        h = pg.Geometry(dict(P.geometry_desc(c), pixel_basis=1), device=-1)
        assert h.info["angle_banks_merged"] == 0
    with pytest.raises(RuntimeError, match="INVALID_ARGUMENT"):
        pg.Geometry(dict(gd, pixel_basis=2), device=-1)
