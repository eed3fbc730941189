"""Median device time (CUDA events) of each public op on one config: forward, JVP, VJP, GN apply,
safeguard (its time includes the stats device-to-host read of the binding)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26745_b200 as pg  # noqa: E402
import pget_data as P  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 20
gd = P.geometry_desc(cid)
if "--pb" in sys.argv:    # the pixel basis (N3, reading R-pb)
    gd["pixel_basis"] = 1
if "--var" in sys.argv:   # the response of reading R-N3
    gd.update(det_radius=1.6, c_slope=0.05, r_slope=0.35)
g = pg.Geometry(gd)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
lam, mu = map(dev, P.make_phantom(cid))
dl, dm = map(dev, P.rod_directions(cid))
y = pg.forward(g, lam, mu)
ops = {
    "forward": lambda: pg.forward(g, lam, mu, y=y),
    "jvp": lambda: pg.jvp(g, lam, mu, dl, dm),
    "vjp": lambda: pg.vjp(g, lam, mu, y),
    "gn": lambda: pg.gn_apply(g, lam, mu, dl, dm, 1e-3, 0.0),
    "safeguard": lambda: pg.safeguard(g, lam, mu, y, dl, dm, lam + dl, mu + dm, 1e-3),
}
if "--lm" in sys.argv:   # one LM iteration (20 CG steps) at u0 for the measurements y = F(u)
    l0, m0 = map(dev, P.initial_guess(gd["n_px"], gd["batch"]))
    ops["lm"] = lambda: pg.gn_cg_step(g, l0, m0, y, 1e-3, 0.0, 20)
if "--solve" in sys.argv:   # a 10-iteration LM solve (N1) from u0 with a box, restarted each repetition
    l0h, m0h = P.initial_guess(gd["n_px"], gd["batch"])
    ls, ms = dev(l0h), dev(m0h)
    def solve():
        ls.copy_(torch.from_numpy(l0h)); ms.copy_(torch.from_numpy(m0h))
        return pg.lm_solve(g, ls, ms, y, 10, 20, alpha0=1e-2, alpha_decay=5.0, k_freeze=3, beta0=0.0,
                           box=(0.0, 2.0, 0.0, 1.0))
    ops["solve10"] = solve
    if "--sgp" in sys.argv:   # the same solve with the SGP inner solver (PGET_LM_SGP)
        def solve_sgp():
            ls.copy_(torch.from_numpy(l0h)); ms.copy_(torch.from_numpy(m0h))
            return pg.lm_solve(g, ls, ms, y, 10, 20, alpha0=1e-2, alpha_decay=5.0, k_freeze=3, beta0=0.0,
                               box=(0.0, 2.0, 0.0, 1.0), sgp=True)
        ops["solve10_sgp"] = solve_sgp
nom = g.info["n_samples_nominal"]
out = {}
for name, f in ops.items():
    for _ in range(3):
        f()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    out[name] = float(np.median(ts))
print(f"cfg{cid}" + ("-pb" if "--pb" in sys.argv else "") + ("-var" if "--var" in sys.argv else ""), " ".join(f"{k}={v:.4f}ms({nom / v / 1e6:.3g}Gs/s)" for k, v in out.items()), flush=True)
