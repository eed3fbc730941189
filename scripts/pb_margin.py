"""Parity margins of the pixel basis (N3, R-pb) on configs 2-4: rel-L2 and max-relative (Q17) errors of
forward, JVP and VJP against the oracle's O14, and of the GN operator (for DESIGN.md)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2604_26745_b200 as pg  # noqa: E402
import pget_data as P  # noqa: E402
from tests.metrics import max_rel, rel_l2  # noqa: E402

dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
host = lambda t: t.cpu().numpy().astype(np.float64)
for cid in (2, 3, 4):
    for extra in ({}, dict(det_radius=1.6, c_slope=0.05, r_slope=0.35)):
        gd = dict(P.geometry_desc(cid), pixel_basis=1, **extra)
        g = pg.Geometry(gd)
        lam, mu = P.make_phantom(cid)
        dl, dm = P.rod_directions(cid)
        lp, mp = P.make_phantom_prime(cid)
        y_o, dy_o = O.jvp(gd, lam, mu, dl, dm, with_y=True)
        w = (O.forward(gd, lp, mp) - y_o).astype(np.float32)
        gl_o, gm_o = O.vjp(gd, lam, mu, w)
        y = host(pg.forward(g, dev(lam), dev(mu)))
        dy = host(pg.jvp(g, dev(lam), dev(mu), dev(dl), dev(dm)))
        gl, gm = (host(t) for t in pg.vjp(g, dev(lam), dev(mu), dev(w)))
        r = {k: (rel_l2(a[0], b[0]), max_rel(a[0], b[0])) for k, a, b in
             (("fwd", y, y_o), ("jvp", dy, dy_o), ("vjp.lam", gl, gl_o), ("vjp.mu", gm, gm_o))}
        print(f"cfg{cid}{' +var' if extra else ''}", " ".join(f"{k}: l2 {a:.2e} max {b:.2e}" for k, (a, b) in r.items()),
              flush=True)
