"""Parity margins of the standalone VJP (max-relative with the 1e-3 floor, relative L2) against the fp64
oracle on configs 1-4 and the mu x20 / x80 stress inputs, for the path selected by the environment
(e.g. PGET_VJP_CACHED=1).  Usage: vjp_margin.py [cid ...]"""
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
cases = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]
for cid in cases:
    for scale in ([1.0, 20.0, 80.0] if cid == 2 else [1.0]):
        gd = P.geometry_desc(cid)
        lam, mu = P.make_phantom(cid)
        lp, mp = P.make_phantom_prime(cid)
        mu = (mu * np.float32(scale)).astype(np.float32)
        g = pg.Geometry(gd)
        y_o = O.forward(gd, lam, mu)
        w = (O.forward(gd, lp, mu if scale != 1.0 else mp) - y_o).astype(np.float32)
        gl, gm = pg.vjp(g, dev(lam), dev(mu), dev(w))
        gl_o, gm_o = O.vjp(gd, lam, mu, w)
        print(f"cfg{cid} mu x{scale:g} [{os.environ.get('PGET_VJP_CACHED', '0')}]: "
              f"lam max_rel {max_rel(host(gl), gl_o):.2e} rel_l2 {rel_l2(host(gl), gl_o):.2e}  "
              f"mu max_rel {max_rel(host(gm), gm_o):.2e} rel_l2 {rel_l2(host(gm), gm_o):.2e}", flush=True)
