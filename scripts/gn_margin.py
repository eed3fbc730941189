"""Relative-L2 error of the GN product (pget_gn_apply) against the fp64 oracle on configs 2 and 3
(the tolerance is 1e-5; prints the margin)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2604_26745_b200 as pg  # noqa: E402
import pget_data as P  # noqa: E402
from tests.metrics import rel_l2  # noqa: E402

dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
for cid in [int(c) for c in sys.argv[1:]] or [2, 3]:
    gd = P.geometry_desc(cid)
    g = pg.Geometry(gd)
    lam, mu = P.make_phantom(cid)
    dl, dm = P.rod_directions(cid)
    ql, qm = pg.gn_apply(g, dev(lam), dev(mu), dev(dl), dev(dm), 1e-3, 0.0)
    ol, om = O.apply_H(gd, lam, mu, 1e-3, 0.0, dl, dm)
    print(f"cfg{cid} gn rel_l2 lam {rel_l2(ql.cpu().numpy().astype(np.float64), ol):.2e} "
          f"mu {rel_l2(qm.cpu().numpy().astype(np.float64), om):.2e}", flush=True)
