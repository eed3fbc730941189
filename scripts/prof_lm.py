"""Run one LM iteration (gn_cg_step, 20 CG steps) on a config, for ncu captures of its small kernels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26745_b200 as pg  # noqa: E402
import pget_data as P  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
gd = P.geometry_desc(cid)
g = pg.Geometry(gd)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
lam, mu = map(dev, P.make_phantom(cid))
y = pg.forward(g, lam, mu)
l0, m0 = map(dev, P.initial_guess(gd["n_px"], gd["batch"]))
sl, sm, st = pg.gn_cg_step(g, l0, m0, y, 1e-3, 0.0, 20)
torch.cuda.synchronize()
print("ok", float(sl.sum()))
