"""Run each projector mode once on a config (for ncu captures): forward, JVP, VJP, GN apply (through
the coefficient cache, as the LM iteration runs it: VJP-mode phase A, cache build, GN-mode phase A,
scatter weights, cached scatter)."""
import os
import sys

os.environ.setdefault("PGET_GN_APPLY_CACHED", "1")

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26745_b200 as pg  # noqa: E402
import pget_data as P  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
gd = P.geometry_desc(cid)
g = pg.Geometry(gd)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
lam, mu = map(dev, P.make_phantom(cid))
dl, dm = map(dev, P.rod_directions(cid))
for _ in range(reps):
    y = pg.forward(g, lam, mu)
    dy = pg.jvp(g, lam, mu, dl, dm)
    gl, gm = pg.vjp(g, lam, mu, dy)
    ql, qm = pg.gn_apply(g, lam, mu, dl, dm, 1e-3, 0.0)
torch.cuda.synchronize()
print("ok", float(y.sum()), float(gl.sum()), float(ql.sum()))
