"""Dump GPU outputs (forward, JVP, VJP) for configs 1-4 to gpurun_out/ for offline
comparison with the oracle (diagnostics only; no oracle call here)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26745_b200 as pg  # noqa: E402
import pget_data as P  # noqa: E402

out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
os.makedirs(out, exist_ok=True)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
for cid in [int(c) for c in (sys.argv[1:] or ["1", "2", "3", "4"])]:
    gd = P.geometry_desc(cid)
    g = pg.Geometry(gd)
    lam, mu = P.make_phantom(cid)
    dl, dm = P.rod_directions(cid)
    lp, mp = P.make_phantom_prime(cid)
    y = pg.forward(g, dev(lam), dev(mu))
    dy = pg.jvp(g, dev(lam), dev(mu), dev(dl), dev(dm))
    w = pg.forward(g, dev(lp), dev(mp)) - y
    gl, gm = pg.vjp(g, dev(lam), dev(mu), w.contiguous())
    np.savez(os.path.join(out, f"dump_cfg{cid}.npz"), y=y.cpu().numpy(), dy=dy.cpu().numpy(),
             w=w.cpu().numpy(), gl=gl.cpu().numpy(), gm=gm.cpu().numpy())
    print("dumped", cid)
