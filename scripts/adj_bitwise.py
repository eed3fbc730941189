"""Write (tag given) or compare VJP and recomputed GN-product outputs of configs 2-4 bitwise: used to
check that a performance change of the adjoint kernels keeps their results bit for bit
(usage: adj_bitwise.py save TAG | adj_bitwise.py cmp TAG_A TAG_B)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
if sys.argv[1] == "save":
    import torch
    import paper_2604_26745_b200 as pg
    import pget_data as P
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    res = {}
    for cid in (2, 3, 4):
        gd = P.geometry_desc(cid)
        g = pg.Geometry(gd)
        lam, mu = P.make_phantom(cid)
        lp, mp = P.make_phantom_prime(cid)
        dl, dm = P.rod_directions(cid)
        w = (pg.forward(g, dev(lp), dev(mp)) - pg.forward(g, dev(lam), dev(mu))).contiguous()
        gl, gm = pg.vjp(g, dev(lam), dev(mu), w)
        ql, qm = pg.gn_apply(g, dev(lam), dev(mu), dev(dl), dev(dm), 1e-3, 0.25)
        for k, v in (("gl", gl), ("gm", gm), ("ql", ql), ("qm", qm)):
            res[f"cfg{cid}_{k}"] = v.cpu().numpy()
        # one LM iteration (cache build, cached gradient, 20 cached GN products)
        l0, m0 = P.initial_guess(gd["n_px"])
        y = pg.forward(g, dev(lam), dev(mu)).contiguous()
        sl, sm, st = pg.gn_cg_step(g, dev(l0), dev(m0), y, 1e-3, 0.0, 20)
        res[f"cfg{cid}_lm_sl"] = sl.cpu().numpy()
        res[f"cfg{cid}_lm_sm"] = sm.cpu().numpy()
    np.savez(os.path.join(out, f"adj_{sys.argv[2]}.npz"), **res)
    print("saved", sys.argv[2])
else:
    a = np.load(os.path.join(out, f"adj_{sys.argv[2]}.npz"))
    b = np.load(os.path.join(out, f"adj_{sys.argv[3]}.npz"))
    for k in a.files:
        print(k, "bitwise equal" if np.array_equal(a[k], b[k]) else f"DIFFER max {np.abs(a[k] - b[k]).max():.3e}")
