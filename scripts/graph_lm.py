"""One LM iteration (pget_gn_cg_step, 20 CG steps) launched directly vs captured once in a CUDA graph
and replayed (every library launch, including the cooperative CG kernel, is capturable)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26745_b200 as pg  # noqa: E402
import pget_data as P  # noqa: E402

for cid in [int(c) for c in sys.argv[1:]] or [1, 2]:
    gd = P.geometry_desc(cid)
    g = pg.Geometry(gd)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    lam, mu = map(dev, P.make_phantom(cid))
    l0, m0 = map(dev, P.initial_guess(gd["n_px"], gd["batch"]))
    y = pg.forward(g, lam, mu)
    sl = torch.empty(g.img_shape, device="cuda")
    sm = torch.empty_like(sl)
    st = pg.stats_buffer(g)
    ws = g.workspace("gn_cg_step")
    step = lambda: pg.gn_cg_step(g, l0, m0, y, 1e-3, 0.0, 20, s_lam=sl, s_mu=sm, stats=st, ws=ws)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    ref = st.clone()

    def timeit(f, n=20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(n):
            f()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / n

    t_direct = timeit(step)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    gr.replay()
    torch.cuda.synchronize()
    same = bool(torch.equal(st, ref))
    t_graph = timeit(gr.replay)
    print(f"cfg{cid} LM direct {t_direct:.3f} ms  graph replay {t_graph:.3f} ms  stats identical: {same}", flush=True)
