"""Diagnose the bench's timed loop: events at step boundaries with and without a host sync per step,
with and without nvidia-smi sampling running (config 2 step: fwd + JVP + VJP + one LM iteration)."""
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26745_b200 as pg  # noqa: E402
import pget_data as P  # noqa: E402

cfg = P.CONFIGS[2]
gd = P.geometry_desc(2)
g = pg.Geometry(gd)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
lam, mu = map(dev, P.make_phantom(2))
dl, dm = map(dev, P.rod_directions(2))
l0, m0 = map(dev, P.initial_guess(128))
y = pg.forward(g, lam, mu)
ym = y.clone()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def step():
    pg.forward(g, lam, mu, y=y)
    pg.jvp(g, lam, mu, dl, dm)
    pg.vjp(g, lam, mu, y)
    pg.gn_cg_step(g, l0, m0, ym, 1e-3, 0.0, 20)


def run(K, sync, flush_between=True):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for a, b in ev:
        if flush_between:
            flush.zero_()
        a.record()
        step()
        b.record()
        if sync:
            b.synchronize()
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in ev])


for _ in range(3):
    step()
for name, kw in [("nosync", dict(sync=False)), ("sync", dict(sync=True)), ("nosync-noflush", dict(sync=False, flush_between=False))]:
    t = run(10, **kw)
    print(f"{name:16s} mean {t.mean():.3f} ms  min {t.min():.3f}  max {t.max():.3f}", flush=True)
FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
          "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
          "clocks_event_reasons.sw_power_cap")
pg.profile_begin(0)
t = run(10, sync=False)
pg.profile_end()
print(f"{'nosync+count':16s} mean {t.mean():.3f} ms  min {t.min():.3f}  max {t.max():.3f}", flush=True)
p = subprocess.Popen(["nvidia-smi", f"--query-gpu={FIELDS}", "--format=csv,noheader,nounits", "-lms", "100"],
                     stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
t = run(10, sync=False)
print(f"{'nosync+smi':16s} mean {t.mean():.3f} ms  min {t.min():.3f}  max {t.max():.3f}", flush=True)
t = run(10, sync=True)
print(f"{'sync+smi':16s} mean {t.mean():.3f} ms  min {t.min():.3f}  max {t.max():.3f}", flush=True)
p.terminate()
