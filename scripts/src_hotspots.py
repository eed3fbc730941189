"""Aggregate an `ncu --page source --print-source cuda,sass --csv` export per CUDA source line:
warp-instructions executed, stall samples, shared wavefronts.  Usage: src_hotspots.py export.csv [top]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = None
cur_line, cur_src = None, None
agg = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        idx = {name: i for i, name in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    if r[0].strip():
        cur_line, cur_src = r[0], r[1]
    try:
        ins = float(r[idx["Instructions Executed"]] or 0)
        smp = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        wf = float(r[idx["L1 Wavefronts Shared"]] or 0)
    except (ValueError, KeyError, IndexError):
        continue
    a = agg[cur_line]
    a[0] += ins
    a[1] += smp
    a[2] += wf
    a[3] = cur_src
tot = [sum(v[k] for v in agg.values()) for k in range(3)]
print(f"total warp-inst {tot[0]:.4g}  stall samples {tot[1]:.4g}  smem wavefronts {tot[2]:.4g}")
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{ln:>5} inst {100 * v[0] / tot[0]:5.1f}%  stall {100 * v[1] / max(tot[1], 1):5.1f}%  wf {100 * v[2] / max(tot[2], 1):5.1f}%  {v[3].strip()[:90]}")
