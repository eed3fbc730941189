"""Summarise ncu evidence for profiles/: per-kernel launch-time shares from a
`--metrics gpu__time_duration.sum --csv` launch list, and key metrics from a `--set full`
report (imported with `ncu -i ... --page raw --csv`).  Also writes profiles/traffic.json
(dram read+write bytes per launch of each projector mode) for bench.py's roofline.traffic."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODES = {"0": "forward", "1": "jvp", "2": "vjp", "3": "gn"}
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"), ("launch__block_size", "block"), ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / instruction"),
    ("dram__bytes_read.sum", "dram read"), ("dram__bytes_write.sum", "dram write"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math throttle"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM SOL %"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for d in data:
        name = d[ki].split("(")[0].replace("void ", "")
        tot[name] += float(d[vi].replace(",", "")) * scale[d[ui]]
        cnt[name] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / T:.1f} % | {v / cnt[k]:.2f} |")
    return out, len(data), T


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        name = d[hdr.index("Kernel Name")]
        if "proj_kernel<" in name:
            mode = MODES.get(name.split("<")[1].split(",")[0].strip(), "?")
        elif "seg_a_kernel<" in name or "seg_b_kernel<" in name:   # segmented adjoint: phase A / B
            mode = MODES.get(name.split("<")[1].split(",")[0].strip(), "?") + (" A" if "seg_a" in name else " B")
        elif "gnb_kernel" in name:       # GN scatter from the coefficient cache (phase B of the GN product)
            mode = "gn B"
        elif "lin_kernel" in name:       # the cache build, once per LM iteration
            mode = "lin"
        else:
            mode = name
        seen = [m for m, _, _ in res]
        if mode in seen:                 # e.g. the VJP-mode phase A that precedes the cache build
            mode = mode + " #%d" % (seen.count(mode) + 1 + sum(1 for x in seen if x.startswith(mode + " #")))
        vals = {}
        for k, lab in KEYS:
            if k in hdr:
                vals[lab] = (d[hdr.index(k)], units[hdr.index(k)])
        res.append((mode, name, vals))
    return res


def main():
    # usage: ncu_summary.py TAG LAUNCH_LIST.csv [FULL.ncu-rep|-] [CONFIG_ID]
    tag = sys.argv[1]
    lst, rep = sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "-"
    cid = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    lines = [f"# ncu summary, round {tag}", "",
             "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` of "
             f"`python bench.py --config {cid} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config` "
             f"(config {cid}; cold-cache, serialised launches: compare shares, not absolute times).", ""]
    if lst == "-":   # no launch list for this capture
        lines = [f"# ncu summary, round {tag}", ""]
    else:
        tab, n, T = launches(lst)
        lines += [f"{n} launches, {T / 1e3:.2f} ms total.", ""] + tab + [""]
    if rep == "-":
        out = os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.md")
        open(out, "w").write("\n".join(lines) + "\n")
        print(out)
        return
    lines += ["Full capture: `ncu --set full --clock-control none --import-source on -k regex:\"proj_kernel|seg_|lin_kernel|gnb_kernel\" -c 8 "
              f"python scripts/prof_ops.py {cid} 1` (one launch of each projector kernel, config {cid}: forward "
              "fused, JVP segmented, VJP as segmented phases A and B, GN as the VJP-mode phase A + cache build (lin) + GN-mode phase A + cached scatter (gnb)).", ""]
    res = full(rep)
    labs = [lab for _, lab in KEYS]
    lines.append("| metric | " + " | ".join(m for m, _, _ in res) + " |")
    lines.append("|---|" + "---|" * len(res))
    for lab in labs:
        cells = []
        for _, _, v in res:
            x = v.get(lab)
            cells.append(f"{x[0]} {x[1]}".strip() if x else "")
        lines.append(f"| {lab} | " + " | ".join(cells) + " |")
    out = os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.md")
    open(out, "w").write("\n".join(lines) + "\n")
    traffic = {}
    for mode, _, v in res:
        rb, wb = v.get("dram read"), v.get("dram write")
        if rb and wb:
            mult = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}
            if "#" in mode or mode == "lin":   # not part of one launch of a mode
                continue
            key = mode.split(" ")[0]   # the two phases of a segmented mode add up to one launch of that mode
            traffic[key] = traffic.get(key, 0.0) + float(rb[0].replace(",", "")) * mult[rb[1]] + \
                float(wb[0].replace(",", "")) * mult[wb[1]]
    # ncu speed-of-light fractions per kernel (the north star's "FP32/SFU issue" roofline as ncu
    # measures it), for bench.py's roofline_ncu
    sol = {}
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for mode, name, v in res:
        def num(lab):
            x = v.get(lab)
            return float(x[0].replace(",", "")) if x else None
        dur = v.get("duration")
        dur_us = float(dur[0].replace(",", "")) * tscale.get(dur[1], 1.0) if dur else None
        sol[mode] = {"kernel": name.split("(")[0].replace("void ", ""), "duration_us": dur_us,
                     "sm_sol_pct": num("SM SOL %"), "issue_active_pct": num("issue active %"),
                     "l1_smem_pct": num("L1/smem throughput %"), "fma_pipe_pct": num("FMA pipe %"),
                     "xu_pipe_pct": num("XU (MUFU) %")}
    sp = os.path.join(ROOT, "profiles", "ncu_sol.json")
    olds = json.load(open(sp)) if os.path.exists(sp) else {}
    olds[f"cfg{cid}"] = sol
    olds.setdefault("sources", {})[f"cfg{cid}"] = f"profiles/ncu_summary_{tag}.md"
    olds["source"] = f"profiles/ncu_summary_{tag}.md"
    json.dump(olds, open(sp, "w"), indent=1)
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    old = json.load(open(tp)) if os.path.exists(tp) else {}
    old[f"cfg{cid}"] = traffic
    old["source"] = f"profiles/ncu_summary_{tag}.md (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch)"
    json.dump(old, open(tp, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
