#!/usr/bin/env python
"""Benchmark of the PGET hot path on B200 (BASELINE.json metric:
"ray-samples/s for fwd/JVP/VJP and ms per LM iteration at 1 B200 vs roofline").

One step = one pass of the whole hot path over one
batch of synthetic config-4 input (BASELINE.json configs[3], the largest single-GPU
configuration with an LM iteration: hexagonal 127-rod assembly, N=256, 720 angles,
2x91 detectors, J=9, Poisson noise at 1e4 peak):
    forward(u) + JVP(u; du) + VJP(u; w) + one LM iteration (20 CG steps, alpha=1e-3,
    beta=0, trial evaluation)
value = nominal ray-sample passes per step x steps x ranks / max-over-ranks device time.
The same JSON line carries `per_config`: forward / JVP / VJP ray-samples/s, ms per LM
iteration and the per-kernel roofline fractions of configs 1-5 (the north star's
"throughput on the five synthetic assemblies"), with config 5's HBM GB/s.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU (torchrun): every rank runs an independent replica (the assemblies are
independent problems; no data-path collective) -> "scaling": "weak".
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ray-samples/s for fwd/JVP/VJP and ms per LM iteration at 1 B200 vs roofline"
SMEM_B_PER_CLK_SM = 128          # guide: smem/L1 crossbar bytes per clock per SM (fallback)
N_SM = 148
REF_ANGLES = {1: 90, 2: 36, 3: 18, 4: 18, 5: 36}   # oracle sample per config: ~1-3 s of host time per step


def smem_peak():
    """Shared-memory data-path peak per SM per clock: the measured LDS.128 figure
    (scripts/micro/smem_bw.cu, profiles/smem_peak.json) when committed, else the guide's nominal 128 B."""
    p = os.path.join(ROOT, "profiles", "smem_peak.json")
    try:
        d = json.load(open(p))
        return float(d["bytes_per_clk_per_sm"]), f"measured LDS.128 peak {d['bytes_per_clk_per_sm']:.1f} B/clk/SM (profiles/smem_peak.json)"
    except Exception:
        return float(SMEM_B_PER_CLK_SM), "nominal 128 B/clk/SM (B200_PROFILING guide)"


def measured_hbm():
    """The pool's measured HBM copy bandwidth (GB/s, MEASURED_PEAKS.json, driver-written), else None."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or None


# algorithmic shared-memory bytes per nominal ray-sample
ALG_BYTES = {"forward": 32, "jvp": 64, "vjp": 32 + 32 + 64, "gn": 64 + 32 + 64}


def lm_passes(n_cg):
    # forward(u) + VJP(r) + n_cg GN products (JVP+VJP each) + JVP(s) + forward(u+s)
    return {"forward": 2, "vjp": 1, "jvp": 1, "gn": n_cg}


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, n in enumerate(names):
                if len(r) > 3 + k and r[3 + k].lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg):
    """The workload string both arms report in `config` (BASELINE.json configs[cfg - 1])."""
    return (f"config {cfg.cid}: {cfg.lattice} phantom, N={cfg.n_px}, {cfg.n_angles} angles, 2x{cfg.n_det} det, "
            f"J={cfg.n_subrays}, B={cfg.batch}; step = fwd + JVP + VJP + 1 LM iteration ({cfg.n_cg} CG, "
            f"alpha={cfg.alpha}, beta=0, trial)")


def max_over_ranks(ms, world, device):
    """Device time of the slowest rank (all_reduce MAX over the process group): the job's clock."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_rate(units_per_step, steps, world, max_ms):
    """Whole-job throughput: every rank runs its own replica of the step (independent assemblies,
    no data-path collective, "scaling": "weak"), timed by the slowest rank."""
    return world * units_per_step * steps / (max_ms * 1e-3)


def reference_arm(args, rank, world):
    """--impl reference: the fp64 oracle (the paper has no code; the oracle is the reference
    arm for this tier) on a bounded sample of the same workload, on the host cores."""
    if rank != 0:
        return 0
    import oracle as O
    import pget_data as P
    cfg = P.CONFIGS[args.config]
    sample = cpu_sample(cfg, args.ref_angles or REF_ANGLES[cfg.cid])
    times = []
    for k in range(args.warmup + args.steps):
        dt, n = run_oracle_step(O, P, cfg, sample)
        if k >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = sample["samples_per_step"] * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "ray-samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(cfg), "sample": sample["desc"]},
        "cpu_baseline": {"value": value, "unit": "ray-samples/s", "cores": O.threads(), "kind": "oracle",
                         "sample": sample["desc"], "cpu_model": cpu_model(),
                         "omp_num_threads": os.environ.get("OMP_NUM_THREADS", f"unset (OpenMP default: {O.threads()} threads)")},
        "e2e": {"value": value, "unit": "ray-samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_sample(cfg, n_angles):
    import oracle as O
    import pget_data as P
    gd = P.geometry_desc(cfg.cid, n_angles=n_angles, batch=1)
    t = O.tables(gd)
    cl = t["clip"]
    nominal = int(np.clip(cl[..., 1] - cl[..., 0] + 1, 0, None).sum())
    lam, mu = P.make_phantom(cfg.cid)
    lam, mu = lam[:1], mu[:1]
    dl, dm = P.rod_directions(cfg.cid)
    dl, dm = dl[:1], dm[:1]
    l0, m0 = P.initial_guess(cfg.n_px)
    y = P.poisson_noise(O.forward(gd, lam, mu), cfg.noise_peak or 1e4, cfg.seed)
    w = (O.forward(gd, lam * 1.05, mu) - O.forward(gd, lam, mu)).astype(np.float32)
    passes = 3 + sum(v * (2 if k == "gn" else 1) for k, v in lm_passes(cfg.n_cg).items())
    return dict(gd=gd, lam=lam, mu=mu, dl=dl, dm=dm, l0=l0, m0=m0, y=y, w=w, nominal=nominal,
                samples_per_step=nominal * passes,
                desc=f"one step (fwd+JVP+VJP+1 LM iteration, {cfg.n_cg} CG) of config {cfg.cid} restricted to "
                     f"{n_angles} of {cfg.n_angles} angles ({nominal} nominal samples/pass, {passes} passes)")


def run_oracle_step(O, P, cfg, s):
    t0 = time.perf_counter()
    O.forward(s["gd"], s["lam"], s["mu"])
    O.jvp(s["gd"], s["lam"], s["mu"], s["dl"], s["dm"])
    O.vjp(s["gd"], s["lam"], s["mu"], s["w"])
    O.gn_cg_step(s["gd"], s["l0"], s["m0"], s["y"], cfg.alpha, 0.0, cfg.n_cg)
    return time.perf_counter() - t0, s["samples_per_step"]


def roofline_ncu(cid, dom):
    """The north star's ncu view of the dominant kernel(s): speed-of-light fractions (issue slots,
    FP32 and SFU pipes, L1/shared) from the committed ncu capture (profiles/ncu_sol.json, written by
    scripts/ncu_summary.py); for the segmented modes one entry per phase kernel, weighted by time."""
    p = os.path.join(ROOT, "profiles", "ncu_sol.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        sol = d.get(f"cfg{cid}", {})
        parts = {k: v for k, v in sol.items() if (k == dom or k.startswith(dom + " ")) and "#" not in k}
        if not parts:
            return None
        out = {"source": d.get("source"), "kernels": parts}
        T = sum(v["duration_us"] or 0.0 for v in parts.values())
        for key in ("sm_sol_pct", "issue_active_pct", "l1_smem_pct", "fma_pipe_pct", "xu_pipe_pct"):
            out[key + "_time_weighted"] = (sum((v[key] or 0.0) * (v["duration_us"] or 0.0) for v in parts.values()) / T
                                           if T else None)
        return out
    except Exception:
        return None


def measure_config(pg, P, cid, flush, sm_mhz, reps=5, **desc_over):
    """Per-config block (not the headline value): forward / JVP / VJP nominal ray-samples/s and ms per
    LM iteration (median over reps of CUDA-event timings on the current stream, L2 flushed before each
    op), the projector launches' algorithmic roofline fractions (bytes per traced sample of
    ALG_BYTES x traced samples / average launch time / shared-memory peak), and for config 5 (the
    batched case) the HBM GB/s of the operations' algorithmic bytes (inputs read + outputs written)."""
    import torch
    cfg = P.CONFIGS[cid]
    gd = P.geometry_desc(cid, **desc_over)
    g = pg.Geometry(gd)
    nominal, traced, traced_j = (g.info[k] for k in ("n_samples_nominal", "n_samples_traced", "n_samples_traced_jvp"))
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    lam, mu = map(dev, P.make_phantom(cid))
    dl, dm = map(dev, P.rod_directions(cid))
    lp, mp = map(dev, P.make_phantom_prime(cid))
    l0, m0 = map(dev, P.initial_guess(cfg.n_px, cfg.batch))
    y_clean = pg.forward(g, lam, mu)
    w = (pg.forward(g, lp, mp) - y_clean).contiguous()
    y_meas = dev(P.poisson_noise(y_clean.cpu().numpy(), cfg.noise_peak or 1e4, cfg.seed))
    y, dy = torch.empty(g.sino_shape, device="cuda"), torch.empty(g.sino_shape, device="cuda")
    gl, gm = torch.empty(g.img_shape, device="cuda"), torch.empty(g.img_shape, device="cuda")
    sl, sm = torch.empty(g.img_shape, device="cuda"), torch.empty(g.img_shape, device="cuda")
    stats = pg.stats_buffer(g)
    ops = {
        "forward": lambda: pg.forward(g, lam, mu, y=y),
        "jvp": lambda: pg.jvp(g, lam, mu, dl, dm, dy=dy),
        "vjp": lambda: pg.vjp(g, lam, mu, w, g_lam=gl, g_mu=gm),
        "lm": lambda: pg.gn_cg_step(g, l0, m0, y_meas, cfg.alpha, 0.0, cfg.n_cg, pg.PGET_GN_EVAL_TRIAL, s_lam=sl,
                                    s_mu=sm, stats=stats),
    }
    nrep = {k: (max(2, reps // 2) if (k == "lm" and cid in (4, 5)) else reps) for k in ops}
    ms = {}
    for k, f in ops.items():
        f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(nrep[k]):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms[k] = statistics.median(ts)
    # per projector launch (CUDA events around each launch inside the library), one more pass
    pg.profile_begin(256)
    for k in ("forward", "jvp", "vjp"):
        flush.zero_()
        ops[k]()
    torch.cuda.synchronize()
    prof = pg.profile_end()
    pg.profile_begin(256)
    ops["lm"]()
    torch.cuda.synchronize()
    prof_lm = pg.profile_end()
    bpc, _ = smem_peak()
    peak = bpc * N_SM * sm_mhz * 1e6
    kern = {}
    for mode, pr in (("forward", prof), ("jvp", prof), ("vjp", prof), ("gn", prof_lm)):
        n = pr["launches"][mode]
        if not n:
            continue
        lms = pr["ms"][mode] / n
        units = traced_j if mode == "jvp" else traced
        ach = ALG_BYTES[mode] * units / (lms * 1e-3)
        kern[mode] = {"launch_ms": lms, "alg_bytes_per_traced_sample": ALG_BYTES[mode], "traced_samples": units,
                      "achieved_GBps": ach / 1e9, "frac": ach / peak}
    out = {
        "workload": f"{cfg.lattice} N={cfg.n_px} angles={cfg.n_angles} J={cfg.n_subrays} B={cfg.batch}"
                    + "".join(f" {k}={v}" for k, v in desc_over.items()),
        "nominal_samples_per_pass": nominal, "traced_samples_per_pass": traced, "traced_samples_jvp": traced_j,
        "forward_ms": ms["forward"], "jvp_ms": ms["jvp"], "vjp_ms": ms["vjp"], "lm_ms": ms["lm"],
        "forward_samples_per_s": nominal / (ms["forward"] * 1e-3),
        "jvp_samples_per_s": nominal / (ms["jvp"] * 1e-3),
        "vjp_samples_per_s": nominal / (ms["vjp"] * 1e-3),
        "lm_samples_per_s": nominal * (3 + 2 * cfg.n_cg) / (ms["lm"] * 1e-3),
        "kernels": kern,
        "reps": nrep,
    }
    if cfg.batch > 1:
        img, sino = 4 * int(np.prod(g.img_shape)), 4 * int(np.prod(g.sino_shape))
        byts = {"forward": 2 * img + sino, "jvp": 4 * img + sino, "vjp": 2 * img + sino + 2 * img}
        tot = sum(byts.values())
        t = (ms["forward"] + ms["jvp"] + ms["vjp"]) * 1e-3
        out["hbm"] = {"alg_bytes_fwd_jvp_vjp": tot, "GBps": tot / t / 1e9,
                      "basis": "inputs read + outputs written once per op (lam, mu, dlam, dmu, w; y, dy, g_lam, g_mu)"}
        # the batched LM's HBM-bound kernel: the GN product streams the coefficient cache (DRAM bytes per
        # launch from the committed ncu capture, profiles/traffic.json) in the launch time measured here
        try:
            tb = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(f"cfg{cid}", {}).get("gn")
        except (OSError, ValueError):
            tb = None
        if tb and "gn" in kern:
            gbs = tb / (kern["gn"]["launch_ms"] * 1e-3) / 1e9
            peak_hbm = measured_hbm()
            out["hbm"]["gn_product"] = {"dram_bytes_per_launch": tb, "launch_ms": kern["gn"]["launch_ms"], "GBps": gbs,
                                        "peak_GBps": peak_hbm, "frac": gbs / peak_hbm if peak_hbm else None,
                                        "basis": "ncu dram read+write per GN launch pair (profiles/traffic.json) / "
                                                 "CUDA-event launch time; peak = MEASURED_PEAKS.json hbm_gbs"}
    del g
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--ref-angles", type=int, default=0, help="oracle sample angles (0: per-config default)")
    ap.add_argument("--no-per-config", action="store_true", help="skip the configs 1-5 block")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the step directly instead of a CUDA graph")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2604_26745_b200 as pg
    import pget_data as P

    if args.warmup < 3:
        args.warmup = 3
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    cfg = P.CONFIGS[args.config]
    gd = P.geometry_desc(cfg.cid)
    g = pg.Geometry(gd, device=local)
    nominal = g.info["n_samples_nominal"]
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()

    # ---- synthetic inputs (seeded; per-rank replica), resident in HBM before timing
    lam_h, mu_h = P.make_phantom(cfg.cid)
    dl_h, dm_h = P.rod_directions(cfg.cid)
    lp_h, mp_h = P.make_phantom_prime(cfg.cid)
    l0_h, m0_h = P.initial_guess(cfg.n_px, cfg.batch)
    lam, mu, dl, dm, lp, mp, l0, m0 = map(dev, (lam_h, mu_h, dl_h, dm_h, lp_h, mp_h, l0_h, m0_h))
    y_clean = pg.forward(g, lam, mu)
    w = (pg.forward(g, lp, mp) - y_clean).contiguous()
    y_meas = dev(P.poisson_noise(y_clean.cpu().numpy(), cfg.noise_peak or 1e4, cfg.seed))
    torch.cuda.synchronize()

    # outputs / workspaces preallocated (the library never allocates)
    y = torch.empty(g.sino_shape, device="cuda")
    dy = torch.empty_like(y)
    gl = torch.empty(g.img_shape, device="cuda")
    gm = torch.empty_like(gl)
    sl = torch.empty_like(gl)
    sm = torch.empty_like(gl)
    stats = pg.stats_buffer(g)
    ws = {op: g.workspace(op) for op in ("forward", "jvp", "vjp", "gn_cg_step")}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def step(ev=None):
        if ev: ev[0].record()
        pg.forward(g, lam, mu, y=y, ws=ws["forward"])
        if ev: ev[1].record()
        pg.jvp(g, lam, mu, dl, dm, dy=dy, ws=ws["jvp"])
        if ev: ev[2].record()
        pg.vjp(g, lam, mu, w, g_lam=gl, g_mu=gm, ws=ws["vjp"])
        if ev: ev[3].record()
        pg.gn_cg_step(g, l0, m0, y_meas, cfg.alpha, 0.0, cfg.n_cg, pg.PGET_GN_EVAL_TRIAL, s_lam=sl, s_mu=sm,
                      stats=stats, ws=ws["gn_cg_step"])
        if ev: ev[4].record()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    passes = {"forward": 1, "jvp": 1, "vjp": 1}
    lmp = lm_passes(cfg.n_cg)
    sample_passes = 3 + sum(v * (2 if k == "gn" else 1) for k, v in lmp.items())
    samples_per_step = nominal * sample_passes

    # ---- the whole step captured once in a CUDA graph (every library launch is capturable, the
    #      cooperative CG kernel included; replays give bit-identical results) and replayed; the
    #      library launches of one step are counted during the capture
    if args.no_graph:
        run_step = step
        per_step_launches = None
    else:
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        gstep = torch.cuda.CUDAGraph()
        pg.profile_begin(0)
        with torch.cuda.graph(gstep, stream=cs):
            step()
        per_step_launches = pg.profile_end()["total_launches"]
        torch.cuda.synchronize()
        run_step = gstep.replay
        for _ in range(2):
            run_step()
        torch.cuda.synchronize()

    # ---- the timed region (value): K whole steps, events at the step boundaries only, library
    #      launches counted (pget_profile_begin(0): counting, no per-launch events)
    se = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    pg.profile_begin(0)
    for k in range(args.steps):
        flush.zero_()                       # L2 flush between timed steps (outside the events)
        se[k][0].record()
        run_step()
        se[k][1].record()
    torch.cuda.synchronize()
    launches = pg.profile_end()["total_launches"]
    if per_step_launches is not None:        # graph replays bypass the host-side counter
        launches = per_step_launches * args.steps
    if world > 1:
        dist.barrier()
    total_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in se), world, "cuda")

    # ---- breakdown pass (not the value): per-phase events and per-projector-launch events
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    pg.profile_begin(args.steps * (8 + 2 * cfg.n_cg) + 64)
    for k in range(args.steps):
        flush.zero_()
        step(evs[k])
    torch.cuda.synchronize()
    prof = pg.profile_end()
    clk = clocks.stop()
    phase = {"forward": 0.0, "jvp": 0.0, "vjp": 0.0, "lm": 0.0}
    for e in evs:
        phase["forward"] += e[0].elapsed_time(e[1])
        phase["jvp"] += e[1].elapsed_time(e[2])
        phase["vjp"] += e[2].elapsed_time(e[3])
        phase["lm"] += e[3].elapsed_time(e[4])

    # ---- end to end through the public API with host buffers (pinned), copies timed
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).pin_memory()
        h_in = [pin(a) for a in (lam_h, mu_h, dl_h, dm_h, l0_h, m0_h)] + [pin(w.cpu().numpy()),
                                                                          pin(y_meas.cpu().numpy())]
        d_in = [torch.empty(x.shape, device="cuda") for x in h_in]
        h_out = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (y, dy, gl, gm, sl, sm, stats)]
        bi = sum(x.numel() * x.element_size() for x in h_in)
        bo = sum(x.numel() * x.element_size() for x in h_out)

        def e2e_step():
            for hh, dd in zip(h_in, d_in):
                dd.copy_(hh, non_blocking=True)
            L, M, DL, DM, L0, M0, W, Y = d_in
            pg.forward(g, L, M, y=y, ws=ws["forward"])
            pg.jvp(g, L, M, DL, DM, dy=dy, ws=ws["jvp"])
            pg.vjp(g, L, M, W, g_lam=gl, g_mu=gm, ws=ws["vjp"])
            pg.gn_cg_step(g, L0, M0, Y, cfg.alpha, 0.0, cfg.n_cg, pg.PGET_GN_EVAL_TRIAL, s_lam=sl, s_mu=sm,
                          stats=stats, ws=ws["gn_cg_step"])
            for hh, dd in zip(h_out, (y, dy, gl, gm, sl, sm, stats)):
                hh.copy_(dd, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        run_e2e = e2e_step
        if not args.no_graph:   # the copies and the step captured together, as the user would
            ce = torch.cuda.Stream()
            ce.wait_stream(torch.cuda.current_stream())
            ge = torch.cuda.CUDAGraph()
            with torch.cuda.graph(ge, stream=ce):
                e2e_step()
            torch.cuda.synchronize()
            run_e2e = ge.replay
            run_e2e()
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            a.record()
            run_e2e()
            b.record()
            b.synchronize()
            tot += a.elapsed_time(b)
        e2e = {"value": job_rate(samples_per_step, args.steps, world, max_over_ranks(tot, world, "cuda")),
               "unit": "ray-samples/s",
               "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo}

    # ---- roofline of the dominant kernel (GN normal product projector) from live CUDA events
    dom = max(prof["ms"], key=lambda k: prof["ms"][k])
    n_launch = max(prof["launches"][dom], 1)
    per_launch_ms = prof["ms"][dom] / n_launch
    traced = g.info["n_samples_traced"]
    units = traced                                      # samples one launch actually evaluates
    achieved_gbs = ALG_BYTES[dom] * units / (per_launch_ms * 1e-3) / 1e9
    sm_mhz = (clk or {}).get("sm_mhz") or 1965.0
    bpc, peak_src = smem_peak()
    peak_gbs = bpc * N_SM * sm_mhz * 1e6 / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"cfg{cfg.cid}", {}).get(dom)
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle as O
        s = cpu_sample(cfg, args.ref_angles or REF_ANGLES[cfg.cid])
        dt, n = run_oracle_step(O, P, cfg, s)
        cpu = {"value": n / dt, "unit": "ray-samples/s", "cores": O.threads(), "kind": "oracle",
               "sample": s["desc"], "cpu_model": cpu_model(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS", f"unset (OpenMP default: {O.threads()} threads)")}

    per_config = None
    if rank == 0 and world == 1 and not args.no_per_config:
        del ws
        torch.cuda.empty_cache()
        per_config = {}
        for cid in (1, 2, 3, 4, 5):
            per_config[f"config {cid}"] = measure_config(pg, P, cid, flush, sm_mhz)
            torch.cuda.empty_cache()
        # the paper's own detector geometry: the banks interleaved by half a pitch, where
        # neither the duplicate angle-banks nor the line pairing apply (every nominal sample is traced)
        for cid in (2, 4):
            per_config[f"config {cid} interleaved banks"] = measure_config(pg, P, cid, flush, sm_mhz,
                                                                           bank1_shift=0.5)
            torch.cuda.empty_cache()

    if rank == 0:
        value = job_rate(samples_per_step, args.steps, world, total_ms)
        K = args.steps
        line = {
            "metric": METRIC, "value": value, "unit": "ray-samples/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload(cfg),
                       "nominal_samples_per_pass": nominal, "traced_samples_per_pass": traced,
                       "angle_banks_merged": bool(g.info["angle_banks_merged"]),
                       "sample_passes_per_step": sample_passes,
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "launch": "direct" if args.no_graph else "the whole step captured once as a CUDA graph, replayed"},
            "per_op": {
                "forward_samples_per_s": nominal * K / (phase["forward"] * 1e-3),
                "jvp_samples_per_s": nominal * K / (phase["jvp"] * 1e-3),
                "vjp_samples_per_s": nominal * K / (phase["vjp"] * 1e-3),
                "lm_ms": phase["lm"] / K,
                "forward_ms": phase["forward"] / K, "jvp_ms": phase["jvp"] / K, "vjp_ms": phase["vjp"] / K,
                "projector_ms_per_launch": {k: (prof["ms"][k] / prof["launches"][k] if prof["launches"][k] else None)
                                            for k in prof["ms"]},
            },
            "roofline": {"bound": "alu", "pipe": f"shared-memory data path ({bpc:.1f} B/clk/SM)", "kernel": ({"gn": "gn: seg_a_kernel<GN> + gnw_kernel + gnb_kernel (recomputed J p, scatter weights, cached fixed-point scatter; per CG step, timed together)",
                                    "vjp": "vjp: seg_a_kernel + seg_b_kernel (segmented adjoint, one launch pair)"}.get(dom, f"proj_kernel<{dom}>")),
                         "achieved": achieved_gbs, "peak": peak_gbs, "unit": "GB/s", "frac": achieved_gbs / peak_gbs,
                         "traffic": traffic,
                         "peak_basis": f"{peak_src} x 148 SMs x {sm_mhz:.0f} MHz (median SM clock under load)",
                         "alg_bytes_per_sample": ALG_BYTES[dom], "units_per_launch": units,
                         "launch_ms": per_launch_ms},
            "roofline_ncu": roofline_ncu(cfg.cid, dom),
            # SURVEY.md 8(d)'s bound model of the LM iteration on NOMINAL samples: 43 pass-equivalents
            # (2 forward x 32 B + 21 VJP-class x 96 B + 20 JVP-class x 64 B per nominal sample) through
            # the shared-memory crossbar; frac > 1 means the line pairing / duplicate merging saved
            # more than the kernels lose to the crossbar
            "lm_bound_model": {
                "bound_ms": nominal * (2 * 32 + 21 * 96 + 20 * 64) / (peak_gbs * 1e9) * 1e3,
                "measured_ms": phase["lm"] / K,
                "frac": (nominal * (2 * 32 + 21 * 96 + 20 * 64) / (peak_gbs * 1e9) * 1e3) / (phase["lm"] / K),
                "basis": f"SURVEY.md 8(d): nominal samples x 3360 B at {peak_src} x 148 SMs x SM clock"},
            "cpu_baseline": cpu,
            "per_config": per_config,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
