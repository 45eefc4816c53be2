#!/usr/bin/env python
"""Benchmark of the SpMV hot path (arXiv 2212.08964) on B200 -- prints ONE JSON line.

  python bench.py [--gpus N --steps K --warmup W] [--config c3] [--schedule merge_path]
  python bench.py --impl reference ...      # the CPU oracle arm (rank 0 only)

A "step" is one pass of the whole merge-path method over the workload: lb_partition (Alg.3
2DSearch), the tile processor and the carry fix-up, all inside one lb_spmv_ex(REPARTITION) call
(N=1).  With N>1 (torchrun, one process per GPU) a step is lb_spmv_multi: the rank's equal-nnz
row shard of R-MAT scale-26 followed by the NCCL all-gather of y.

value = nonzeros processed by all ranks / max-over-ranks step time, in GNZ/s.  Inputs are
resident in HBM when the timed region starts; they are larger than L2 (no flush between steps).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import lbgen  # noqa: E402

FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="c1..c6 (default: c3 at N=1, c5 at N>1)")
    ap.add_argument("--schedule", default="merge_path")
    ap.add_argument("--items-per-tile", type=int, default=0, help="merge-path tile length L (0: library default)")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / cpu_baseline / clocks (profiling runs)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="budget for the cpu_baseline sample")
    ap.add_argument("--multi", action="store_true", help="use the multi-GPU step even at world size 1 (testing)")
    ap.add_argument("--overlap", action="store_true",
                    help="multi-GPU step with LB_SPMV_CHUNKED: each chunk's rows all-gathered while the next computes")
    ap.add_argument("--fused", action="store_true",
                    help="multi-GPU step with the all-gather fused into the tile kernel (lb_spmv_multi_fused)")
    ap.add_argument("--classes", default="c2,c4,c5",
                    help="extra matrix classes reported beside the headline at N=1 ('' = none)")
    ap.add_argument("--hot-slots", type=int, default=0,
                    help="hot-column plan (lb_csr_plan_hot_x) slot budget: 0 = library default, -1 = no plan")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers

def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        if "hbm_gbs" in d:
            return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (torch copy, read+write)"
    return FALLBACK_HBM_GBS, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def compulsory_bytes(rows, cols, nnz):
    """col+val 8 B/nnz, offsets 4(rows+1), y 4 rows, x 4 cols (read at least once)."""
    return 8 * nnz + 4 * (rows + 1) + 4 * rows + 4 * cols


def ncu_traffic(cfg, sched, L, kernel, hot_slots=None):
    """DRAM bytes per launch of this kernel from a committed ncu --set full capture (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(f"{cfg}/{sched}/L{L}" + (f"/hot{hot_slots}" if hot_slots else ""))
    if e is None or e.get("kernel") != kernel.split(" ")[0]:
        return None
    return e.get("dram_bytes_per_launch")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms while running."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.out = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
                self.out, _ = self.p.communicate()

    def summary(self):
        if not self.out:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"], "samples": 0}
        rows = []
        for ln in self.out.strip().splitlines():
            f = [c.strip() for c in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append(dict(sm=float(f[1]), smax=float(f[2]), power=float(f[3]), util=float(f[4]),
                                 hw=f[5], hwt=f[6], swt=f[7], pcap=f[8]))
            except ValueError:
                continue
        load = [r for r in rows if r["util"] > 0] or rows
        if not load:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = {"hw": "hw_slowdown", "hwt": "hw_thermal_slowdown", "swt": "sw_thermal_slowdown",
                 "pcap": "sw_power_cap"}
        reasons = sorted({n for r in load for k, n in names.items() if r[k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(r["sm"] for r in load), "sm_max_mhz": max(r["smax"] for r in load),
                "reasons": reasons, "samples": len(load), "power_w_median": statistics.median(r["power"] for r in load),
                "power_w_max": max(r["power"] for r in load)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- per-class reporting

def graph_median(fn, reps: int = 50, warm: int = 5):
    """median over `reps` back-to-back replays of one CUDA-graph-captured call, each
    bracketed by CUDA events on the capturing stream, after `warm` warm-up replays."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(warm):
        g.replay()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for a, b in evs:
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    del g
    return float(np.median(ts)), float(ts[0]), float(ts[-1])


def traced_kernel_ms(M, x, y, sched, n: int = 50) -> float:
    """Mean duration of the main kernel over n back-to-back steps (lb_csr_trace_phases: CUDA events on
    the launch stream around each call's tile kernel)."""
    M.trace_phases(n)
    for _ in range(n):
        M.spmv(x, y, sched, repartition=True)
    tr = M.trace_read()
    M.trace_phases(0)
    return float(np.mean(tr[:, 1]))


def class_report(cfg: str, dev, reps: int = 50) -> dict:
    """BASELINE's metric is per matrix class: the step rate of merge-path (plain CSR and with the x-reuse
    plan), of the schedule AUTO picks, the dominant kernel's roofline fraction and its ncu DRAM bytes."""
    import paper_2212_08964_b200 as lb
    A = lbgen.make_config(cfg, "float", device=dev)
    x = lbgen.x_for_config(cfg, A.cols, "float", device=dev)
    rows, cols, nnz = A.rows, A.cols, A.nnz
    M = lb.CsrMatrix.from_csr(A, device=dev, validate=True)
    del A
    y = torch.empty(rows, device=dev)
    alg = compulsory_bytes(rows, cols, nnz)
    peak, _ = peak_hbm()
    out = {"desc": lbgen.CONFIG_DESC.get(cfg, cfg), "rows": rows, "nnz": nnz, "algorithmic_bytes": alg,
           "timing": f"median of {reps} CUDA-graph replays of one lb_spmv_ex(REPARTITION) step (CUDA events)"}

    def entry(sched):
        med, lo, hi = graph_median(lambda: M.spmv(x, y, sched, repartition=True), reps)
        kms = traced_kernel_ms(M, x, y, sched)
        return {"value": round(nnz / (med * 1e-3) / 1e9, 2), "unit": "GNZ/s", "ms": round(med, 5),
                "ms_min_max": [round(lo, 5), round(hi, 5)], "kernel": M.kernel_name(sched),
                "kernel_ms": round(kms, 5), "roofline_frac": round(alg / (kms * 1e-3) / 1e9 / peak, 4)}

    auto = M.select_schedule()
    out["auto_schedule"] = auto
    out["merge_path_no_plan"] = entry("merge_path")
    out["merge_path_no_plan"]["traffic"] = ncu_traffic(cfg, "merge_path", M.items_per_tile,
                                                       out["merge_path_no_plan"]["kernel"])
    if auto != "merge_path":
        out["auto"] = entry(auto)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hot_n, hot_nnz = M.plan_hot_x(0)
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t0) * 1e3
    if hot_n:
        info = M.plan_info()
        e = entry("merge_path")
        e["traffic"] = ncu_traffic(cfg, "merge_path", M.items_per_tile, e["kernel"], hot_n)
        e["plan"] = {"hot_cols": hot_n, "hot_nnz_frac": round(hot_nnz / max(nnz, 1), 4),
                     "warm_cols": info["warm_cols"], "warm_nnz_frac": round(info["warm_nnz"] / max(nnz, 1), 4),
                     "build_ms": round(build_ms, 2)}
        gain = out["merge_path_no_plan"]["ms"] - e["ms"]
        e["plan"]["break_even_steps"] = int(np.ceil(build_ms / gain)) if gain > 0 else None
        out["merge_path_plan"] = e
    else:
        out["merge_path_plan"] = {"skipped": "lb_csr_plan_hot_x found no column worth a slot"}
    M.plan_hot_x(-1)
    best = max((v for k, v in out.items() if isinstance(v, dict) and "value" in v), key=lambda v: v["value"])
    out["best"] = {"value": best["value"], "kernel": best["kernel"]}
    del M, x, y
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- reference arm (CPU oracle)

def cpu_sample(A: lbgen.Csr, x: torch.Tensor, target_nnz: int):
    """Leading rows of the workload holding ~target_nnz nonzeros, as host arrays."""
    off = A.row_offsets
    r = int(torch.searchsorted(off.to(torch.int64), torch.tensor([target_nnz], device=off.device)).item())
    r = max(1, min(r, A.rows))
    o = off[: r + 1].cpu()
    n = int(o[-1])
    return o, A.col_idx[:n].cpu(), A.values[:n].cpu(), x.cpu(), r, n


def time_oracle(sample, seconds: float, min_reps: int = 5):
    """The oracle SpMV (OpenMP over rows, fp64, the -O3 -march=native build of the same oracle.c) on the
    sample: median over >= min_reps repetitions, repeating until `seconds` have passed."""
    import oracle
    o, c, v, xx, r, n = sample
    oracle.spmv(o, c, v, xx, threads=True, timing=True)  # warm (and builds the native copy)
    ts, t_all = [], time.perf_counter()
    while len(ts) < min_reps or time.perf_counter() - t_all < seconds:
        t0 = time.perf_counter()
        oracle.spmv(o, c, v, xx, threads=True, timing=True)
        ts.append(time.perf_counter() - t0)
    med = float(np.median(ts))
    return n / med / 1e9, len(ts), time.perf_counter() - t_all


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_extras(sample, seconds: float) -> dict:
    """SURVEY 8(d) oracle timing beside the GPU: the single-threaded oracle SpMV and the brute-force
    (two-pointer walk, O(rows + nnz)) merge-path partitioner on the same sample, each median of up to 5."""
    import oracle
    o, c, v, xx, r, n = sample

    def med(fn):
        ts = []
        t_end = time.perf_counter() + seconds
        while len(ts) < 5 and (not ts or time.perf_counter() < t_end):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return float(np.median(ts)), len(ts)

    t1, n1 = med(lambda: oracle.spmv(o, c, v, xx, threads=False, timing=True))
    tp, npart = med(lambda: oracle.partition(o, 1016))
    return {"cpu_model": cpu_model(), "os_cpu_count": os.cpu_count(),
            "single_thread": {"value": round(n / t1 / 1e9, 4), "unit": "GNZ/s", "reps": n1,
                              "timing": "median (oracle.spmv, fp64, 1 thread)"},
            "partition_bruteforce": {"ms": round(tp * 1e3, 2), "items": int(r + n), "L": 1016, "reps": npart,
                                     "timing": "median (oracle.partition: two-pointer walk, 1 thread)"}}


def run_reference(args, cfg):
    world, rank, local = dist_env()
    if rank != 0:
        return
    import oracle
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    A = lbgen.make_config(cfg, "float", device=dev)
    x = lbgen.x_for_config(cfg, A.cols, "float", device=dev)
    sample = cpu_sample(A, x, 16_000_000 if cfg != "c1" else A.nnz)
    o, c, v, xx, r, n = sample
    for _ in range(args.warmup):
        oracle.spmv(o, c, v, xx, threads=True, timing=True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.spmv(o, c, v, xx, threads=True, timing=True)
    dt = time.perf_counter() - t0
    val = n * args.steps / dt / 1e9
    desc = f"leading {r} rows ({n} nnz) of {cfg}, full x; oracle.spmv_omp (fp64, gcc -O3 -march=native) per step"
    print(json.dumps({
        "impl": "reference", "metric": "SpMV GNZ/s", "value": round(val, 4), "unit": "GNZ/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg, "desc": lbgen.CONFIG_DESC.get(cfg, cfg), "sample": desc},
        "cpu_baseline": {"value": round(val, 4), "unit": "GNZ/s", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": round(val, 4), "unit": "GNZ/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ----------------------------------------------------------------------------- our arm

def run_single(args, cfg):
    import paper_2212_08964_b200 as lb
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    A = lbgen.make_config(cfg, "float", device=dev)
    x = lbgen.x_for_config(cfg, A.cols, "float", device=dev)
    rows, cols, nnz = A.rows, A.cols, A.nnz
    M = lb.CsrMatrix.from_csr(A, device=dev, validate=True)
    M.set_items_per_tile(args.items_per_tile)
    args.items_per_tile = M.items_per_tile
    y = torch.empty(rows, device=dev)
    stream = torch.cuda.current_stream()
    sched = args.schedule

    def step():
        M.spmv(x, y, sched, repartition=True)

    # the plain-CSR rate first (no plan), then the per-matrix hot-column plan the timed steps use
    no_plan = None
    plan = None
    if args.hot_slots >= 0 and sched == "merge_path":
        for _ in range(3):
            step()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_np = max(10, min(args.steps, 200))
        ea.record(stream)
        for _ in range(n_np):
            step()
        eb.record(stream)
        torch.cuda.synchronize()
        ms_np = ea.elapsed_time(eb) / n_np
        no_plan = {"value": round(nnz / (ms_np * 1e-3) / 1e9, 3), "ms_per_step": round(ms_np, 5),
                   "kernel": M.kernel_name(sched), "steps": n_np}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hot_n, hot_nnz = M.plan_hot_x(args.hot_slots)
        torch.cuda.synchronize()
        build_ms = (time.perf_counter() - t0) * 1e3
        plan = {"kind": "hot-column plan (lb_csr_plan_hot_x, DESIGN.md 6b)", "slots_requested": args.hot_slots,
                "hot_cols": hot_n, "hot_nnz_frac": round(hot_nnz / max(nnz, 1), 4),
                "build_ms": round(build_ms, 2), "built": "once per matrix, before the timed region",
                "break_even_steps": None}

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device()) if not args.no_extras else None
    if sampler:
        sampler.__enter__()
        # soak so the sampler sees steady-state clocks even if K steps are short
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 1.0:
            step()
        torch.cuda.synchronize()
    n0 = lb.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # every timed step records CUDA events on the launch stream around its kernels
    # (lb_csr_trace_phases), so the dominant kernel's duration is measured inside the timed region
    M.trace_phases(args.steps)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = lb.launch_count() - n0
    if sampler:
        sampler.__exit__()
    tr = M.trace_read()
    M.trace_phases(0)
    ms = e0.elapsed_time(e1) / args.steps
    value = nnz / (ms * 1e-3) / 1e9
    ph = np.mean(tr, axis=0)  # (partition, main, fix-up) ms per step, mean over the K timed steps
    main_ms = float(ph[1])
    main_share = main_ms / ms
    # the same step captured in a CUDA graph: median of 50 replays (SURVEY 8(d) reporting)
    g_med, g_min, g_max = graph_median(step, 50)
    alg = compulsory_bytes(rows, cols, nnz)
    peak, peak_src = peak_hbm()
    achieved = alg / (main_ms * 1e-3) / 1e9
    rec = {
        "metric": "SpMV GNZ/s", "value": round(value, 3), "unit": "GNZ/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (lbgen counter-hash generator, seeded)",
        "config": {"workload": cfg, "desc": lbgen.CONFIG_DESC.get(cfg, cfg), "rows": rows, "cols": cols, "nnz": nnz,
                   "schedule": sched, "items_per_tile": args.items_per_tile, "parallelism": "1 GPU",
                   "values": "uniform [-1,1) fp32", "step": "lb_spmv_ex(REPARTITION): partition" + (" + hot x gather" if plan and plan["hot_cols"] else "")
                   + " + tiles + fixup",
                   "l2": "inputs (%.2f GB) larger than the 126 MB L2; no flush between steps" % (alg / 1e9)},
        "plan": plan,
        "no_plan": no_plan,
        "gpu_launches": int(launches),
        "phase_ms": {"partition": round(float(ph[0]), 5), "main": round(float(ph[1]), 5), "fixup": round(float(ph[2]), 5),
                     "main_share": round(main_share, 4),
                     "from": "mean over the K timed steps of CUDA events recorded on the launch stream around each "
                             "phase (lb_csr_trace_phases)"},
        "graph": {"value": round(nnz / (g_med * 1e-3) / 1e9, 3), "unit": "GNZ/s", "median_ms": round(g_med, 5),
                  "min_max_ms": [round(g_min, 5), round(g_max, 5)],
                  "timing": "median of 50 replays of the step captured in a CUDA graph, CUDA events around each"},
        "roofline": {"bound": "hbm", "kernel": M.kernel_name(sched),
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic(cfg, sched, args.items_per_tile, M.kernel_name(sched),
                                          plan["hot_cols"] if plan and plan["hot_cols"] else None),
                     "algorithmic_bytes": alg,
                     "peak_source": peak_src,
                     "kernel_ms": round(main_ms, 5),
                     "kernel_ms_from": "mean duration of the tile kernel over the K timed steps (CUDA events on its "
                                       "launch stream, recorded by the library around every launch)"},
    }
    # the stream+gather ceiling of this matrix on this GPU (no row structure), measured live; the kernel
    # side of these two ratios is 20 short phase-timed calls, so both sides run at the same clocks
    ph_short = np.mean(np.array([M.phase_times(x, y, sched) for _ in range(20)]), axis=0)
    try:
        probe_ms = M.probe_stream_gather(x, reps=20)
        rec["roofline_gather"] = {
            "bound": "l1tex gather (~1 L1TEX line per clock per SM for random 4-byte x[col] not served from shared memory)",
            "achieved": round(nnz / (float(ph_short[1]) * 1e-3) / 1e9, 2), "peak": round(nnz / (probe_ms * 1e-3) / 1e9, 2),
            "unit": "GNZ/s", "frac": round(probe_ms / float(ph_short[1]), 4),
            "timing": "both right after the timed region: the kernel's phase-call time vs 20 probe passes",
            "peak_source": "lb_probe_stream_gather: same col/val/x" + (" and the same x-reuse plan (hot x in shared memory)"
                                                                     if plan and plan["hot_cols"] else "")
                           + ", 256-bit stream loads + gathers, no rows"}
    except Exception as e:  # pragma: no cover
        rec["roofline_gather"] = {"error": str(e)}
    # the read-only stream rate of this matrix's col_idx + values (no gathers): the in-repo stream
    # microbenchmark of SURVEY 8(d); the tile kernel's algorithmic GB/s against it
    try:
        st_ms = M.probe_stream(reps=20)
        st_gbs = 8.0 * nnz / (st_ms * 1e-3) / 1e9
        ach_ph = alg / (float(ph_short[1]) * 1e-3) / 1e9
        rec["roofline_stream"] = {
            "bound": "hbm (read-only stream)", "achieved": round(ach_ph, 1), "peak": round(st_gbs, 1), "unit": "GB/s",
            "frac": round(ach_ph / st_gbs, 4),
            "timing": "both right after the timed region: the kernel's phase-call time (algorithmic bytes) vs 20 probe passes",
            "peak_source": "lb_probe_stream: col_idx + values of this matrix, 256-bit evict-first loads, no gathers"}
    except Exception as e:  # pragma: no cover
        rec["roofline_stream"] = {"error": str(e)}
    if plan is not None and no_plan is not None and ms < no_plan["ms_per_step"]:
        plan["break_even_steps"] = int(np.ceil(plan["build_ms"] / (no_plan["ms_per_step"] - ms)))
    if args.no_extras:
        print(json.dumps(rec))
        return
    rec["clocks"] = sampler.summary()

    # end to end through the public C-ABI calls with HOST buffers, host<->device copies inside the timed
    # region.  `e2e`: the iterative-solver call lb_spmv_host_x -- the matrix (with its x-reuse plan) is
    # uploaded once, like a model's weights, and every step copies x in from pinned host memory, runs the
    # same lb_spmv_ex(REPARTITION) step and copies y out (the call synchronises; host clock per step).
    # `e2e_full_upload`: lb_spmv_host -- the whole CSR + x uploaded every step (PCIe-bound).
    hx, hy = x.cpu().pin_memory(), torch.empty(rows).pin_memory()
    chunked = plan is not None
    M.spmv_host(hx, hy, sched, repartition=True, chunked=chunked)
    n_e2e = max(20, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        M.spmv_host(hx, hy, sched, repartition=True, chunked=chunked)
    dq = (time.perf_counter() - t0) / n_e2e
    e2e_iter = {"value": round(nnz / dq / 1e9, 3), "unit": "GNZ/s", "h2d_bytes_per_step": 4 * cols,
                "d2h_bytes_per_step": 4 * rows, "steps": n_e2e, "ms_per_step": round(dq * 1e3, 4),
                "api": "lb_spmv_host_x" + ("(REPARTITION | CHUNKED: y rows copied out per tile-range launch while "
                                           "the next range computes)" if chunked else "(REPARTITION)")
                       + " (A resident on the device, created once; per step: pinned H2D of x, the SpMV, D2H of "
                         "y, stream sync; host clock)"}
    # `e2e`: independent right-hand sides streamed through lb_spmv_host_x_async (three staging slots: step
    # k's H2D, step k-1's SpMV and step k-2's D2H overlap), one x and one y buffer per step in pinned
    # host memory, a wait at the end; host clock around all of it.
    nb = 4
    hxs = [hx.clone().pin_memory() for _ in range(nb)]
    hys = [torch.empty(rows).pin_memory() for _ in range(nb)]
    for i in range(nb):
        M.spmv_host_async(hxs[i], hys[i], sched, repartition=True)
    M.spmv_host_wait()
    n_async = max(50, args.e2e_steps)  # a longer stream: the 3-deep pipeline's fill is amortised
    t0 = time.perf_counter()
    for i in range(n_async):
        M.spmv_host_async(hxs[i % nb], hys[i % nb], sched, repartition=True)
    M.spmv_host_wait()
    da = (time.perf_counter() - t0) / n_async
    rec["e2e"] = {"value": round(nnz / da / 1e9, 3), "unit": "GNZ/s", "h2d_bytes_per_step": 4 * cols,
                  "d2h_bytes_per_step": 4 * rows, "steps": n_async, "ms_per_step": round(da * 1e3, 4),
                  "api": "lb_spmv_host_x_async + lb_spmv_host_x_wait (A resident on the device, created once; "
                         "per step: pinned H2D of that step's x, lb_spmv_ex(REPARTITION), D2H of its y; copies "
                         "of neighbouring steps overlap the SpMV; host clock over all steps + the final wait)"}
    rec["e2e_iterative"] = e2e_iter
    h = lb.HostSpmv(rows, cols, nnz, device=dev)
    ho, hc, hv = A.row_offsets.cpu().pin_memory(), A.col_idx.cpu().pin_memory(), A.values.cpu().pin_memory()
    h(ho, hc, hv, hx, hy, sched)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        h(ho, hc, hv, hx, hy, sched)
    dt = (time.perf_counter() - t0) / args.e2e_steps
    rec["e2e_full_upload"] = {"value": round(nnz / dt / 1e9, 3), "unit": "GNZ/s",
                              "h2d_bytes_per_step": 4 * (rows + 1) + 8 * nnz + 4 * cols,
                              "d2h_bytes_per_step": 4 * rows, "api": "lb_spmv_host (pinned host buffers: CSR + x "
                              "uploaded every step, transient handle without a plan)", "steps": args.e2e_steps}
    del h
    torch.cuda.empty_cache()

    # CPU oracle on a bounded sample of the same workload
    import oracle
    sample = cpu_sample(A, x, 32_000_000 if cfg != "c1" else A.nnz)
    gnz, reps, dt = time_oracle(sample, args.cpu_seconds)
    rec["cpu_baseline"] = {"value": round(gnz, 4), "unit": "GNZ/s", "cores": oracle.num_threads(), "kind": "oracle",
                           "sample": f"leading {sample[4]} rows ({sample[5]} nnz) of {cfg} with full x, {reps} reps "
                                     f"in {dt:.1f} s, median rep (oracle.spmv_omp, fp64, gcc -O3 -march=native)"}
    rec["cpu_baseline"].update(oracle_extras(sample, max(2.0, args.cpu_seconds / 2)))
    # the other matrix classes of BASELINE's metric ("per matrix class"), one GPU each
    classes = [c for c in args.classes.split(",") if c and c != cfg]
    if classes:
        del M, A, x, y, hx, hy, hxs, hys, ho, hc, hv
        torch.cuda.empty_cache()
        rec["classes"] = {}
        for c in classes:
            rec["classes"][c] = class_report(c, dev)
    print(json.dumps(rec))


def run_multi(args, cfg):
    import torch.distributed as dist
    import paper_2212_08964_b200 as lb
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    A = lbgen.make_config(cfg, "float", device=dev)
    x = lbgen.x_for_config(cfg, A.cols, "float", device=dev)
    rows, cols, nnz = A.rows, A.cols, A.nnz
    b = lb.shard_bounds(A.row_offsets, world)
    off, col, val = lb.shard_csr(A.row_offsets, A.col_idx, A.values, b, rank)
    del A
    torch.cuda.empty_cache()
    M = lb.CsrMatrix(int(b[rank + 1] - b[rank]), cols, off, col, val, validate=True)
    M.set_items_per_tile(args.items_per_tile)
    comm = lb.Comm.from_process_group(local)
    y = torch.empty(rows, device=dev)
    stream = torch.cuda.current_stream()

    peer = comm.peer_buffer(y) if args.fused else None

    def step():
        if peer is not None:
            comm.spmv_multi_fused(M, b, x, peer, args.schedule, repartition=True)
        else:
            comm.spmv_multi(M, b, x, y, args.schedule, repartition=True, chunked=args.overlap)

    def timed(fn, n):
        dist.barrier()
        torch.cuda.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for _ in range(n):
            fn()
        eb.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([ea.elapsed_time(eb) / n], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt[0])

    # plain-CSR step rate first, then each rank plans its own shard (x-reuse plan)
    no_plan, plan = None, None
    if args.hot_slots >= 0 and args.schedule == "merge_path":
        for _ in range(3):
            step()
        n_np = max(5, min(args.steps, 50))
        ms_np = timed(step, n_np)
        no_plan = {"value": round(nnz / (ms_np * 1e-3) / 1e9, 3), "ms_per_step": round(ms_np, 5), "steps": n_np}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hot_n, hot_nnz = M.plan_hot_x(args.hot_slots)
        torch.cuda.synchronize()
        info = M.plan_info()
        bt = torch.tensor([(time.perf_counter() - t0) * 1e3], device=dev)
        dist.all_reduce(bt, op=dist.ReduceOp.MAX)
        plan = {"kind": "x-reuse plan per shard (lb_csr_plan_hot_x, DESIGN.md 6b)", "slots_requested": args.hot_slots,
                "rank0_hot_cols": hot_n, "rank0_hot_nnz_frac": round(hot_nnz / max(M.nnz, 1), 4),
                "rank0_warm_cols": info["warm_cols"], "rank0_warm_nnz_frac": round(info["warm_nnz"] / max(M.nnz, 1), 4),
                "build_ms_max_over_ranks": round(float(bt[0]), 2), "built": "once per shard, before the timed region"}

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # SURVEY 8(c) p10, asserted once before timing: after the step every rank holds a bitwise-identical
    # y (an NCCL all-reduce of per-rank hashes, lb_comm_check_replicas)
    same, _ = comm.check_replicas(peer.y if peer is not None else y)
    if not same:
        raise RuntimeError("ranks disagree on y after the multi-GPU step (lb_comm_check_replicas)")
    sampler = ClockSampler(local) if (rank == 0 and not args.no_extras) else None
    if sampler:
        sampler.__enter__()
    if not args.no_extras:
        # soak (every rank, same count) so the sampler sees steady-state clocks even if K steps are short
        n_soak = max(1, int(1000.0 / max(ms_np if no_plan else 1.0, 0.05)))
        for _ in range(n_soak):
            step()
        torch.cuda.synchronize()
    n0 = lb.launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    launches = lb.launch_count() - n0
    if sampler:
        sampler.__exit__()
    ms_local = e0.elapsed_time(e1) / args.steps
    # SpMV-only (no exchange) time of this rank's shard
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    f0.record(stream)
    for _ in range(args.steps):
        M.spmv(x, y[int(b[rank]):int(b[rank + 1])], args.schedule)
    f1.record(stream)
    torch.cuda.synchronize()
    spmv_ms_local = f0.elapsed_time(f1) / args.steps
    # exchange only (all-gather(v) of y): its time and bus bandwidth per rank
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    g0.record(stream)
    for _ in range(args.steps):
        comm.allgather_rows(b, y)
    g1.record(stream)
    torch.cuda.synchronize()
    ag_ms_local = g0.elapsed_time(g1) / args.steps
    # e2e through the public API: every step copies this rank's shard (CSR arrays) and x from pinned
    # host memory into the handle's borrowed arrays, runs the same multi-GPU step (exchange included)
    # and reads this rank's rows of y back; CUDA events on the stream, max over ranks
    e2e_ms_local, h2d_local, d2h_local = 0.0, 0, 0
    full_ms_local, full_h2d_local = 0.0, 0
    if not args.no_extras:
        b0, b1 = int(b[rank]), int(b[rank + 1])
        h_x = x.cpu().pin_memory()
        h_y = torch.empty(b1 - b0, pin_memory=True)
        # e2e: the shard (and its plan) stays resident; every step copies x in and this rank's y rows out
        h2d_local = h_x.numel() * 4
        d2h_local = h_y.numel() * 4

        def e2e_step():
            x.copy_(h_x, non_blocking=True)
            step()
            h_y.copy_(y[b0:b1], non_blocking=True)

        e2e_step()
        e2e_ms_local = timed(e2e_step, max(20, args.e2e_steps))
        # e2e_full_upload: the shard CSR is copied in as well, every step
        srcs = [(M.row_offsets, M.row_offsets.cpu().pin_memory()), (M.col_idx, M.col_idx.cpu().pin_memory()),
                (M.values, M.values.cpu().pin_memory()), (x, h_x)]
        full_h2d_local = sum(h.numel() * h.element_size() for _, h in srcs)

        def full_step():
            for d_t, h_t in srcs:
                d_t.copy_(h_t, non_blocking=True)
            step()
            h_y.copy_(y[b0:b1], non_blocking=True)

        full_step()
        full_ms_local = timed(full_step, args.e2e_steps)
    t = torch.tensor([ms_local, spmv_ms_local, e2e_ms_local, float(h2d_local), float(d2h_local), ag_ms_local,
                      full_ms_local, float(full_h2d_local)], dtype=torch.float64, device=dev)
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    ms, spmv_ms, e2e_ms, ag_ms = float(tmax[0]), float(tmax[1]), float(tmax[2]), float(tmax[5])
    h2d_total, d2h_total = int(t[3]), int(t[4])
    full_ms, full_h2d_total = float(tmax[6]), int(t[7])
    if rank == 0:
        rec = {
            "metric": "SpMV GNZ/s", "value": round(nnz / (ms * 1e-3) / 1e9, 3), "unit": "GNZ/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (lbgen, seeded)",
            "config": {"workload": cfg, "desc": lbgen.CONFIG_DESC.get(cfg, cfg), "rows": rows, "nnz": nnz,
                       "schedule": args.schedule, "parallelism": f"row shards x{world} (equal nnz), NCCL all-gather of y",
                       "step": ("lb_spmv_multi_fused(REPARTITION): shard partition + SpMV whose epilogue stores y "
                                "into every rank's buffer over NVLink + barrier") if args.fused else
                               ("lb_spmv_multi_ex(REPARTITION | CHUNKED): shard partition + SpMV as tile-range launches, "
                                "each chunk's rows all-gathered (NCCL broadcast group) while the next computes")
                               if args.overlap else
                               "lb_spmv_multi_ex(REPARTITION): shard partition + SpMV + all-gather(v) of y",
                       "l2": "inputs larger than L2; no flush"},
            "plan": plan,
            "no_plan": no_plan,
            "replicas_bitwise_equal": True,
            "gpu_launches": int(launches),
            "spmv_only": {"value": round(nnz / (spmv_ms * 1e-3) / 1e9, 3), "unit": "GNZ/s", "ms": round(spmv_ms, 5),
                          "per_gpu": round(nnz / world / (spmv_ms * 1e-3) / 1e9, 3)},
            "exchange": {"ms": round(ag_ms, 5), "op": "lb_allgather_rows (NCCL group of ncclBroadcast, root = each rank)",
                         "bytes_received_per_rank_max": int(4 * (rows - min(int(b[k + 1] - b[k]) for k in range(world)))),
                         "bus_GB/s": round(4 * (rows - min(int(b[k + 1] - b[k]) for k in range(world))) / (ag_ms * 1e-3) / 1e9, 1)
                         if ag_ms > 0 else None},
            "e2e": None if args.no_extras else {
                "value": round(nnz / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GNZ/s", "h2d_bytes_per_step": h2d_total,
                "d2h_bytes_per_step": d2h_total, "steps": max(20, args.e2e_steps),
                "api": "per rank (shard resident): pinned H2D of x, the same multi-GPU step, D2H of the rank's y "
                       "rows; CUDA events, max over ranks; bytes summed over ranks"},
            "e2e_full_upload": None if args.no_extras else {
                "value": round(nnz / (full_ms * 1e-3) / 1e9, 3), "unit": "GNZ/s",
                "h2d_bytes_per_step": full_h2d_total, "d2h_bytes_per_step": d2h_total, "steps": args.e2e_steps,
                "api": "per rank: pinned H2D of the shard CSR + x every step, the multi-GPU step, D2H of y rows"},
        }
        # roofline of rank 0's tile kernel on its shard (phase times: CUDA events on the launch stream)
        ph = [M.phase_times(x, y[int(b[0]):int(b[1])], args.schedule) for _ in range(10)]
        main_ms = float(np.mean([p_[1] for p_ in ph]))
        alg = compulsory_bytes(M.rows, cols, M.nnz)
        peak, peak_src = peak_hbm()
        achieved = alg / (main_ms * 1e-3) / 1e9
        rec["roofline"] = {"bound": "hbm", "kernel": M.kernel_name(args.schedule), "achieved": round(achieved, 1),
                           "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                           "algorithmic_bytes": alg, "peak_source": peak_src,
                           "kernel_ms_from": "rank 0 shard: mean of 10 lb_spmv_phase_times calls"}
        if sampler:
            rec["clocks"] = sampler.summary()
        print(json.dumps(rec))
    if peer is not None:
        peer.close()
    comm.close()
    dist.destroy_process_group()


def main():
    args = parse()
    world, rank, _ = dist_env()
    if args.impl == "reference":
        cfg = args.config or ("c3" if world == 1 else "c5")
        run_reference(args, cfg)
        return
    if world > 1 or args.multi:
        run_multi(args, args.config or "c5")
    else:
        run_single(args, args.config or "c3")


if __name__ == "__main__":
    main()
