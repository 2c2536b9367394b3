#!/usr/bin/env python
"""Benchmark: Gkeys/s of the in-place IPS4o sort of 2^30 uint64 Uniform keys
on B200 (BASELINE.json metric), plus the HBM roofline of the dominant kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--n LOG2N] [--dist uniform_u64] [--algo tree|digit]

One step = one full ips4o_sort of the whole array (all SURVEY 8(a) rows:
pre-pass, sampling, classification, boundaries, stripe fix, permutation,
cleanup, scheduling, base case; the levels are planned and launched by the
device) on inputs already resident in HBM.  Before every step (outside the
timed region) the working array is restored from a pristine device copy; the
8 GiB input is far larger than the 126 MB L2, so no extra L2 flush is needed.
Timing: CUDA events on the sorting stream around the asynchronous ips4o_sort,
bracketed by barrier + synchronize; max over ranks.  The per-kernel times
(roofline) come from separate untimed steps with device timing stamps
(ips4o_stats, opt.timing).  N > 1 runs independent replicas (DESIGN
"Multi-GPU: replicas only"), weak scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DTYPES = {"u64": 0, "f64": 1, "pair": 2, "rec100": 3}
ELEM = {0: 8, 1: 8, 2: 16, 3: 100}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=30, help="log2 of the element count")
    ap.add_argument("--dist", default="uniform_u64")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--algo", default="tree", choices=["tree", "digit"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-log2", type=int, default=25, help="oracle sample size (log2)")
    ap.add_argument("--stat-steps", type=int, default=3, help="untimed steps with per-kernel device timing")
    ap.add_argument("--no-c1", action="store_true", help="skip the c1 (2^20) hot/cold-L2 extra")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        time.sleep(0.05)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- helpers
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


NOMINAL_HBM_GBS = 8000.0  # BASELINE.json's "~8 TB/s" contract


def ncu_traffic():
    """DRAM bytes per step of each kernel family from the committed ncu launch
    list of the same workload (profiles/r2_ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "r2_ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


def make_input(dist: str, n: int, seed: int):
    import numpy as np

    import synth_inputs as gen

    a = gen.generate(dist, n, seed)
    return np.ascontiguousarray(a)


def cpu_baseline(dist: str, log2n: int, seed: int) -> dict:
    """The oracle as it stands (single-threaded C mergesort) on a bounded
    sample of the same workload: the first 2^log2n keys of the same stream."""
    import oracle

    n = 1 << log2n
    a = make_input(dist, n, seed)
    dt = {"f64": 1, "pair": 2, "rec100": 3}.get(dist.split("_")[-1], 0)
    if dist == "pairs":
        dt = 2
    if dist == "records100":
        dt = 3
    oracle.build()
    t0 = time.perf_counter()
    oracle.sort_inplace(a, dt)
    t = time.perf_counter() - t0
    full = 1 << 30
    return {"value": n / t / 1e9, "unit": "Gkeys/s", "cores": 1, "kind": "oracle",
            "sample": f"first 2^{log2n} keys of the {dist} stream (seed {seed}), "
                      f"single-threaded top-down mergesort, {t:.2f} s",
            # a mergesort's time grows as n log n: the rate at 2^30 estimated
            # from the sample (the sample itself is what was measured)
            "value_at_2p30_nlogn_estimate": n / t / 1e9 * log2n / 30.0,
            "host_cpu": _cpu_model(), "nproc": os.cpu_count(), "threads_used": 1, "full_n": full}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank float over all ranks (the contract's max-over-ranks
    timing); identity without torch.distributed.  NCCL needs a device tensor,
    gloo a CPU one."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=device if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(n_per_rank: int, world: int, steps: int, max_total_ms: float) -> float:
    """Whole-job Gkeys/s: every rank sorts its own n keys per step (replicas,
    weak scaling); time = max over ranks."""
    return world * n_per_rank * steps / (max_total_ms / 1e3) / 1e9


def c1_hot_cold(ips, dev, stream, reps: int = 10) -> dict:
    """BASELINE config 1 (2^20 uint64 Uniform, seed 1; 8 MiB, L2-resident):
    device time per sort with the input hot in L2 (sorted back to back) and
    cold (L2 flushed by writing a 512 MiB buffer before every rep)."""
    import numpy as np
    import torch

    import synth_inputs as gen

    n = 1 << 20
    src = torch.from_numpy(gen.uniform_u64(n, 1).view(np.int64)).to(dev)
    work = torch.empty_like(src)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for mode in ("hot", "cold"):
        ts = []
        for r in range(reps + 2):
            work.copy_(src)
            if mode == "cold":
                flush.fill_(r & 0xFF)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ips.sort(work, 0)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        out[mode] = {"ms": statistics.mean(ts), "min_ms": min(ts), "Gkeys_s": n / (statistics.mean(ts) / 1e3) / 1e9}
    out["workload"] = "c1: 2^20 uint64 Uniform (seed 1), 8 MiB"
    del flush
    return out


def dist_dtype(dist: str) -> int:
    return {"pairs": 2, "records100": 3}.get(dist, 1 if dist.endswith("_f64") else 0)


# ----------------------------------------------------------------- reference arm
def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    import numpy as np

    import oracle

    oracle.build()
    dt = dist_dtype(args.dist)
    log2 = min(args.cpu_log2 - 2, args.n)   # per step: a bounded sample
    n = 1 << log2
    a = make_input(args.dist, n, args.seed)
    times = []
    for i in range(args.warmup + args.steps):
        b = a.copy()
        t0 = time.perf_counter()
        oracle.sort_inplace(b, dt)
        t = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(t)
    tot = sum(times)
    val = n * len(times) / tot / 1e9
    line = {
        "impl": "reference", "metric": "Gkeys/s sorted in place, 2^30 uint64 Uniform; HBM GB/s per partition pass",
        "value": val, "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64" if dt == 0 else ["u64", "f64", "pair", "rec100"][dt],
        "data": "synthetic",
        "config": {"workload": f"{args.dist} n=2^{args.n} (reference arm: oracle on a 2^{log2} sample per step)",
                   "n": 1 << args.n, "seed": args.seed},
        "cpu_baseline": {"value": val, "unit": "Gkeys/s", "cores": 1, "kind": "oracle",
                         "sample": f"first 2^{log2} keys of the {args.dist} stream per step",
                         "host_cpu": _cpu_model()},
        "e2e": {"value": val, "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def run_ours(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch

    import paper_2009_13569_b200 as ips
    from paper_2009_13569_b200 import build

    build.build()
    ips.load()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dt = dist_dtype(args.dist)
    D = ELEM[dt]
    n = 1 << args.n
    algo = ips.DIGIT if args.algo == "digit" else ips.TREE
    host = make_input(args.dist, n, args.seed + rank)
    hbytes = np.ascontiguousarray(host).view(np.uint8).reshape(-1)
    pristine = torch.empty(n * D, dtype=torch.uint8, device=dev)
    pristine.copy_(torch.from_numpy(hbytes))
    work = torch.empty_like(pristine)
    stream = torch.cuda.current_stream(dev)

    def one_step(stats: bool):
        work.copy_(pristine)
        torch.cuda.synchronize(dev)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        if stats:  # synchronises inside (reads the device control block back)
            st = ips.sort_ex(work, dt, algo=algo, timing=True)
        else:      # the asynchronous product call: one stream-ordered enqueue
            st = ips.sort(work, dt, algo=algo)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        return ev0.elapsed_time(ev1), st

    for _ in range(args.warmup):
        one_step(False)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local_rank)
    clk.start()
    times = []
    for _ in range(args.steps):
        t, _ = one_step(False)
        times.append(t)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    total_ms = max_over_ranks(sum(times), dev)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    # per-kernel device times (globaltimer stamps) from separate untimed steps
    stats = [one_step(True)[1] for _ in range(args.stat_steps)]
    # correctness guard on the last result (cheap, on device): non-decreasing
    chk_ok = None
    if dt == 0:
        w = work.view(torch.int64)
        # unsigned compare via xor of the sign bit
        s = w ^ torch.tensor(-(2**63), dtype=torch.int64, device=dev)
        chk_ok = bool((s[1:] >= s[:-1]).all().item())
    if rank != 0:
        return
    value = aggregate_value(n, world, args.steps, total_ms)
    st = stats[-1]
    km = {k: statistics.mean(s["kernel_ms"][k] for s in stats) for k in stats[0]["kernel_ms"]}
    # roofline of the dominant kernel family
    elems_levels = sum(st["elems_per_level"])
    alg = {
        "classify": 2 * D * elems_levels,
        "permute": 2 * D * elems_levels,
        "basecase": 2 * D * st["basecase_elems"],
        "prepass": D * n,
    }
    fams = {k: km[k] for k in alg if km.get(k, 0) > 0}
    dom = max(fams, key=fams.get) if fams else "classify"
    peak, peak_src = peaks()
    achieved = alg[dom] / (km[dom] / 1e3) / 1e9 if km.get(dom) else None
    traffic = ncu_traffic()
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak if achieved else None,
            "frac_of_nominal_8000": achieved / NOMINAL_HBM_GBS if achieved else None,
            "traffic": (traffic or {}).get(dom), "traffic_unit": "DRAM bytes per step (ncu, profiles/r2_ncu_traffic.json)",
            "peak_source": peak_src,
            "alg_bytes_per_step": alg[dom], "kernel_ms_per_step": km[dom],
            "timing": "device globaltimer stamps per kernel (earliest CTA start to latest warp end), "
                      f"mean of {len(stats)} untimed steps"}
    # per level and per pass: algorithmic GB/s of the partition passes
    levels = []
    for r, rk in enumerate(st.get("round_kernel_ms", [])):
        ne = st["elems_per_level"][r]
        row = {"level": r + 1, "tasks": st["tasks_per_level"][r], "elems": ne}
        for k in ("classify", "permute"):
            ms = statistics.mean(s["round_kernel_ms"][r][k] for s in stats)
            gbs = 2 * D * ne / (ms / 1e3) / 1e9 if ms else None
            row[k] = {"ms": ms, "alg_GBps": gbs, "frac": gbs / peak if gbs else None,
                      "frac_of_nominal_8000": gbs / NOMINAL_HBM_GBS if gbs else None}
        levels.append(row)
    bms = km.get("basecase", 0)
    base_row = {"ms": bms, "alg_GBps": alg["basecase"] / (bms / 1e3) / 1e9 if bms else None}
    if base_row["alg_GBps"]:
        base_row["frac"] = base_row["alg_GBps"] / peak
        base_row["frac_of_nominal_8000"] = base_row["alg_GBps"] / NOMINAL_HBM_GBS
    # algorithmic whole-sort reading: 2 n D per partition level (+ base case)
    L_eff = elems_levels / n
    sort_ms = total_ms / args.steps
    roof_sort = {"levels_eff": L_eff,
                 "frac_partition_2nDL": (2 * n * D * L_eff / (peak * 1e9)) / (
                     (km["classify"] + km["permute"] + km["stripe_fix"] + km["cleanup"] + km["sample"]
                      + km["boundaries"] + km["schedule"]) / 1e3) if L_eff else None,
                 "frac_sort_2nD_L_plus_1": (2 * n * D * (L_eff + 1) / (peak * 1e9)) / (sort_ms / 1e3),
                 "frac_sort_2nD_L_plus_1_of_nominal_8000": (2 * n * D * (L_eff + 1) / (NOMINAL_HBM_GBS * 1e9)) / (sort_ms / 1e3),
                 "per_level": levels, "basecase": base_row}
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        pin = torch.empty(n * D, dtype=torch.uint8).pin_memory()
        src = torch.from_numpy(hbytes)
        et = []
        for i in range(args.e2e_steps + 1):
            pin.copy_(src)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            ips.sort_host(pin, dt, algo=algo)
            t1 = time.perf_counter()
            if i > 0:
                et.append(t1 - t0)
        e2e = {"value": n * len(et) / sum(et) / 1e9, "unit": "Gkeys/s",
               "h2d_bytes_per_step": n * D, "d2h_bytes_per_step": n * D,
               "path": "ips4o_sort_host (pinned host buffer; H2D + sort + D2H inside the call)"}
    c1 = None
    if not args.no_c1 and dt == 0 and args.n >= 20:
        c1 = c1_hot_cold(ips, dev, stream)
    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline(args.dist, min(args.cpu_log2, args.n), args.seed)
    line = {
        "metric": "Gkeys/s sorted in place, 2^30 uint64 Uniform; HBM GB/s per partition pass",
        "value": value, "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": ["u64", "f64", "pair", "rec100"][dt], "data": "synthetic",
        "config": {"workload": f"{args.dist} n=2^{args.n} ({'IPS4o tree' if algo == 0 else 'IPS2Ra digit'})",
                   "n_per_gpu": n, "seed": args.seed, "algo": args.algo,
                   "l2": "inputs (8 GiB) larger than L2; working array restored from a pristine copy "
                         "before each step, outside the timed region",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
        "roofline": roof, "roofline_sort": roof_sort,
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
        # kernels launched per sort (round 0 by the host, later rounds by the
        # device planner; counted by the library) x timed steps
        "gpu_launches": int(st["kernel_launches"]) * args.steps,
        "gpu_launches_per_step": int(st["kernel_launches"]),
        "kernel_ms_per_step": km, "levels": st["levels"], "tasks_per_level": st["tasks_per_level"],
        "basecase_tasks": st["basecase_tasks"], "scratch_bytes": st["scratch_bytes"],
        "sorted_check": chk_ok, "step_ms": times, "c1_l2": c1,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
