"""Time every BASELINE.json config (and the NEXT-2 inputs) on one GPU: one
JSON line per input with ms, Gkeys/s, levels and per-kernel ms.

    python tools/bench_configs.py [--reps 3] [--algo tree|digit] [--only c3]

Same timing rules as bench.py (CUDA events on the sorting stream around one
ips4o_sort, input restored from a pristine device copy outside the timed
region, warm-up discarded); correctness is the GPU tests' job.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

INPUTS = [  # (config, distribution, log2 n, seed)
    ("c1", "uniform_u64", 20, 1),
    ("c2", "uniform_f64", 28, 2), ("c2", "exponential_f64", 28, 2), ("c2", "almost_sorted_f64", 28, 2),
    ("c2", "sorted_f64", 28, 2), ("c2", "reverse_sorted_f64", 28, 2),
    ("c3", "rootdup_u64", 30, 3), ("c3", "twodup_u64", 30, 3), ("c3", "zipf_u64", 30, 3), ("c3", "ones_u64", 30, 3),
    ("c4", "pairs", 28, 4),
    ("c5", "records100", 24, 5),
    ("head", "uniform_u64", 30, 42),
    ("next2", "uniform_u32", 30, 6), ("next2", "eightdup_u64", 30, 3), ("next2", "zero_u64", 30, 3),
    ("next2", "quartets", 26, 7),
]
DT = {"pairs": 2, "records100": 3, "quartets": 5}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--algo", default="tree")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2009_13569_b200 as ips
    import synth_inputs as gen

    ips.load()
    algo = ips.DIGIT if a.algo == "digit" else ips.TREE
    st = torch.cuda.current_stream()
    for cfg, dist, lg, seed in INPUTS:
        if a.only and a.only not in (cfg, dist):
            continue
        dt = DT.get(dist, 1 if dist.endswith("_f64") else 4 if dist.endswith("_u32") else 0)
        n = 1 << lg
        host = np.ascontiguousarray(gen.generate(dist, n, seed)).view(np.uint8).reshape(-1)
        src = torch.from_numpy(host).cuda()
        del host
        work = torch.empty_like(src)
        times, last = [], None
        for r in range(a.reps + 1):
            work.copy_(src)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s = ips.sort_ex(work, dt, algo=algo, timing=True)
            e1.record(st)
            torch.cuda.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
                last = s
        ms = statistics.mean(times)
        print(json.dumps({"config": cfg, "dist": dist, "n": n, "algo": a.algo, "ms": round(ms, 3),
                          "gkeys_s": round(n / ms / 1e6, 2), "levels": last["levels"],
                          "tasks_per_level": last["tasks_per_level"], "easy_input": last["easy_input"],
                          "kernel_ms": {k: round(v, 3) for k, v in last["kernel_ms"].items() if v}}), flush=True)
        del src, work
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
