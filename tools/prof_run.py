"""Run a few sorts of a synthetic input (for ncu / compute-sanitizer runs).

    python tools/prof_run.py --n 26 [--dist uniform_u64] [--reps 2] [--algo tree]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=26)
    ap.add_argument("--dist", default="uniform_u64")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--algo", default="tree")
    ap.add_argument("--base-cap", type=int, default=0)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--max-levels", type=int, default=0)
    ap.add_argument("--alpha-min", type=int, default=0)
    ap.add_argument("--nexact", type=int, default=0, help="element count (overrides --n)")
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2009_13569_b200 as ips
    import synth_inputs as gen

    dt = {"pairs": 2, "records100": 3, "quartets": 5}.get(a.dist, 1 if a.dist.endswith("_f64") else 4 if a.dist.endswith("_u32") else 0)
    host = np.ascontiguousarray(gen.generate(a.dist, a.nexact or (1 << a.n), 42)).view(np.uint8).reshape(-1)
    src = torch.from_numpy(host).cuda()
    work = torch.empty_like(src)
    algo = ips.DIGIT if a.algo == "digit" else ips.TREE
    for r in range(a.reps):
        work.copy_(src)
        st = ips.sort_ex(work, dt, algo=algo, base_cap=a.base_cap, timing=True, max_levels=a.max_levels, alpha_min=a.alpha_min)
        torch.cuda.synchronize()
        print(r, {k: round(v, 3) for k, v in st["kernel_ms"].items() if v}, st["levels"], st["tasks_per_level"])
    if a.check and dt == 0:
        g = work.cpu().numpy().view(np.uint64)
        assert np.all(g[1:] >= g[:-1])
        print("sorted ok")


if __name__ == "__main__":
    main()
