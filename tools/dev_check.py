"""Development check on the GPU: a few sorts of the chosen element type at
several sizes and distributions (output compared with numpy's sort for
key-only types, with the oracle's parity checker otherwise), then timing of
the 2^30 (or --n) run by kernel family.  Not a test: the GPU tests are.

    python tools/dev_check.py [--dt 0] [--n 30] [--reps 3] [--algo tree] [--dists a,b]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

DISTS = {0: ["uniform_u64", "rootdup_u64", "twodup_u64", "zipf_u64", "eightdup_u64"],
         1: ["uniform_f64", "exponential_f64", "almost_sorted_f64"],
         2: ["pairs"], 3: ["records100"], 4: ["uniform_u32"], 5: ["quartets"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dt", type=int, default=0)
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--algo", default="tree")
    ap.add_argument("--dists", default="")
    ap.add_argument("--no-check", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2009_13569_b200 as ips
    import synth_inputs as gen

    algo = ips.DIGIT if a.algo == "digit" else ips.TREE
    dists = a.dists.split(",") if a.dists else DISTS[a.dt]
    bad = 0
    if not a.no_check:
        import oracle
        for dist in dists:
            for lg, extra in ((12, {}), (17, {}), (20, {}), (22, {"base_cap": 2000}), (24, {})):
                for n in (1 << lg, (1 << lg) + 12345):
                    h = np.ascontiguousarray(gen.generate(dist, n, 11))
                    t = torch.from_numpy(h.view(np.uint8).reshape(-1).copy()).cuda()
                    ips.sort_ex(t, a.dt, algo=algo, **extra)
                    torch.cuda.synchronize()
                    g = t.cpu().numpy().view(h.dtype).reshape(h.shape)
                    if h.ndim == 1:
                        ok = np.array_equal(g, np.sort(h))
                    else:
                        ok = oracle.parity(g, oracle.sort(h, a.dt), a.dt) == -1
                    if not ok:
                        bad += 1
                        print("MISMATCH", dist, n, extra, flush=True)
        print("check:", "ok" if not bad else f"{bad} failures", "status", ips.device_status(), flush=True)
    for dist in dists:
        host = np.ascontiguousarray(gen.generate(dist, 1 << a.n, 42)).view(np.uint8).reshape(-1)
        src = torch.from_numpy(host).cuda()
        work = torch.empty_like(src)
        st = torch.cuda.current_stream()
        ms = []
        for r in range(a.reps + 1):
            work.copy_(src)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ips.sort(work, a.dt, algo=algo)
            e1.record(st)
            torch.cuda.synchronize()
            if r:
                ms.append(e0.elapsed_time(e1))
        work.copy_(src)
        s = ips.sort_ex(work, a.dt, algo=algo, timing=True)
        torch.cuda.synchronize()
        print(f"{dist} 2^{a.n}: {min(ms):.3f} ms (mean {sum(ms)/len(ms):.3f}) levels {s['levels']} {s['tasks_per_level']}",
              {k: round(v, 3) for k, v in s["kernel_ms"].items() if v > 0.02}, flush=True)
        del src, work
        torch.cuda.empty_cache()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
