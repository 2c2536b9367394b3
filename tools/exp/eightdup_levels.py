"""Diagnostic: bucket sizes / key ranges of EightDup's first two partitioning
steps (ips4o_partition_step on the whole array, then on a few level-1 buckets)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2009_13569_b200 as p
import synth_inputs as gen
dist = sys.argv[1] if len(sys.argv) > 1 else "eightdup_u64"
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 30
a = torch.from_numpy(gen.generate(dist, 1 << lg, 42).view(np.int64)).cuda()
info = p.partition_step(a, p.U64)
E = np.array(info["E"], dtype=np.int64)
print({k: v for k, v in info.items() if k not in ("E", "tree", "splitter")})
def desc(t, E, tag):
    sz = np.diff(E)
    h = t.cpu().numpy().view(np.uint64)
    rng = []
    for j in range(len(sz)):
        if sz[j] > 0:
            seg = h[E[j]:E[j + 1]]
            rng.append(int(seg.max()) - int(seg.min()))
        else:
            rng.append(0)
    rng = np.array(rng)
    print(tag, "buckets", len(sz), "nonempty", int((sz > 0).sum()), "size pct", np.percentile(sz, [0, 10, 50, 90, 100]).astype(int).tolist(),
          "range pct", np.percentile(rng, [0, 10, 50, 90, 100]).astype(int).tolist(),
          "n>65535", int((sz > 65535).sum()), "n>32768", int((sz > 32768).sum()), "single-key", int(((rng == 0) & (sz > 0)).sum()))
    return sz, rng
sz, rng = desc(a, E, "L1")
order = np.argsort(-sz)
for j in list(order[:3]) + list(order[len(order) // 2:len(order) // 2 + 2]):
    if rng[j] == 0 or sz[j] < 100000:
        continue
    sub = a[E[j]:E[j + 1]].clone()
    inf2 = p.partition_step(sub, p.U64)
    print(" L2 of bucket", j, "size", sz[j], "range", rng[j], {k: v for k, v in inf2.items() if k not in ("E", "tree", "splitter")})
    desc(sub, np.array(inf2["E"], dtype=np.int64), "  L2")
