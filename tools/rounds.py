"""Per-round kernel times of one sort (ips4o_stats.round_kernel_ms):
    python tools/rounds.py <dist> <log2 n> [algo] [dtype]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_13569_b200 as ips
import synth_inputs as gen

dist, lg = sys.argv[1], int(sys.argv[2])
algo = ips.DIGIT if len(sys.argv) > 3 and sys.argv[3] == "digit" else ips.TREE
DT = {"pairs": 2, "records100": 3, "quartets": 5}
dt = int(sys.argv[4]) if len(sys.argv) > 4 else DT.get(dist, 1 if dist.endswith("_f64") else 4 if dist.endswith("_u32") else 0)
h = np.ascontiguousarray(gen.generate(dist, 1 << lg, 42)).view(np.uint8).reshape(-1)
src = torch.from_numpy(h).cuda()
w = torch.empty_like(src)
for rep in range(2):
    w.copy_(src)
    s = ips.sort_ex(w, dt, algo=algo, timing=True)
torch.cuda.synchronize()
print(dist, lg, "levels", s["levels"], s["tasks_per_level"], "elems", s["elems_per_level"], "base tasks", s["basecase_tasks"])
for r, d in enumerate(s["round_kernel_ms"]):
    print("  round", r, {k: round(v, 3) for k, v in d.items()})
print("  total", {k: round(v, 3) for k, v in s["kernel_ms"].items() if v > 0.01})
