"""Debug: one sort of n uint64 keys with stats (timing), repeated."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2009_13569_b200 as p
import synth_inputs as gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
algo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
a = torch.from_numpy(gen.uniform_u64(n, 42).view(np.int64)).cuda()
for r in range(reps):
    t = a.clone()
    torch.cuda.synchronize()
    st = p.sort_ex(t, p.U64, timing=True, algo=algo)
    print(st["levels"], st["tasks_per_level"], {k: round(v, 3) for k, v in st["kernel_ms"].items() if v}, flush=True)
