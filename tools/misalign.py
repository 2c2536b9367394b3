import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2009_13569_b200 as ips, synth_inputs as gen
n = 1 << 30
h = gen.uniform_u64(n + 8, 42)
src = torch.from_numpy(h.view(np.int64)).cuda()
w = torch.empty_like(src)
for off in (0, 1, 2, 4):
    for rep in range(3):
        w.copy_(src)
        s = ips.sort_ex(w[off:off + n], 0, timing=True)
    torch.cuda.synchronize()
    print("offset", off, [{k: round(v, 3) for k, v in d.items()} for d in s["round_kernel_ms"]], round(s["kernel_ms"]["total"], 3))
