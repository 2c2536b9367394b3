"""Debug driver: run small sorts one per subprocess with a timeout, print stats."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, %r)
import paper_2009_13569_b200 as p, synth_inputs as gen, oracle
n, dt, opts = %d, %d, %s
a = gen.uniform_u64(n, 1) if dt == 0 else gen.pairs(n, 4)
t = torch.from_numpy(a.view(np.int64)).cuda()
t0 = time.time()
st = p.sort_ex(t, dt, **opts)
torch.cuda.synchronize()
g = t.cpu().numpy().view(a.dtype).reshape(a.shape)
ok = oracle.parity(g, oracle.sort(a, dt), dt) == -1
print("n=%%d dt=%%d opts=%%s ok=%%s %%.3fs levels=%%d tasks=%%s launches=%%d scratch=%%d status=%%d" %% (n, dt, opts, ok, time.time()-t0, st["levels"], st["tasks_per_level"], st["kernel_launches"], st["scratch_bytes"], p.device_status()), flush=True)
print({k: round(v, 3) for k, v in st["kernel_ms"].items() if v})
'''
cases = [(1000, 0, {}), (30000, 0, {}), (1 << 16, 0, {}), (1 << 20, 0, {}), (1 << 20, 0, {"skip_prepass": True}),
         (1 << 20, 0, {"algo": 1}), (1 << 22, 0, {}), (1 << 24, 0, {"timing": True}), (1 << 18, 0, {"base_cap": 512}),
         (1 << 20, 2, {}), (1 << 26, 0, {"timing": True})]
if len(sys.argv) > 1:
    cases = cases[: int(sys.argv[1])]
for n, dt, opts in cases:
    try:
        r = subprocess.run([sys.executable, "-c", CASE % (ROOT, n, dt, repr(opts))], capture_output=True, text=True, timeout=60)
        print(r.stdout.strip() or r.stderr[-1500:], flush=True)
    except subprocess.TimeoutExpired as e:
        print("TIMEOUT", n, dt, opts, (e.stdout or b"")[-500:], flush=True)
