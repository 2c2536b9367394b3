"""Small sorts of every dtype with both classifiers (n <= 2^16), for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck); each result
is checked against the oracle.  python tools/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2009_13569_b200 as p
import synth_inputs as gen

GEN = {p.U64: lambda n, s: gen.uniform_u64(n, s), p.F64: lambda n, s: gen.exponential_f64(n, s),
       p.PAIR: lambda n, s: gen.pairs(n, s), p.REC100: lambda n, s: gen.records100(n, s),
       p.U32: lambda n, s: gen.uniform_u32(n, s), p.QUARTET: lambda n, s: gen.quartets(n, s)}
bad = 0
for dt, g in GEN.items():
    for n, opts in [(3000, {}), (50_001, {"base_cap": 300}), (65_536, {"algo": p.DIGIT, "base_cap": 500}),
                    (40_000, {"skip_prepass": True, "base_cap": 700})]:
        a = np.ascontiguousarray(g(n, 7))
        t = torch.from_numpy(a.view(np.uint8).reshape(-1).copy()).cuda()
        st = p.sort_ex(t, dt, **opts)
        r = t.cpu().numpy().view(a.dtype).reshape(a.shape)
        ok = oracle.parity(r, oracle.sort(a, dt), dt) == -1
        bad += not ok
        print(f"dtype {dt} n {n} {opts}: levels {st['levels']} ok {ok}", flush=True)
# an easy input (reverse), a graph-free async call, and the device status word
a = gen.reverse_sorted_f64(20_000, 3)
t = torch.from_numpy(a.copy()).cuda()
p.sort(t, p.F64)
torch.cuda.synchronize()
bad += oracle.parity(t.cpu().numpy(), oracle.sort(a, p.F64), p.F64) != -1
print("device status", p.device_status(), "failures", bad)
sys.exit(1 if bad else 0)
