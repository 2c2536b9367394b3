"""A/B: time ips4o_sort (no stats) of uniform u64 keys with a given libips4o.so.
usage: python tools/ab_lib.py LIB n [reps]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth_inputs as gen

lib = ctypes.CDLL(sys.argv[1])
lib.ips4o_sort.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
n = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
src = torch.from_numpy(gen.uniform_u64(n, 42).view(np.int64)).cuda()
work = torch.empty_like(src)
st = torch.cuda.current_stream()
ts = []
for r in range(reps + 3):
    work.copy_(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    rc = lib.ips4o_sort(work.data_ptr(), n, 0, st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    assert rc == 0, rc
    if r >= 3:
        ts.append(e0.elapsed_time(e1))
w = work.cpu().numpy().view(np.uint64)
assert np.all(w[1:] >= w[:-1])
print(f"{sys.argv[1].split('/')[-1]:>22s} n=2^{n.bit_length()-1}: mean {np.mean(ts):.3f} ms  min {np.min(ts):.3f}  -> {n/np.mean(ts)/1e6:.2f} Gkeys/s", flush=True)
