"""Per-kernel-family times (stats, timing=True) of one lib: python tools/ab_stats.py LIB n"""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2009_13569_b200 as p
import synth_inputs as gen
import ctypes
L = ctypes.CDLL(sys.argv[1])
L.ips4o_sort_ex.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                            ctypes.POINTER(p.Options), ctypes.POINTER(p.Stats)]
n = int(sys.argv[2])
src = torch.from_numpy(gen.uniform_u64(n, 42).view(np.int64)).cuda()
acc = None
for r in range(6):
    t = src.clone()
    torch.cuda.synchronize()
    o = p.Options()
    o.timing = 1
    s = p.Stats()
    assert L.ips4o_sort_ex(t.data_ptr(), n, 0, torch.cuda.current_stream().cuda_stream, ctypes.byref(o), ctypes.byref(s)) == 0
    st = s.as_dict()
    if r >= 2:
        km = np.array([st["kernel_ms"][k] for k in p.KERNEL_NAMES])
        acc = km if acc is None else acc + km
acc /= 4
print(sys.argv[1].split("/")[-2], {k: round(float(v), 3) for k, v in zip(p.KERNEL_NAMES, acc) if v})
