"""B200-native in-place samplesort partitioning step (IPS4o / IPS2Ra,
arXiv 2009.13569) -- thin Python binding of the C ABI in include/ips4o.h.

Only argument marshalling happens here: every step of the sort runs in the
CUDA kernels of ``csrc/`` (libips4o.so, sm_100a).  There is no CPU fallback:
if the shared library is missing or no B200 is present, the calls raise.
PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "U64", "F64", "PAIR", "REC100", "U32", "QUARTET", "TREE", "DIGIT",
    "load", "sort", "sort_ex", "sort_host", "partition_step", "classify",
    "scratch_bytes", "dtype_info", "device_status", "release_memory", "Options", "Stats", "IPS4OError",
]

U64, F64, PAIR, REC100, U32, QUARTET = 0, 1, 2, 3, 4, 5
TREE, DIGIT = 0, 1
ELEM_BYTES = {U64: 8, F64: 8, PAIR: 16, REC100: 100, U32: 4, QUARTET: 32}
KERNEL_NAMES = ["prepass", "sample", "classify", "boundaries", "stripe_fix", "permute",
                "cleanup", "schedule", "basecase", "reverse", "plan", "total"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libips4o.so")
MAX_LEVELS_REPORTED = 16


class IPS4OError(RuntimeError):
    pass


class Options(ctypes.Structure):
    _fields_ = [
        ("algo", ctypes.c_int32), ("k_max", ctypes.c_int32), ("seed", ctypes.c_uint64),
        ("alpha_min", ctypes.c_int32), ("base_cap", ctypes.c_int32), ("max_levels", ctypes.c_int32),
        ("skip_prepass", ctypes.c_int32), ("skip_basecase", ctypes.c_int32), ("timing", ctypes.c_int32),
        ("arena_mb", ctypes.c_int32), ("reserved", ctypes.c_int32 * 6),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("scratch_bytes", ctypes.c_uint64), ("levels", ctypes.c_int32), ("easy_input", ctypes.c_int32),
        ("tasks_per_level", ctypes.c_uint64 * MAX_LEVELS_REPORTED),
        ("elems_per_level", ctypes.c_uint64 * MAX_LEVELS_REPORTED),
        ("basecase_tasks", ctypes.c_uint64), ("basecase_elems", ctypes.c_uint64),
        ("equal_elems", ctypes.c_uint64), ("kernel_ms", ctypes.c_float * 12),
        ("kernel_launches", ctypes.c_uint64), ("deferred_tasks", ctypes.c_uint64),
        ("round_kernel_ms", (ctypes.c_float * 4) * MAX_LEVELS_REPORTED),
    ]

    def as_dict(self) -> dict:
        lv = self.levels
        return {
            "scratch_bytes": int(self.scratch_bytes), "levels": int(lv),
            "easy_input": int(self.easy_input),
            "tasks_per_level": [int(x) for x in self.tasks_per_level[:lv]],
            "elems_per_level": [int(x) for x in self.elems_per_level[:lv]],
            "basecase_tasks": int(self.basecase_tasks), "basecase_elems": int(self.basecase_elems),
            "equal_elems": int(self.equal_elems),
            "kernel_ms": {k: float(v) for k, v in zip(KERNEL_NAMES, self.kernel_ms)},
            "kernel_launches": int(self.kernel_launches),
            "deferred_tasks": int(self.deferred_tasks),
            "round_kernel_ms": [dict(zip(("classify", "permute", "basecase", "other"),
                                         (float(x) for x in self.round_kernel_ms[r]))) for r in range(min(lv, MAX_LEVELS_REPORTED))],
        }


class DtypeInfo(ctypes.Structure):
    _fields_ = [("elem_bytes", ctypes.c_int32), ("block_elems", ctypes.c_int32),
                ("kidx_max", ctypes.c_int32), ("base_cap", ctypes.c_int32), ("key_bytes", ctypes.c_int32)]


class StepInfo(ctypes.Structure):
    _fields_ = [
        ("algo", ctypes.c_int32), ("num_buckets", ctypes.c_int32), ("l", ctypes.c_int32),
        ("equality", ctypes.c_int32), ("shift", ctypes.c_int32), ("k_req", ctypes.c_int32),
        ("k_used", ctypes.c_int32),
        ("samples", ctypes.c_int32), ("kidx_budget", ctypes.c_int32), ("level", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("E", ctypes.POINTER(ctypes.c_uint64)), ("tree", ctypes.c_void_p), ("splitter", ctypes.c_void_p),
        ("lut_log", ctypes.c_int32), ("reserved0", ctypes.c_int32),
    ]


EXPORTS = ["ips4o_sort", "ips4o_sort_ex", "ips4o_sort_host", "ips4o_scratch_bytes",
           "ips4o_status_string", "ips4o_get_dtype_info", "ips4o_partition_step", "ips4o_classify",
           "ips4o_device_status", "ips4o_release_memory", "ips4o_sample", "ips4o_select_splitters",
           "ips4o_partition_splitters"]

_lib = None


def load(path: str = LIB_PATH):
    """Load libips4o.so (raises if it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise IPS4OError(f"{path} not built; run python -m paper_2009_13569_b200.build")
    L = ctypes.CDLL(path)
    vp, u64, ci = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
    L.ips4o_sort.argtypes = [vp, u64, ci, vp]
    L.ips4o_sort.restype = ci
    L.ips4o_sort_ex.argtypes = [vp, u64, ci, vp, ctypes.POINTER(Options), ctypes.POINTER(Stats)]
    L.ips4o_sort_ex.restype = ci
    L.ips4o_sort_host.argtypes = [vp, u64, ci, ctypes.POINTER(Options), ctypes.POINTER(Stats)]
    L.ips4o_sort_host.restype = ci
    L.ips4o_scratch_bytes.argtypes = [u64, ci, ctypes.POINTER(Options)]
    L.ips4o_scratch_bytes.restype = u64
    L.ips4o_status_string.argtypes = [ci]
    L.ips4o_status_string.restype = ctypes.c_char_p
    L.ips4o_get_dtype_info.argtypes = [ci, ctypes.POINTER(DtypeInfo)]
    L.ips4o_get_dtype_info.restype = ci
    L.ips4o_partition_step.argtypes = [vp, u64, ci, vp, ctypes.POINTER(Options), ctypes.POINTER(StepInfo)]
    L.ips4o_partition_step.restype = ci
    L.ips4o_classify.argtypes = [vp, u64, ci, vp, ci, ci, vp, vp]
    L.ips4o_classify.restype = ci
    L.ips4o_device_status.argtypes = [ci, ctypes.POINTER(ctypes.c_uint32), ci]
    L.ips4o_device_status.restype = ci
    L.ips4o_release_memory.argtypes = [ci]
    L.ips4o_release_memory.restype = ci
    L.ips4o_sample.argtypes = [vp, u64, ci, vp, u64, u64, vp]
    L.ips4o_sample.restype = ci
    L.ips4o_select_splitters.argtypes = [vp, u64, ci, vp, ci, vp]
    L.ips4o_select_splitters.restype = ci
    L.ips4o_partition_splitters.argtypes = [vp, u64, ci, vp, vp, ci, ctypes.POINTER(ctypes.c_uint64)]
    L.ips4o_partition_splitters.restype = ci
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        msg = load().ips4o_status_string(rc).decode()
        raise IPS4OError(f"ips4o error {rc}: {msg}")


def _options(algo=TREE, k_max=0, seed=0, alpha_min=0, base_cap=0, max_levels=0,
             skip_prepass=False, skip_basecase=False, timing=False, arena_mb=0) -> Options:
    o = Options()
    o.arena_mb = arena_mb
    o.algo, o.k_max, o.seed, o.alpha_min = algo, k_max, seed, alpha_min
    o.base_cap, o.max_levels = base_cap, max_levels
    o.skip_prepass, o.skip_basecase, o.timing = int(skip_prepass), int(skip_basecase), int(timing)
    return o


def _tensor_args(t, dtype: int):
    """(ptr, n, stream) of a contiguous CUDA tensor holding n elements."""
    import torch

    if not t.is_cuda:
        raise IPS4OError("expected a CUDA tensor (use sort_host for host memory)")
    if not t.is_contiguous():
        raise IPS4OError("expected a contiguous tensor")
    nbytes = t.numel() * t.element_size()
    D = ELEM_BYTES[dtype]
    if nbytes % D:
        raise IPS4OError(f"tensor of {nbytes} bytes is not a whole number of {D}-byte elements")
    stream = torch.cuda.current_stream(t.device).cuda_stream
    return t.data_ptr(), nbytes // D, stream


def sort(t, dtype: int, **opts):
    """Sort the elements of CUDA tensor ``t`` in place (stream-ordered)."""
    ptr, n, stream = _tensor_args(t, dtype)
    if opts:
        o = _options(**opts)
        _check(load().ips4o_sort_ex(ptr, n, dtype, stream, ctypes.byref(o), None))
    else:
        _check(load().ips4o_sort(ptr, n, dtype, stream))
    return t


def sort_ex(t, dtype: int, **opts) -> dict:
    """Sort in place and return the statistics (synchronises the stream)."""
    ptr, n, stream = _tensor_args(t, dtype)
    o = _options(**opts)
    s = Stats()
    _check(load().ips4o_sort_ex(ptr, n, dtype, stream, ctypes.byref(o), ctypes.byref(s)))
    return s.as_dict()


def sort_ptr(ptr: int, n: int, dtype: int, stream: int = 0, **opts) -> None:
    o = _options(**opts)
    _check(load().ips4o_sort_ex(ptr, n, dtype, stream, ctypes.byref(o), None))


def sort_host(a, dtype: int, **opts) -> dict:
    """End-to-end sort of a HOST buffer (numpy array or CPU tensor) in place:
    H2D copy, device sort, D2H copy inside the call."""
    if hasattr(a, "data_ptr"):
        ptr, nbytes = a.data_ptr(), a.numel() * a.element_size()
    else:
        ptr, nbytes = a.ctypes.data, a.nbytes
    D = ELEM_BYTES[dtype]
    o = _options(**opts)
    s = Stats()
    _check(load().ips4o_sort_host(ptr, nbytes // D, dtype, ctypes.byref(o), ctypes.byref(s)))
    return s.as_dict()


def device_status(device: int = 0, clear: bool = False) -> int:
    """Error flags the device code raised on ``device`` (0 = none); read after
    synchronising the streams that ran sorts."""
    f = ctypes.c_uint32(0)
    _check(load().ips4o_device_status(device, ctypes.byref(f), int(clear)))
    return int(f.value)


def release_memory(device: int = 0) -> None:
    _check(load().ips4o_release_memory(device))


def scratch_bytes(n: int, dtype: int, **opts) -> int:
    o = _options(**opts)
    return int(load().ips4o_scratch_bytes(n, dtype, ctypes.byref(o)))


def dtype_info(dtype: int) -> dict:
    d = DtypeInfo()
    _check(load().ips4o_get_dtype_info(dtype, ctypes.byref(d)))
    return {k: getattr(d, k) for k, _ in DtypeInfo._fields_}


def partition_step(t, dtype: int, **opts) -> dict:
    """Run ONE partitioning step over the whole tensor (test hook).  Returns
    the bucket boundaries E and the classifier (raw key form)."""
    import numpy as np

    ptr, n, stream = _tensor_args(t, dtype)
    info_d = dtype_info(dtype)
    kb, kmax = info_d["key_bytes"], info_d["kidx_max"]
    E = (ctypes.c_uint64 * (2 * kmax + 2))()
    tree = (ctypes.c_uint8 * (kmax * kb))()
    spl = (ctypes.c_uint8 * (kmax * kb))()
    info = StepInfo()
    info.E = ctypes.cast(E, ctypes.POINTER(ctypes.c_uint64))
    info.tree = ctypes.cast(tree, ctypes.c_void_p)
    info.splitter = ctypes.cast(spl, ctypes.c_void_p)
    o = _options(**opts)
    _check(load().ips4o_partition_step(ptr, n, dtype, stream, ctypes.byref(o), ctypes.byref(info)))
    K, l = info.num_buckets, info.l
    leaves = 1 << l
    return {
        "algo": info.algo, "num_buckets": K, "l": l, "equality": bool(info.equality),
        "shift": info.shift, "k_req": info.k_req, "k_used": info.k_used, "samples": info.samples, "seed": int(info.seed),
        "kidx_budget": info.kidx_budget,
        "E": np.array(E[: K + 1], dtype=np.uint64),
        "tree": np.frombuffer(bytes(tree), dtype=np.uint8)[: leaves * kb].copy(),
        "splitter": np.frombuffer(bytes(spl), dtype=np.uint8)[: leaves * kb].copy(),
        "key_bytes": kb, "lut_log": info.lut_log,
    }


def classify(elems, dtype: int, splitters_raw: bytes, u: int, equality: bool, out):
    """Device classification of CUDA tensor ``elems`` with the tree built from
    u sorted unique raw splitter keys; bucket ids into CUDA int32 tensor ``out``."""
    ptr, n, stream = _tensor_args(elems, dtype)
    buf = ctypes.create_string_buffer(bytes(splitters_raw), len(splitters_raw))
    _check(load().ips4o_classify(ptr, n, dtype, ctypes.cast(buf, ctypes.c_void_p), u, int(equality),
                                 out.data_ptr(), stream))
    return out


# ---------------------------------------------------------------- distributed samplesort steps
def sample(t, dtype: int, m: int, seed: int, out) -> None:
    """ips4o_sample: m samples (DESIGN R8 draw, `seed`) of CUDA tensor t into
    CUDA tensor out (m elements), stream-ordered."""
    ptr, n, stream = _tensor_args(t, dtype)
    optr, on, _ = _tensor_args(out, dtype)
    if on < m:
        raise IPS4OError("out holds fewer than m elements")
    _check(load().ips4o_sample(ptr, n, dtype, stream, m, seed, optr))


def select_splitters(samples, dtype: int, parts: int, out) -> None:
    """ips4o_select_splitters: sort CUDA tensor `samples` in place and write the
    parts-1 equidistant picks into CUDA tensor out, stream-ordered."""
    ptr, n, stream = _tensor_args(samples, dtype)
    optr, on, _ = _tensor_args(out, dtype)
    if on < parts - 1:
        raise IPS4OError("out holds fewer than parts - 1 elements")
    _check(load().ips4o_select_splitters(ptr, n, dtype, stream, parts, optr))


def partition_splitters(t, dtype: int, splitters, nspl: int) -> list:
    """ips4o_partition_splitters: partition CUDA tensor t in place into nspl+1
    ranges by the nspl sorted splitters (CUDA tensor); returns the nspl+2
    range bounds (synchronous)."""
    ptr, n, stream = _tensor_args(t, dtype)
    sptr, sn, _ = _tensor_args(splitters, dtype)
    if sn < nspl:
        raise IPS4OError("splitters holds fewer than nspl elements")
    b = (ctypes.c_uint64 * (nspl + 2))()
    _check(load().ips4o_partition_splitters(ptr, n, dtype, stream, sptr, nspl, b))
    return [int(x) for x in b]

