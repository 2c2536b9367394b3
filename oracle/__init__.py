"""CPU oracle for the IPS4o / IPS2Ra partitioning step (arXiv 2009.13569).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product package ``paper_2009_13569_b200`` never imports it and
shares no code with it.

The arithmetic lives in ``oracle.c`` (plain C, one thread); this module only
builds/loads it with ctypes and marshals numpy arrays.  Citations are in
``oracle.h``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

U64, F64, PAIR, REC100, U32, QUARTET = 0, 1, 2, 3, 4, 5
ELEM_BYTES = {U64: 8, F64: 8, PAIR: 16, REC100: 100, U32: 4, QUARTET: 32}
DTYPE_NAMES = {"u64": U64, "f64": F64, "pair": PAIR, "rec100": REC100, "u32": U32, "quartet": QUARTET}

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc into oracle/liboracle.so (no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"]
        )
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, u64, i64, ci = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int
        L.orc_elem_bytes.argtypes = [ci]
        L.orc_elem_bytes.restype = ctypes.c_size_t
        L.orc_less.argtypes = [ci, vp, vp]
        L.orc_less.restype = ci
        L.orc_check_input.argtypes = [ci, vp, u64]
        L.orc_check_input.restype = i64
        L.orc_mergesort.argtypes = [vp, u64, ci]
        L.orc_mergesort.restype = ci
        L.orc_insertion_sort.argtypes = [vp, u64, ci]
        L.orc_insertion_sort.restype = ci
        L.orc_is_sorted.argtypes = [vp, u64, ci]
        L.orc_is_sorted.restype = ci
        L.orc_multiset_hash.argtypes = [vp, u64, ci]
        L.orc_multiset_hash.restype = u64
        L.orc_parity_check.argtypes = [vp, vp, u64, ci]
        L.orc_parity_check.restype = i64
        L.orc_sample_index.argtypes = [u64, ctypes.c_uint32, u64, u64, u64]
        L.orc_sample_index.restype = u64
        L.orc_select_splitters.argtypes = [vp, u64, ci, ci, ci, vp,
                                           ctypes.POINTER(ci), ctypes.POINTER(ci)]
        L.orc_select_splitters.restype = ci
        L.orc_build_tree.argtypes = [vp, ci, ci, vp, vp]
        L.orc_build_tree.restype = ci
        L.orc_classify_linear.argtypes = [vp, ci, ci, ci, vp]
        L.orc_classify_linear.restype = ci
        L.orc_classify_tree.argtypes = [vp, vp, ci, ci, ci, vp]
        L.orc_classify_tree.restype = ci
        L.orc_radix_digit.argtypes = [ci, vp, ci, ci]
        L.orc_radix_digit.restype = ctypes.c_uint32
        L.orc_log_digit.argtypes = [ctypes.c_uint64, ci]
        L.orc_log_digit.restype = ctypes.c_uint32
        L.orc_boundaries.argtypes = [vp, ci, u64, vp, vp]
        L.orc_boundaries.restype = None
        L.orc_histogram.argtypes = [vp, u64, ci, vp, ci, ci, vp]
        L.orc_histogram.restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def as_bytes(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a).view(np.uint8).reshape(-1)


def nelems(a: np.ndarray, dtype: int) -> int:
    return a.nbytes // ELEM_BYTES[dtype]


def sort(a: np.ndarray, dtype: int) -> np.ndarray:
    """Return a sorted copy of ``a`` (the oracle: plain mergesort)."""
    out = np.ascontiguousarray(a).copy()
    rc = lib().orc_mergesort(_ptr(out), nelems(out, dtype), dtype)
    if rc != 0:
        raise MemoryError("oracle mergesort failed")
    return out


def sort_inplace(a: np.ndarray, dtype: int) -> None:
    rc = lib().orc_mergesort(_ptr(a), nelems(a, dtype), dtype)
    if rc != 0:
        raise MemoryError("oracle mergesort failed")


def insertion_sort(a: np.ndarray, dtype: int) -> np.ndarray:
    out = np.ascontiguousarray(a).copy()
    lib().orc_insertion_sort(_ptr(out), nelems(out, dtype), dtype)
    return out


def is_sorted(a: np.ndarray, dtype: int) -> bool:
    a = np.ascontiguousarray(a)
    return bool(lib().orc_is_sorted(_ptr(a), nelems(a, dtype), dtype))


def multiset_hash(a: np.ndarray, dtype: int) -> int:
    a = np.ascontiguousarray(a)
    return int(lib().orc_multiset_hash(_ptr(a), nelems(a, dtype), dtype))


def check_input(a: np.ndarray, dtype: int) -> int:
    a = np.ascontiguousarray(a)
    return int(lib().orc_check_input(dtype, _ptr(a), nelems(a, dtype)))


def parity(g: np.ndarray, o: np.ndarray, dtype: int) -> int:
    """-1 if GPU result ``g`` matches oracle result ``o``, else first bad index."""
    g = np.ascontiguousarray(g)
    o = np.ascontiguousarray(o)
    assert g.nbytes == o.nbytes
    return int(lib().orc_parity_check(_ptr(g), _ptr(o), nelems(o, dtype), dtype))


def less(dtype: int, a: np.ndarray, b: np.ndarray) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return bool(lib().orc_less(dtype, _ptr(a), _ptr(b)))


def sample_index(seed: int, level: int, begin: int, size: int, j: int) -> int:
    return int(lib().orc_sample_index(seed, level, begin, size, j))


def select_splitters(sorted_sample: np.ndarray, k: int, kidx_max: int, dtype: int):
    """Return (splitters ndarray (u elements), equality, k_final)."""
    s = np.ascontiguousarray(sorted_sample)
    D = ELEM_BYTES[dtype]
    m = s.nbytes // D
    out = np.zeros(max(k - 1, 1) * D, dtype=np.uint8)
    eq = ctypes.c_int(0)
    kf = ctypes.c_int(0)
    u = lib().orc_select_splitters(_ptr(s), m, k, kidx_max, dtype, _ptr(out),
                                   ctypes.byref(eq), ctypes.byref(kf))
    return out[: u * D].copy(), bool(eq.value), int(kf.value)


def build_tree(splitters: np.ndarray, dtype: int):
    """Return (tree bytes, splitter bytes, l) for u unique splitters."""
    sp = np.ascontiguousarray(splitters).view(np.uint8).reshape(-1)
    D = ELEM_BYTES[dtype]
    u = sp.nbytes // D
    leaves = 1
    while leaves < u + 1:
        leaves *= 2
    tree = np.zeros(leaves * D, dtype=np.uint8)
    spl = np.zeros(leaves * D, dtype=np.uint8)
    l = lib().orc_build_tree(_ptr(sp), u, dtype, _ptr(tree), _ptr(spl))
    return tree, spl, int(l)


def classify_linear(splitter: np.ndarray, l: int, equality: bool, dtype: int, e: np.ndarray) -> int:
    sp = np.ascontiguousarray(splitter)
    e = np.ascontiguousarray(e)
    return int(lib().orc_classify_linear(_ptr(sp), l, int(equality), dtype, _ptr(e)))


def classify_tree(tree: np.ndarray, splitter: np.ndarray, l: int, equality: bool, dtype: int,
                  e: np.ndarray) -> int:
    t = np.ascontiguousarray(tree)
    sp = np.ascontiguousarray(splitter)
    e = np.ascontiguousarray(e)
    return int(lib().orc_classify_tree(_ptr(t), _ptr(sp), l, int(equality), dtype, _ptr(e)))


def radix_digit(dtype: int, e: np.ndarray, shift: int, bits: int) -> int:
    e = np.ascontiguousarray(e)
    return int(lib().orc_radix_digit(dtype, _ptr(e), shift, bits))


def log_digit(d: int, M: int) -> int:
    """Logarithmic digit of the offset d (DESIGN R33)."""
    return int(lib().orc_log_digit(int(d), int(M)))


def boundaries(count, b: int):
    c = np.ascontiguousarray(np.asarray(count, dtype=np.uint64))
    k = c.size
    E = np.zeros(k + 1, dtype=np.uint64)
    d = np.zeros(k + 1, dtype=np.uint64)
    lib().orc_boundaries(_ptr(c), k, b, _ptr(E), _ptr(d))
    return E, d


def histogram(a: np.ndarray, dtype: int, splitter: np.ndarray, l: int, equality: bool) -> np.ndarray:
    a = np.ascontiguousarray(a)
    sp = np.ascontiguousarray(splitter)
    K = (1 << (l + 1)) if equality else (1 << l)
    h = np.zeros(K, dtype=np.uint64)
    lib().orc_histogram(_ptr(a), nelems(a, dtype), dtype, _ptr(sp), l, int(equality), _ptr(h))
    return h


def elements(a: np.ndarray, dtype: int) -> np.ndarray:
    """View any buffer as an (n, D) uint8 matrix of elements."""
    return as_bytes(a).reshape(-1, ELEM_BYTES[dtype])


def sample_tree(arr: np.ndarray, dtype: int, begin: int, size: int, seed: int, level: int,
                k: int, alpha: int, kidx_max: int):
    """Sub-oracle of the sampling phase (DESIGN R8): draw m = alpha*k
    samples with sample_index, sort them with the oracle, select splitters,
    build the tree.  Returns dict(tree, splitter, l, equality, k, u)."""
    E = elements(arr, dtype)
    m = alpha * k
    idx = [sample_index(seed, level, begin, size, j) for j in range(m)]
    samp = np.ascontiguousarray(E[np.asarray(idx, dtype=np.int64)])
    samp = sort(samp, dtype)
    sp, eq, kf = select_splitters(samp, k, kidx_max, dtype)
    tree, spl, l = build_tree(sp, dtype)
    return dict(tree=tree, splitter=spl, l=l, equality=eq, k=kf, u=sp.size // ELEM_BYTES[dtype])
