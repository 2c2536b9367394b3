"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/ips4o.h declares; host-side argument validation (no GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ips4o.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ips4o_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2009_13569_b200 import build

    build.build()
    import paper_2009_13569_b200 as p

    return p.load()


def test_header_declares_the_survey_entry_points():
    fns = declared_functions()
    for f in ["ips4o_sort", "ips4o_sort_ex", "ips4o_scratch_bytes", "ips4o_status_string"]:
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    import paper_2009_13569_b200 as p

    for f in declared_functions():
        assert hasattr(lib, f), f"{f} declared in include/ips4o.h but not exported"
    assert set(declared_functions()) == set(p.EXPORTS)


def test_built_for_sm100a():
    import subprocess

    from paper_2009_13569_b200 import build

    so = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def test_argument_validation_without_gpu(lib):
    import paper_2009_13569_b200 as p

    # n <= 1 returns 0 without device work
    assert lib.ips4o_sort(None, 0, p.U64, None) == 0
    assert lib.ips4o_sort(None, 1, p.U64, None) == 0
    # unknown dtype, NULL pointer, misaligned pointer
    assert lib.ips4o_sort(None, 10, 7, None) == -1
    assert lib.ips4o_sort(None, 10, p.U64, None) == -1
    # alignment: 4 B for U32, 8 B for U64/F64, 16 B for the others (ips4o.h)
    assert lib.ips4o_sort(ctypes.c_void_p(4), 10, p.U64, None) == -1
    assert lib.ips4o_sort(ctypes.c_void_p(2), 10, p.U32, None) == -1
    assert lib.ips4o_sort(ctypes.c_void_p(8), 10, p.PAIR, None) == -1
    assert lib.ips4o_sort(ctypes.c_void_p(8), 10, p.REC100, None) == -1
    assert lib.ips4o_sort(ctypes.c_void_p(16), 1 << 32, p.U64, None) == -1
    # k_max < 4 is rejected for the tree (no progress guarantee), allowed for digits
    o = p.Options()
    o.k_max = 2
    assert lib.ips4o_sort_ex(ctypes.c_void_p(16), 10, p.U64, None, ctypes.byref(o), None) == -1
    o.k_max = 3
    o.algo = p.DIGIT
    assert lib.ips4o_sort_ex(ctypes.c_void_p(16), 10, p.U64, None, ctypes.byref(o), None) == -1
    # well-formed calls on a machine without a GPU report it
    if not _has_gpu():
        assert lib.ips4o_sort(ctypes.c_void_p(8), 10, p.U64, None) == -4
        o.k_max = 2
        assert lib.ips4o_sort_ex(ctypes.c_void_p(16), 10, p.U64, None, ctypes.byref(o), None) == -4
        f = ctypes.c_uint32(7)
        assert lib.ips4o_device_status(0, ctypes.byref(f), 0) == 0 and f.value == 0
    assert lib.ips4o_status_string(-1).decode() == "invalid argument"
    assert "sm_100" in lib.ips4o_status_string(-4).decode()


def test_dtype_info_and_scratch_bound(lib):
    import paper_2009_13569_b200 as p

    for dt, D in p.ELEM_BYTES.items():
        info = p.dtype_info(dt)
        assert info["elem_bytes"] == D
        # whole 32-byte sectors per block
        assert (info["block_elems"] * D) % 32 == 0
        assert info["kidx_max"] in (128, 256)
        assert info["base_cap"] * D <= 200 * 1024
    # scratch grows sub-linearly relative to the input (in-place)
    n = 1 << 30
    sb = p.scratch_bytes(n, p.U64)
    assert 0 < sb < 0.15 * n * 8
