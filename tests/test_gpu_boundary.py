"""The boundary contract of include/ips4o.h on the GPU:
stream-asynchronous calls (the recursion is planned and launched on the
device, Alg. 2), CUDA-graph capture and replay, pointer alignment
per dtype, levels with more than 65535 tasks, the k_max rule of the tree, the
bounded arena (rounds that defer tasks), and the device status word.  Every
sorted result is compared with the oracle (tolerance 0)."""
import ctypes

import numpy as np
import pytest

import synth_inputs as gen
from gpu_util import PAIR, U32, U64, from_dev, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ips():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2009_13569_b200 import build

    build.build()
    import paper_2009_13569_b200 as p

    p.load()
    return p


def test_sort_returns_before_the_work_completes(ips, orc):
    """ips4o_sort enqueues and returns (no host synchronisation): right after
    the call the stream still has work; the result is the oracle's."""
    import torch

    n = 1 << 26
    a = gen.uniform_u64(n, 11)
    t = to_dev(a)
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        ips.sort(t, U64)
        busy = not s.query()
    s.synchronize()
    assert busy, "the stream was idle right after ips4o_sort returned"
    assert orc.parity(from_dev(t, a), orc.sort(a, U64), U64) == -1
    assert ips.device_status() == 0


@pytest.mark.parametrize("dtype,n,kind", [(U64, 1 << 22, "uniform"), (U64, 3_000_017, "dups"), (PAIR, 1 << 20, "uniform"),
                                          (U32, 100_003, "uniform"), (U64, 20_000, "uniform")])
def test_graph_capture_and_replay(ips, orc, dtype, n, kind):
    """The whole sort (scratch allocation, host-launched round 0, device-planned
    later rounds, free) is captured into a CUDA graph and replayed on fresh
    inputs; every replay equals the oracle."""
    import torch

    rng = np.random.default_rng(n)
    if dtype == U64:
        a0 = gen.uniform_u64(n, 3) if kind == "uniform" else rng.integers(0, n // 50, n).astype(np.uint64)
    elif dtype == U32:
        a0 = gen.uniform_u32(n, 3)
    else:
        a0 = gen.pairs(n, 3)
    t = to_dev(a0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ips.sort(t, dtype)  # first call on the device: creates the pool and status word
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ips.sort(t, dtype)
    for seed in (5, 6):
        if dtype == U64:
            a = gen.uniform_u64(n, seed) if kind == "uniform" else rng.integers(0, n // 50, n).astype(np.uint64)
        elif dtype == U32:
            a = gen.uniform_u32(n, seed)
        else:
            a = gen.pairs(n, seed)
        t.copy_(to_dev(a))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert orc.parity(from_dev(t, a), orc.sort(a, dtype), dtype) == -1, seed
    assert ips.device_status() == 0


def test_pointer_alignment_per_dtype(ips, orc):
    """U64/F64 need 8-byte alignment (not 16), U32 4 bytes; PAIR 16 bytes."""
    import torch

    n = 300_001
    a = gen.uniform_u64(n + 1, 9)
    t = to_dev(a)
    sub = t[8:]  # the elements 1..n: 8-byte aligned, not 16
    assert sub.data_ptr() % 16 == 8
    ips.sort(sub, U64)
    torch.cuda.synchronize()
    g = from_dev(t, a)
    assert g[0] == a[0]
    assert orc.parity(g[1:], orc.sort(a[1:], U64), U64) == -1
    b = gen.uniform_u32(n + 1, 9)
    tb = to_dev(b)
    ips.sort(tb[4:], U32)
    gb = from_dev(tb, b)
    assert orc.parity(gb[1:], orc.sort(b[1:], U32), U32) == -1
    pr = gen.pairs(1001, 2)
    tp = to_dev(pr)
    with pytest.raises(ips.IPS4OError):
        ips.sort(tp[8:8 + 16 * 1000], PAIR)


def test_level_with_more_than_65535_tasks(ips, orc):
    """A small base-case capacity forces > 65535 tasks at level 3 (the cleanup
    grids are flattened; gridDim.y would cap them at 65535).  A large arena
    lets that level run as ONE round; with the default arena it runs in
    several rounds."""
    import torch

    n = 1 << 25
    a = gen.uniform_u64(n, 21)
    t = to_dev(a)
    st = ips.sort_ex(t, U64, base_cap=64, arena_mb=6144)
    g = from_dev(t, a)
    assert max(st["tasks_per_level"]) > 65535, st["tasks_per_level"]
    assert orc.parity(g, orc.sort(a, U64), U64) == -1
    t.copy_(to_dev(a))
    st = ips.sort_ex(t, U64, base_cap=64)
    assert max(st["tasks_per_level"]) < 65536 and st["levels"] > 3, st["tasks_per_level"]
    assert orc.parity(from_dev(t, a), orc.sort(a, U64), U64) == -1
    del t
    torch.cuda.empty_cache()


def test_k_max_rule_of_the_tree(ips, orc):
    """k_max = 2 is rejected for the tree (one splitter equal to the maximum
    would leave everything in one bucket); k_max = 4 sorts a majority-maximum
    input; k_max = 2 is fine for the digit extractor."""
    import torch

    n = 200_003
    rng = np.random.default_rng(4)
    a = np.where(rng.random(n) < 0.7, np.uint64(2**64 - 1), rng.integers(0, 2**63, n).astype(np.uint64))
    t = to_dev(a)
    with pytest.raises(ips.IPS4OError):
        ips.sort_ex(t, U64, k_max=2, base_cap=1000)
    st = ips.sort_ex(t, U64, k_max=4, base_cap=1000)
    assert orc.parity(from_dev(t, a), orc.sort(a, U64), U64) == -1
    assert st["levels"] >= 1
    t2 = to_dev(a)
    ips.sort_ex(t2, U64, k_max=2, algo=ips.DIGIT, base_cap=1000)
    assert orc.parity(from_dev(t2, a), orc.sort(a, U64), U64) == -1
    torch.cuda.synchronize()


def test_rounds_defer_tasks_when_the_arena_is_full(ips, orc):
    """Skewed second levels (many more tasks than the arena was sized for)
    run in several rounds; the result is unchanged."""
    n = 1 << 22
    rng = np.random.default_rng(8)
    # a few dense clusters and a sparse background: level 2 tasks are very unequal
    a = np.concatenate([rng.integers(0, 1 << 20, n // 2), rng.integers(0, 2**64 - 1, n - n // 2, dtype=np.uint64)])
    a = a.astype(np.uint64)
    rng.shuffle(a)
    t = to_dev(a)
    st = ips.sort_ex(t, U64, base_cap=128, arena_mb=1)  # the arena holds the root level only
    assert orc.parity(from_dev(t, a), orc.sort(a, U64), U64) == -1
    assert st["deferred_tasks"] > 0, st
    t.copy_(to_dev(a))
    st = ips.sort_ex(t, U64, base_cap=128)
    assert st["deferred_tasks"] == 0, st
    assert orc.parity(from_dev(t, a), orc.sort(a, U64), U64) == -1


def test_device_status_word(ips):
    f = ctypes.c_uint32(99)
    assert ips.load().ips4o_device_status(0, ctypes.byref(f), 0) == 0
    assert f.value == 0
    assert ips.load().ips4o_device_status(-1, ctypes.byref(f), 0) == -1
    ips.release_memory(0)
