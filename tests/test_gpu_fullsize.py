"""Parity at BASELINE.json's full sizes (the five configs + the 2^30 headline),
in the launch configuration bench.py times (default options, one ips4o_sort).

Every result is compared element by element with the oracle's output
(oracle.parity, tolerance 0), or with an exact closed form of the
sorted input where the distribution has one (RootDup, AlmostSorted,
Sorted/ReverseSorted, Ones, Zero) or an exact O(n) pin (pairs: the values are
the permutation 0..n-1).  At 2^28-2^30 the oracle's single-threaded mergesort
takes minutes per input, so those sorts run as background host processes
started at collection time (tests/oracle_jobs.py, conftest.py) while the other
GPU tests run; these tests are ordered last and wait for their job.
Set IPS4O_SKIP_FULLSIZE=1 to skip (e.g. on small GPUs).
"""
import math
import os

import numpy as np
import pytest

import synth_inputs as gen
from gpu_util import F64, PAIR, QUARTET, REC100, U32, U64

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CH = 1 << 24
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


@pytest.fixture(scope="module")
def ips():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if os.environ.get("IPS4O_SKIP_FULLSIZE"):
        pytest.skip("IPS4O_SKIP_FULLSIZE set")
    from paper_2009_13569_b200 import build

    build.build()
    import paper_2009_13569_b200 as p

    p.load()
    return p


def words(a):
    return np.ascontiguousarray(a).view(np.uint64).reshape(-1)


def mhash(a) -> int:
    """Order-independent multiset hash over 8-byte words grouped per element."""
    w = words(a)
    per = a.dtype.itemsize * (a.shape[1] if a.ndim == 2 else 1) // 8
    s = np.uint64(0)
    with np.errstate(over="ignore"):
        for c0 in range(0, w.size, CH * per):
            x = w[c0:c0 + CH * per].reshape(-1, per)
            h = np.full(x.shape[0], np.uint64(0x0123456789ABCDEF))
            for c in range(per):
                z = h ^ x[:, c]
                z = (z ^ (z >> np.uint64(30))) * M1
                z = (z ^ (z >> np.uint64(27))) * M2
                h = z ^ (z >> np.uint64(31))
            s = s + h.sum(dtype=np.uint64)
    return int(s)


def nondecreasing(keys) -> bool:
    for c0 in range(0, keys.size - 1, CH):
        k = keys[c0:c0 + CH + 1]
        if not np.all(k[1:] >= k[:-1]):
            return False
    return True


def order_stat_ok(inp_keys, out_keys, idx) -> bool:
    v = out_keys[idx]
    lt = 0
    le = 0
    for c0 in range(0, inp_keys.size, CH * 4):
        k = inp_keys[c0:c0 + CH * 4]
        lt += int(np.count_nonzero(k < v))
        le += int(np.count_nonzero(k <= v))
    return lt <= idx < le


def oracle_equal(pool, orc, g, name, n, seed, dtype):
    """Element-by-element comparison of the GPU output with the oracle's
    sorted copy of the same seeded input (written by the background job)."""
    assert pool is not None, "oracle job pool not started"
    path = pool.wait(name, n, seed)
    o = np.memmap(path, dtype=g.dtype, mode="r", shape=g.shape)
    bad = orc.parity(g, o, dtype)
    del o
    assert bad == -1, f"{name} 2^{n.bit_length() - 1}: GPU output differs from the oracle at {bad}"


def run(ips, a, dtype):
    import torch

    b = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    t = torch.from_numpy(b).to("cuda")
    ips.sort(t, dtype)  # default options: the configuration bench.py times
    torch.cuda.synchronize()
    g = t.cpu().numpy().view(a.dtype).reshape(a.shape)
    del t
    torch.cuda.empty_cache()
    return g


def sampled(ips, a, g, keyf, nsamp=6, seed=0):
    rng = np.random.default_rng(seed)
    ka, kg = keyf(a), keyf(g)
    n = kg.size
    for i in [0, n - 1] + list(rng.integers(0, n, nsamp)):
        assert order_stat_ok(ka, kg, int(i)), f"order statistic {i} wrong"


def test_c1_uniform_u64_full_oracle(ips, orc):
    a = gen.uniform_u64(1 << 20, 1)
    g = run(ips, a, U64)
    assert orc.parity(g, orc.sort(a, U64), U64) == -1


@pytest.mark.parametrize("name", ["uniform_f64", "exponential_f64", "almost_sorted_f64",
                                  "sorted_f64", "reverse_sorted_f64"])
def test_c2_doubles(ips, orc, oracle_pool, name):
    n = 1 << 28
    a = gen.generate(name, n, 2)
    assert orc.check_input(a[: 1 << 20], F64) == -1
    g = run(ips, a, F64)
    if name in ("uniform_f64", "exponential_f64"):
        del a
        oracle_equal(oracle_pool, orc, g, name, n, 2, F64)
        return
    assert nondecreasing(g)
    assert mhash(g) == mhash(a)
    if name == "almost_sorted_f64":
        assert np.array_equal(g, np.arange(n, dtype=np.float64))
    elif name == "sorted_f64":
        assert np.array_equal(g, a)
    elif name == "reverse_sorted_f64":
        assert np.array_equal(g, a[::-1])


@pytest.mark.parametrize("name", ["rootdup_u64", "twodup_u64", "zipf_u64", "ones_u64",
                                  "eightdup_u64", "zero_u64"])
def test_c3_duplicates(ips, orc, oracle_pool, name):
    """c3 (+ the paper's EightDup and Zero)."""
    n = 1 << 30
    a = gen.generate(name, n, 3)
    g = run(ips, a, U64)
    if name == "rootdup_u64":
        r = math.isqrt(n)
        for c0 in range(0, n, CH):
            j = np.arange(c0, min(n, c0 + CH), dtype=np.uint64)
            assert np.array_equal(g[c0:c0 + CH], j // np.uint64(r))
        return
    if name == "ones_u64":
        assert np.all(g == 1)
        return
    if name == "zero_u64":
        assert not g.any()
        return
    if name in ("twodup_u64", "eightdup_u64"):
        del a
        oracle_equal(oracle_pool, orc, g, name, n, 3, U64)
        return
    assert name == "zipf_u64"
    # counting sort over the 2^20 ranks (an independent pin of the oracle's
    # output at this size): sampled value runs
    cnt = np.zeros(gen.ZIPF_VALUES + 1, dtype=np.int64)
    for c0 in range(0, n, CH):
        cnt += np.bincount(a[c0:c0 + CH].astype(np.int64), minlength=gen.ZIPF_VALUES + 1)
    del a
    ends = np.cumsum(cnt)
    starts = ends - cnt
    for v in np.nonzero(cnt)[0][:: max(1, np.count_nonzero(cnt) // 2000)]:
        assert np.all(g[starts[v]:ends[v]] == v)
    oracle_equal(oracle_pool, orc, g, name, n, 3, U64)


def test_u32_uniform_2p28(ips, orc, oracle_pool):
    """32-bit keys at 2^28 against the full oracle."""
    n = 1 << 28
    a = gen.uniform_u32(n, 6)
    g = run(ips, a, U32)
    del a
    oracle_equal(oracle_pool, orc, g, "uniform_u32", n, 6, U32)


def test_quartet_2p24_full_oracle(ips, orc):
    """Quartet (Alg. 3) at 2^24 (512 MiB) against the
    full oracle: identical key sequence and record multisets."""
    n = 1 << 24
    a = gen.quartets(n, 7)
    g = run(ips, a, QUARTET)
    assert orc.parity(g, orc.sort(a, QUARTET), QUARTET) == -1


def test_c4_pairs(ips, orc):
    n = 1 << 28
    a = gen.pairs(n, 4)
    g = run(ips, a, PAIR)
    assert nondecreasing(g[:, 0])
    # exact multiset pin: values are the permutation 0..n-1
    # and every output pair is the input pair its value names
    vals = g[:, 1].astype(np.int64)
    seen = np.zeros(n, dtype=bool)
    seen[vals] = True
    assert seen.all()
    for c0 in range(0, n, CH):
        v = vals[c0:c0 + CH]
        assert np.array_equal(a[v], g[c0:c0 + CH])


def test_c5_records_full_oracle(ips, orc):
    n = 1 << 24
    a = gen.records100(n, 5)
    g = run(ips, a, REC100)
    assert orc.parity(g, orc.sort(a, REC100), REC100) == -1


def test_headline_uniform_u64(ips, orc, oracle_pool):
    """The 2^30 headline bench.py times (seed 42), against the full oracle."""
    n = 1 << 30
    a = gen.uniform_u64(n, 42)
    g = run(ips, a, U64)
    del a
    oracle_equal(oracle_pool, orc, g, "uniform_u64", n, 42, U64)
