"""Parity at BASELINE.json's full sizes (the five configs + the 2^30 headline),
in the launch configuration bench.py times (default options, one ips4o_sort).

At these sizes the oracle's full mergesort takes minutes, so each result is
checked with:
  * properties that hold at any size: output non-decreasing and an identical
    multiset (order-independent 64-bit hash of the element bytes, computed
    here in numpy, independent of the CUDA path);
  * sampled outputs the oracle-side definition gives one by one: for random
    positions i, out[i] is the i-th order statistic of the input
    (#{x < out[i]} <= i < #{x <= out[i]}, counted on the input);
  * closed forms and counting sorts where the distribution has them
    (RootDup, AlmostSorted, Sorted/ReverseSorted, Ones, Zipf);
  * the full oracle where it finishes in seconds (c1, and c5 records).
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
def test_c2_doubles(ips, orc, name):
    n = 1 << 28
    a = gen.generate(name, n, 2)
    assert orc.check_input(a[: 1 << 20], F64) == -1
    g = run(ips, a, F64)
    assert nondecreasing(g)
    assert mhash(g) == mhash(a)
    if name == "almost_sorted_f64":
        assert np.array_equal(g, np.arange(n, dtype=np.float64))
    elif name == "sorted_f64":
        assert np.array_equal(g, a)
    elif name == "reverse_sorted_f64":
        assert np.array_equal(g, a[::-1])
    else:
        sampled(ips, a, g, lambda x: x)


@pytest.mark.parametrize("name", ["rootdup_u64", "twodup_u64", "zipf_u64", "ones_u64",
                                  "eightdup_u64", "zero_u64"])
def test_c3_duplicates(ips, orc, name):
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
    assert nondecreasing(g)
    if name == "zipf_u64":
        # counting sort over the 2^20 ranks: exact expected output
        cnt = np.zeros(gen.ZIPF_VALUES + 1, dtype=np.int64)
        for c0 in range(0, n, CH):
            cnt += np.bincount(a[c0:c0 + CH].astype(np.int64), minlength=gen.ZIPF_VALUES + 1)
        ends = np.cumsum(cnt)
        starts = ends - cnt
        for v in np.nonzero(cnt)[0][:: max(1, np.count_nonzero(cnt) // 2000)]:
            assert np.all(g[starts[v]:ends[v]] == v)
        assert mhash(g) == mhash(a)
        return
    assert mhash(g) == mhash(a)
    sampled(ips, a, g, lambda x: x)


def test_u32_uniform_2p28(ips, orc):
    """32-bit keys at 2^28: non-decreasing, identical
    multiset, sampled order statistics, and the full oracle on a 2^22 prefix
    sorted separately."""
    n = 1 << 28
    a = gen.uniform_u32(n, 6)
    g = run(ips, a, U32)
    assert nondecreasing(g)
    assert mhash(g.astype(np.uint64)) == mhash(a.astype(np.uint64))
    sampled(ips, a, g, lambda x: x)
    b = a[: 1 << 22].copy()
    gb = run(ips, b, U32)
    assert orc.parity(gb, orc.sort(b, U32), U32) == -1


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


def test_headline_uniform_u64(ips, orc):
    n = 1 << 30
    a = gen.uniform_u64(n, 42)
    g = run(ips, a, U64)
    assert nondecreasing(g)
    assert mhash(g) == mhash(a)
    sampled(ips, a, g, lambda x: x, nsamp=4)
