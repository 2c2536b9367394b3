"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle.

Tolerance 0 (BASELINE.json north_star): U64/F64 byte-identical output; PAIR and
REC100 identical key sequence and identical record multiset inside every run
of equal keys (oracle.parity).  Sizes span several tiles, stripes and blocks
with ragged tails; base_cap is lowered in some cases to force several
partitioning levels at sizes the oracle finishes in seconds.
"""
import math

import numpy as np
import pytest

import synth_inputs as gen
from gpu_util import (F64, PAIR, QUARTET, REC100, U32, U64, from_dev, gpu_sort, key_bytes_of,
                      splitters_as_elements, to_dev)

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


def make(dtype, n, seed, kind="uniform"):
    rng = np.random.default_rng(seed)
    if kind == "zipf":  # Zipf ranks (the splitters crowd the low end: logarithmic lookup table)
        z = gen.zipf_u64(n, seed)
        if dtype == U64:
            return z
        if dtype == F64:
            return z.astype(np.float64) * 0.5
        if dtype == U32:
            return z.astype(np.uint32)
        if dtype == PAIR:
            p = gen.pairs(n, seed)
            p[:, 0] = z
            return p
        if dtype == QUARTET:
            q = gen.quartets(n, seed)
            q[:, 0] = 0
            q[:, 1] = z
            return q
        r = gen.records100(n, seed)
        r[:, :10] = 0
        r[:, 6:10] = z.astype(">u4").view(np.uint8).reshape(-1, 4)
        return r
    if dtype == QUARTET:
        q = gen.quartets(n, seed)
        if kind == "dups":
            q[:, 0] = rng.integers(0, 2, n).astype(np.uint64)
            q[:, 1] = rng.integers(0, 3, n).astype(np.uint64)
            q[:, 2] = rng.integers(0, max(2, n // 16), n).astype(np.uint64)
        if kind == "few":
            q[:, :3] = 0
            q[:, 2] = rng.integers(0, 3, n).astype(np.uint64)
        return q
    if dtype == U32:
        if kind == "uniform":
            return gen.uniform_u32(n, seed)
        if kind == "dups":
            return rng.integers(0, max(2, n // 16), n).astype(np.uint32)
        if kind == "few":
            return rng.integers(0, 3, n).astype(np.uint32)
        return np.sort(gen.uniform_u32(n, seed))
    if dtype == U64:
        if kind == "uniform":
            return gen.uniform_u64(n, seed)
        if kind == "dups":
            return rng.integers(0, max(2, n // 16), n).astype(np.uint64)
        if kind == "few":
            return rng.integers(0, 3, n).astype(np.uint64)
    if dtype == F64:
        if kind == "uniform":
            return gen.uniform_f64(n, seed)
        if kind == "dups":
            return np.round(gen.exponential_f64(n, seed), 2)
        if kind == "few":
            return rng.choice([-1.5, 0.0, 2.25], n)
    if dtype == PAIR:
        p = gen.pairs(n, seed)
        if kind == "dups":
            p[:, 0] = rng.integers(0, max(2, n // 16), n).astype(np.uint64)
        if kind == "few":
            p[:, 0] = rng.integers(0, 3, n).astype(np.uint64)
        return p
    r = gen.records100(n, seed)
    if kind == "dups":
        r[:, 2:10] = 0
        r[:, 1] = r[:, 1] % 4
    if kind == "few":
        r[:, :10] = 0
        r[:, 9] = rng.integers(0, 3, n).astype(np.uint8)
    return r


def check(orc, a, g, dtype):
    o = orc.sort(a, dtype)
    bad = orc.parity(g, o, dtype)
    assert bad == -1, f"mismatch at index {bad} (n={a.shape[0] if a.ndim else a.size})"


# ----------------------------------------------------------------- classifier
@pytest.mark.parametrize("dtype", [U64, F64, PAIR, REC100, U32, QUARTET])
@pytest.mark.parametrize("eq", [False, True])
def test_device_classifier_matches_oracle(ips, orc, dtype, eq):
    """The tree_bucket used by the classification/permutation kernels equals the
    oracle's linear-scan definition P:432-437 on 10^4 elements."""
    import torch

    n = 10000
    a = make(dtype, n, 3, "dups")
    D = orc.ELEM_BYTES[dtype]
    E = orc.elements(a, dtype)
    idx = np.unique(np.random.default_rng(5).integers(0, n, 60))
    sp = orc.sort(np.ascontiguousarray(E[idx]).reshape(-1), dtype).reshape(-1, D)
    # unique splitters under the dtype order
    uniq = [sp[0]]
    for r in sp[1:]:
        if orc.less(dtype, uniq[-1], r):
            uniq.append(r)
    uniq = np.stack(uniq)
    u = uniq.shape[0]
    raw = key_bytes_of(uniq.reshape(-1), dtype).tobytes()
    tree, spl, l = orc.build_tree(uniq.reshape(-1), dtype)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    ips.classify(to_dev(a), dtype, raw, u, eq, out)
    got = out.cpu().numpy()
    for i in range(0, n, 7):
        want = orc.classify_linear(spl, l, eq, dtype, E[i])
        assert got[i] == want, (i, got[i], want)


# ----------------------------------------------------------------- one level
@pytest.mark.parametrize("dtype", [U64, F64, PAIR, REC100, U32, QUARTET])
@pytest.mark.parametrize("n,kind", [(5003, "uniform"), (100003, "uniform"), (70001, "dups"),
                                    (40000, "few"), (1 << 20, "uniform"), (1 << 20, "zipf")])
def test_partition_step_tree(ips, orc, dtype, n, kind):
    """K1..K5 of one level: the sampled tree is bit-identical to
    the oracle's recomputation (same counter-based samples); E equals the
    oracle histogram prefix; every element of [E_j, E_{j+1}) classifies to j;
    each bucket holds exactly the oracle-sorted output restricted to it."""
    if dtype == REC100 and n > 200000:
        n = 200003
    a = make(dtype, n, 11, kind)
    t = to_dev(a)
    info = ips.partition_step(t, dtype, base_cap=2048)
    g = from_dev(t, a)
    K, l, eq = info["num_buckets"], info["l"], info["equality"]
    leaves = 1 << l
    # K1 parity
    st = orc.sample_tree(a, dtype, 0, n, info["seed"], 0, info["k_req"],
                         info["samples"] // info["k_req"], info["kidx_budget"])
    assert st["l"] == l and st["equality"] == eq and st["k"] == info["k_used"]
    kb = info["key_bytes"]
    D = orc.ELEM_BYTES[dtype]
    o_tree = key_bytes_of(st["tree"], dtype).reshape(-1)
    o_spl = key_bytes_of(st["splitter"], dtype).reshape(-1)
    assert np.array_equal(info["splitter"], o_spl), "splitters differ from the oracle's"
    assert np.array_equal(info["tree"][kb:], o_tree[kb:]), "tree differs from the oracle's"
    assert K == (2 * leaves if eq else leaves)
    if kind == "zipf" and dtype in (U64, U32, PAIR):
        assert info["lut_log"] > 0, "Zipf keys should take the logarithmic lookup table"
    if kind == "uniform" and n >= (1 << 20):
        assert info["lut_log"] == 0
    # K3 parity: E equals the oracle histogram prefix with these splitters
    spl_el = splitters_as_elements(info["splitter"], dtype, leaves)
    hist = orc.histogram(a, dtype, spl_el, l, eq)
    E = info["E"]
    assert E[0] == 0 and E[-1] == n
    assert np.array_equal(np.diff(E.astype(np.int64)), hist.astype(np.int64))
    # K5 parity: bucket contents
    o = orc.sort(a, dtype)
    Ge = orc.elements(g, dtype)
    Oe = orc.elements(o, dtype)
    rng = np.random.default_rng(1)
    for j in range(K):
        e0, e1 = int(E[j]), int(E[j + 1])
        if e1 == e0:
            continue
        probe = [e0, e1 - 1] + list(rng.integers(e0, e1, min(20, e1 - e0)))
        for i in probe:
            assert orc.classify_linear(spl_el, l, eq, dtype, Ge[i]) == j
        seg = orc.sort(np.ascontiguousarray(Ge[e0:e1]).reshape(-1), dtype)
        assert orc.parity(seg, np.ascontiguousarray(Oe[e0:e1]).reshape(-1), dtype) == -1, j


@pytest.mark.parametrize("nvals,shuffle", [(140, False), (200, True), (131, True), (250, False)])
def test_partition_step_equality_budget(ips, orc, nvals, shuffle):
    """R10 (DESIGN): more unique equality splitters than bucket indices.  With
    nvals heavy key values every value is picked; 140, 131 and 200 values are
    thinned (never two neighbours dropped); 250 cannot be thinned enough.  The tree must equal
    the oracle's; every bucket holds exactly its oracle-sorted range."""
    n = 1 << 21
    a = (np.arange(n, dtype=np.uint64) % np.uint64(nvals)) * np.uint64(7919)
    if shuffle:
        a = np.random.default_rng(nvals).permutation(a)
    t = to_dev(a)
    info = ips.partition_step(t, U64, base_cap=2048)
    g = from_dev(t, a)
    st = orc.sample_tree(a, U64, 0, n, info["seed"], 0, info["k_req"],
                         info["samples"] // info["k_req"], info["kidx_budget"])
    assert st["l"] == info["l"] and st["equality"] == info["equality"] and st["k"] == info["k_used"]
    assert np.array_equal(info["splitter"], key_bytes_of(st["splitter"], U64).reshape(-1))
    E = info["E"]
    o = orc.sort(a, U64)
    for j in range(info["num_buckets"]):
        e0, e1 = int(E[j]), int(E[j + 1])
        assert np.array_equal(np.sort(g[e0:e1]), o[e0:e1]), j
    if nvals < 250:
        # thinned, not halved: an open bucket holds a dropped splitter's keys
        # and at most one unpicked value (140 and 131: none)
        assert info["equality"] and info["k_used"] == info["k_req"]
        vmax = 1 if nvals < 200 else 2
        assert np.diff(E.astype(np.int64)).max() <= vmax * (n // nvals + 1)


@pytest.mark.parametrize("dtype", [U64, F64, PAIR, REC100, U32, QUARTET])
@pytest.mark.parametrize("n", [5003, 300007])
def test_partition_step_digit(ips, orc, dtype, n):
    """IPS2Ra step: bucket j holds exactly the elements whose
    digit (key >> shift) & (2^l - 1) is j, and the partition is consistent with
    the oracle's sorted output."""
    a = make(dtype, n, 12, "uniform")
    t = to_dev(a)
    info = ips.partition_step(t, dtype, algo=ips.DIGIT, base_cap=2048)
    g = from_dev(t, a)
    E = info["E"]
    K, sh, bits = info["num_buckets"], info["shift"], info["l"]
    assert K == 1 << bits and E[0] == 0 and E[-1] == n
    Ge = orc.elements(g, dtype)
    Oe = orc.elements(orc.sort(a, dtype), dtype)
    for j in range(K):
        e0, e1 = int(E[j]), int(E[j + 1])
        for i in range(e0, e1, max(1, (e1 - e0) // 16)):
            assert orc.radix_digit(dtype, Ge[i], sh, bits) == j
        if e1 > e0:
            seg = orc.sort(np.ascontiguousarray(Ge[e0:e1]).reshape(-1), dtype)
            assert orc.parity(seg, np.ascontiguousarray(Oe[e0:e1]).reshape(-1), dtype) == -1


@pytest.mark.parametrize("dtype", [U64, U32, PAIR])
@pytest.mark.parametrize("n", [300007, 1 << 21])
def test_partition_step_digit_adaptive(ips, orc, dtype, n):
    """Sample-adaptive IPS2Ra extractor (DESIGN R33): on Zipf keys
    the plain digit puts most of the sample into bucket 0, so the step uses the
    logarithmic digit of key - min key (lut_log = M > 0); bucket j holds
    exactly the elements whose oracle log digit is j, no bucket holds most of
    the input, and the partition is consistent with the oracle's sort."""
    a = make(dtype, n, 12, "zipf")
    t = to_dev(a)
    info = ips.partition_step(t, dtype, algo=ips.DIGIT, base_cap=2048)
    g = from_dev(t, a)
    E = info["E"]
    K, M = info["num_buckets"], info["lut_log"]
    assert M > 0 and info["shift"] == 0 and K == 1 << info["l"]
    assert E[0] == 0 and E[-1] == n
    z = gen.zipf_u64(n, 12)
    kmin = int(z.min())
    assert orc.log_digit(int(z.max()) - kmin, M) < K <= 256
    Ge = orc.elements(g, dtype)
    Oe = orc.elements(orc.sort(a, dtype), dtype)
    gk = (g if dtype != PAIR else g.reshape(-1, 2)[:, 0]).astype(np.uint64)
    sizes = np.diff(E.astype(np.int64))
    assert sizes.max() < n // 4  # the plain digit's bucket 0 holds > half of Zipf
    for j in range(K):
        e0, e1 = int(E[j]), int(E[j + 1])
        for i in range(e0, e1, max(1, (e1 - e0) // 16)):
            assert orc.log_digit(int(gk[i]) - kmin, M) == j
        if e1 > e0:
            assert orc.log_digit(int(gk[e1 - 1]) - kmin, M) == j
            seg = orc.sort(np.ascontiguousarray(Ge[e0:e1]).reshape(-1), dtype)
            assert orc.parity(seg, np.ascontiguousarray(Oe[e0:e1]).reshape(-1), dtype) == -1


@pytest.mark.parametrize("dtype", [U64, F64, U32, PAIR])
@pytest.mark.parametrize("n", [100003, 1 << 21, 5 * (1 << 20) + 17])
def test_sort_digit_adaptive_zipf(ips, orc, dtype, n):
    """Full IPS2Ra sorts of Zipf keys (adaptive extractor at the root, plain
    digits below) against the oracle."""
    a = make(dtype, n, 7, "zipf")
    g, _ = gpu_sort(a, dtype, algo=ips.DIGIT)
    check(orc, a, g, dtype)
    g, _ = gpu_sort(a, dtype, algo=ips.DIGIT, base_cap=1024)
    check(orc, a, g, dtype)


# ----------------------------------------------------------------- full sorts
SIZES = [0, 1, 2, 3, 31, 32, 33, 63, 64, 65, 4095, 4097, 24575, 24576, 24577, 49153, 100003]


@pytest.mark.parametrize("dtype", [U64, F64, PAIR, REC100, U32, QUARTET])
@pytest.mark.parametrize("n", SIZES)
def test_sort_sizes(ips, orc, dtype, n):
    a = make(dtype, n, n + 1, "uniform")
    g, _ = gpu_sort(a, dtype)
    check(orc, a, g, dtype)


@pytest.mark.parametrize("dtype", [U64, F64, PAIR, REC100, U32, QUARTET])
@pytest.mark.parametrize("kind", ["uniform", "dups", "few"])
@pytest.mark.parametrize("base_cap", [300, 1024])
def test_sort_deep_recursion(ips, orc, dtype, kind, base_cap):
    """Small base capacity forces 2-4 partitioning levels at oracle-friendly n."""
    n = 150001 if dtype != REC100 else 40001
    a = make(dtype, n, 21, kind)
    g, st = gpu_sort(a, dtype, base_cap=base_cap)
    check(orc, a, g, dtype)
    if kind == "uniform" and n > 256 * base_cap:
        assert st["levels"] >= 2


@pytest.mark.parametrize("dtype", [U64, F64, PAIR, REC100, U32, QUARTET])
@pytest.mark.parametrize("kind", ["uniform", "dups", "few"])
def test_sort_digit_algo(ips, orc, dtype, kind):
    n = 200003 if dtype != REC100 else 50001
    a = make(dtype, n, 31, kind)
    g, st = gpu_sort(a, dtype, algo=ips.DIGIT, base_cap=1024)
    check(orc, a, g, dtype)


@pytest.mark.parametrize("dtype", [U64, QUARTET])
def test_digit_sparse_keys_measured(ips, orc, dtype):
    """IPS2Ra on keys whose used bits are far apart (DESIGN R27): the level
    after a futile digit measures its exact range, so the recursion depth stays
    bounded by the used bits, not by the key width."""
    n = 1 << 20
    rng = np.random.default_rng(41)
    if dtype == U64:
        a = (rng.integers(0, 256, n).astype(np.uint64) << np.uint64(56)) | rng.integers(0, 1 << 20, n).astype(
            np.uint64
        )
    else:
        a = gen.quartets(n, 41)  # b: 20 bits of 64, c: 64 bits
        a[:, 0] = rng.integers(0, 256, n).astype(np.uint64)  # a: 8 bits
    g, st = gpu_sort(a, dtype, algo=ips.DIGIT, base_cap=1024)
    check(orc, a, g, dtype)
    # level 1: digit = a (256 tasks of ~4096); level 2: the digit right below a
    # is all zero (every task lands in one bucket, flagged); level 3 measures
    # the range of b and splits it.  Without the measurement the zero bits
    # between a and b would cost one futile level per digit.
    assert st["levels"] <= 3, st["tasks_per_level"]


@pytest.mark.parametrize("dtype", [U64, F64, U32])
@pytest.mark.parametrize("nvals", [5000, 40000])
def test_narrow_range_counting_base_case(ips, orc, dtype, nvals):
    """Key-only buckets whose key range is narrow are counted exactly in the
    base case whatever their size (K6 sends them there, K7 writes them from
    the counts); with base_cap=1000 most level-1 buckets exceed 2M."""
    n = (1 << 20) + 11
    rng = np.random.default_rng(nvals)
    v = rng.integers(0, nvals, n)
    if dtype == U64:
        a = (v.astype(np.uint64) + np.uint64(3 << 40))
    elif dtype == U32:
        a = (v + 123456).astype(np.uint32)
    else:
        # consecutive doubles (adjacent order-preserving keys) on both sides of 0
        ulp = np.float64(2.0**-52)
        a = np.where(v % 2 == 0, 1.0 + (v // 2) * ulp, -(1.0 + (v // 2) * ulp)).astype(np.float64)
    g, st = gpu_sort(a, dtype, base_cap=1000)
    check(orc, a, g, dtype)


@pytest.mark.parametrize("dtype", [U64, F64, U32])
@pytest.mark.parametrize("kind", ["random", "rootdup", "edge"])
def test_count_first_narrow_tasks(ips, orc, dtype, kind):
    """Children larger than the base case whose key range holds at most 4096
    values are counted and written from the counts (k_count.cuh): 2^25 keys
    over ~1000 values give level-1 buckets of ~131K elements and a few values
    each.  'edge' puts the values at the top of the key range (lo + v near
    the maximum key) and mixes in a wide tail so that some buckets are not
    narrow."""
    n = (1 << 25) + 5
    rng = np.random.default_rng(17)
    if kind == "random":
        v = rng.integers(0, 1000, n)
    elif kind == "rootdup":
        v = np.arange(n) % 1024
    else:
        v = rng.integers(0, 3000, n)
    if dtype == U64:
        a = v.astype(np.uint64) + (np.uint64(2**64 - 4000) if kind == "edge" else np.uint64(7 << 33))
        if kind == "edge":
            a[: n // 8] = gen.uniform_u64(n // 8, 5)
    elif dtype == U32:
        a = (v + (2**32 - 4000 if kind == "edge" else 99)).astype(np.uint32)
        if kind == "edge":
            a[: n // 8] = gen.uniform_u32(n // 8, 5)
    else:
        ulp = np.float64(2.0**-52)
        a = np.where(v % 2 == 0, 3.0 + (v // 2) * 2 * ulp, -(3.0 + (v // 2) * 2 * ulp)).astype(np.float64)
        if kind == "edge":
            a[: n // 8] = gen.uniform_f64(n // 8, 5)
    g, st = gpu_sort(a, dtype)
    check(orc, a, g, dtype)
    assert st["basecase_elems"] + st["equal_elems"] <= n


def _patterns(n, rng):
    m = np.uint64(2**64 - 1)
    u = gen.uniform_u64(n, 77)
    pats = {
        "all_equal": np.full(n, 42, dtype=np.uint64),
        "one_min": np.concatenate([np.full(n - 1, 9, dtype=np.uint64), [np.uint64(0)]]),
        "one_max": np.concatenate([np.full(n - 1, 9, dtype=np.uint64), [m]]),
        "alternating": (np.arange(n) % 2).astype(np.uint64),
        "many_max": np.where(rng.random(n) < 0.5, m, u).astype(np.uint64),
        "extremes": np.where(rng.random(n) < 0.5, np.uint64(0), m).astype(np.uint64),
        "k_distinct": (u % np.uint64(256)).astype(np.uint64),
        "sorted": np.sort(u),
        "reverse": np.sort(u)[::-1].copy(),
        "one_swap": None,
        "organ_pipe": np.concatenate([np.arange(n // 2), np.arange(n - n // 2)[::-1]]).astype(np.uint64),
        "skew_one_bucket": np.where(rng.random(n) < 0.97, np.uint64(5), u).astype(np.uint64),
        "zipf": gen.zipf_u64(n, 3),
        "twodup": gen.twodup_u64(n),
        "rootdup": gen.rootdup_u64(n),
    }
    s = np.sort(u)
    i = n // 3
    s[i], s[i + 1] = s[i + 1], s[i]
    pats["one_swap"] = s
    return pats


@pytest.mark.parametrize("name", ["all_equal", "one_min", "one_max", "alternating", "many_max",
                                  "extremes", "k_distinct", "sorted", "reverse", "one_swap",
                                  "organ_pipe", "skew_one_bucket", "zipf", "twodup", "rootdup"])
@pytest.mark.parametrize("base_cap", [0, 700])
def test_sort_value_patterns(ips, orc, name, base_cap):
    """SURVEY 8(c).3 value patterns (u64), default and forced recursion."""
    n = 200003
    a = _patterns(n, np.random.default_rng(9))[name]
    g, st = gpu_sort(a, U64, base_cap=base_cap)
    check(orc, a, g, U64)


@pytest.mark.parametrize("dtype", [U64, F64, PAIR, U32])
@pytest.mark.parametrize("kind", ["uniform", "dups", "few", "almost"])
def test_sort_sample_precheck_path(ips, orc, dtype, kind):
    """n >= 2^22: the sampled pre-check replaces the full pre-pass and the
    level-1 classification measures the key range (TF_MINMAX); 'almost'
    (sorted with a few swaps) usually sends it back to the full pre-pass."""
    n = (1 << 22) + 3
    if kind == "almost":
        a = make(dtype, n, 41, "uniform")
        if dtype == PAIR:
            a = a[np.argsort(a[:, 0], kind="stable")]
            a[[100, 101]] = a[[101, 100]]
        else:
            a = np.sort(a)
            a[[n // 2, n // 2 + 1]] = a[[n // 2 + 1, n // 2]]
    else:
        a = make(dtype, n, 41, kind)
    g, st = gpu_sort(a, dtype)
    check(orc, a, g, dtype)


def test_easy_inputs_reported(ips, orc):
    n = 100000
    s = np.sort(gen.uniform_u64(n, 1))
    g, st = gpu_sort(s, U64)
    assert st["easy_input"] == 1 and np.array_equal(g, s)
    g, st = gpu_sort(s[::-1].copy(), U64)
    assert st["easy_input"] == 2 and np.array_equal(g, s)
    g, st = gpu_sort(np.full(n, 3, dtype=np.uint64), U64)
    assert st["easy_input"] == 3


def test_f64_specials(ips, orc):
    """Negative values, +-inf, subnormals, +-DBL_MAX, +0.0 (no -0.0, no NaN)."""
    rng = np.random.default_rng(4)
    special = np.array([-np.inf, np.inf, -1.7976931348623157e308, 1.7976931348623157e308,
                        5e-324, -5e-324, 2.2250738585072014e-308, 0.0, -1.0, 1.0])
    n = 120001
    a = np.where(rng.random(n) < 0.3, special[rng.integers(0, special.size, n)],
                 rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n))
    a = a + 0.0
    assert orc.check_input(a, F64) == -1
    for bc in (0, 500):
        g, _ = gpu_sort(a, F64, base_cap=bc)
        check(orc, a, g, F64)


def test_rec100_extras(ips, orc):
    """Keys equal in bytes 0..8 differing in byte 9; keys differing only in
    byte 0; payloads all distinct so multiset errors are visible."""
    rng = np.random.default_rng(6)
    n = 30001
    r = gen.records100(n, 5)
    r[: n // 2, :9] = 7
    r[n // 2:, 1:10] = 0
    for bc in (0, 300):
        g, _ = gpu_sort(r, REC100, base_cap=bc)
        check(orc, r, g, REC100)


@pytest.mark.parametrize("dtype", [U64, U32, PAIR, QUARTET])
@pytest.mark.parametrize("algo", ["tree", "digit"])
@pytest.mark.parametrize("base_cap", [0, 500])
def test_scratch_is_reported_and_bounded(ips, orc, dtype, algo, base_cap):
    """The peak scratch of a sort never exceeds ips4o_scratch_bytes (deep
    recursion, split base cases, K0m measurement of IPS2Ra included)."""
    n = (1 << 21) + 5
    a = make(dtype, n, 2, "uniform")
    g, st = gpu_sort(a, dtype, base_cap=base_cap, algo=ips.DIGIT if algo == "digit" else ips.TREE)
    assert 0 < st["scratch_bytes"] <= ips.scratch_bytes(n, dtype, base_cap=base_cap), st["scratch_bytes"]
    check(orc, a, g, dtype)


def test_sort_host_end_to_end(ips, orc):
    import torch

    n = 300001
    a = gen.uniform_u64(n, 8)
    h = a.copy()
    st = ips.sort_host(h, U64)          # pageable host memory -> staged copies
    check(orc, a, h, U64)
    pin = torch.from_numpy(a.view(np.int64).copy()).pin_memory()
    ips.sort_host(pin, U64)             # pinned host memory -> direct copies
    check(orc, a, pin.numpy().view(np.uint64), U64)


def test_non_default_stream(ips, orc):
    import torch

    n = 250000
    a = gen.uniform_u64(n, 12)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        t = to_dev(a)
        ips.sort(t, U64)
    s.synchronize()
    check(orc, a, t.cpu().numpy().view(np.uint64), U64)


def test_deterministic(ips):
    a = gen.uniform_u64(1 << 20, 3)
    g1, _ = gpu_sort(a, U64)
    g2, _ = gpu_sort(a, U64)
    assert np.array_equal(g1, g2)


@pytest.mark.parametrize("dtype", [U64, F64, PAIR, U32, QUARTET])
@pytest.mark.parametrize("kind", ["uniform", "dups"])
def test_split_base_case(ips, orc, dtype, kind):
    """K7s: with base_cap M = 1000 and 256 buckets of ~1500 elements, most
    buckets are sorted by the two-pass split base case (M < m <= 2M); any
    that cannot be split go to a next level.  Parity with the oracle."""
    n = 256 * 1500 + 7
    a = make(dtype, n, 33, kind)
    g, st = gpu_sort(a, dtype, base_cap=1000)
    check(orc, a, g, dtype)
    if kind == "uniform":
        # nearly every bucket fits the split (levels beyond 1 hold few tasks)
        assert st["levels"] == 1 or sum(st["tasks_per_level"][1:]) < 32, st["tasks_per_level"]


# ------------------------------------------------- randomized differential test
ALIGN = {U64: 8, F64: 8, PAIR: 16, REC100: 16, U32: 4, QUARTET: 16}  # ips4o.h: minimum alignment per type
ELEM_B = {U64: 8, F64: 8, PAIR: 16, REC100: 100, U32: 4, QUARTET: 32}


def random_case(i):
    """Case i of a fixed, seeded family: element type, size (log-uniform up to
    ~2^21), value distribution, algorithm, options and a buffer offset at the
    type's minimum alignment."""
    rng = np.random.default_rng(9000 + i)
    dtype = [U64, F64, PAIR, REC100, U32, QUARTET][i % 6]
    nmax = 21 if dtype in (U64, F64, U32) else (19 if dtype != REC100 else 17)
    n = int(2 ** rng.uniform(1, nmax)) + int(rng.integers(0, 3))
    kind = ["uniform", "dups", "few", "zipf"][int(rng.integers(0, 4))]
    opts = {}
    if rng.integers(0, 2):
        opts["algo"] = 1  # ips.DIGIT
    if rng.integers(0, 2):
        opts["base_cap"] = int(2 ** rng.uniform(6, 12))
    if rng.integers(0, 3) == 0:
        opts["k_max"] = int(2 ** rng.integers(2, 9))
    if rng.integers(0, 4) == 0:
        opts["skip_prepass"] = True
    off = int(rng.integers(0, 8)) * ALIGN[dtype]
    return dtype, n, kind, opts, off


@pytest.mark.parametrize("i", range(240))
def test_random_cases_with_guard_bands(ips, orc, i):
    """The sort of a sub-range of a larger device buffer, starting at the
    type's minimum alignment (8 B for U64/F64, 4 B for U32, 16 B otherwise):
    the result equals the oracle's and the bytes before and after the range
    are untouched (no write outside [ptr, ptr + n D))."""
    import torch

    dtype, n, kind, opts, off = random_case(i)
    assert ips.DIGIT == 1
    a = make(dtype, n, 7000 + i, kind)
    b = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    G = 4096
    buf = torch.full((G + off + b.size + G,), 0xA5, dtype=torch.uint8, device="cuda")
    lo, hi = G + off, G + off + b.size
    buf[lo:hi].copy_(torch.from_numpy(b))
    st = ips.sort_ex(buf[lo:hi], dtype, **opts)
    torch.cuda.synchronize()
    assert ips.device_status(0) == 0
    assert bool((buf[:lo] == 0xA5).all()) and bool((buf[hi:] == 0xA5).all()), f"guard bands overwritten ({dtype}, n={n}, {opts})"
    g = buf[lo:hi].cpu().numpy().view(a.dtype).reshape(a.shape)
    check(orc, a, g, dtype)
    assert st["levels"] >= 0
