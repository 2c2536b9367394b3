"""Pins for the CPU oracle (-m "not gpu").

The oracle is pinned against things other than itself: an independently
written brute-force insertion sort, Python's sorted() with independently
written key functions, numpy's sort, closed forms of the paper's
distributions, a counting sort, and the SPEC/SURVEY worked vectors
(tests/golden/).  Each block names the paper passage it pins.
"""
import itertools
import json
import math
import os
import struct

import numpy as np
import pytest

import synth_inputs as gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U64, F64, PAIR, REC100, U32, QUARTET = 0, 1, 2, 3, 4, 5


# ----------------------------------------------------------------- helpers
def py_key(dtype, rec: bytes):
    """Independent Python key functions (Alg. 3/4)."""
    if dtype == U64:
        return struct.unpack("<Q", rec)[0]
    if dtype == U32:
        return struct.unpack("<I", rec)[0]
    if dtype == QUARTET:
        return struct.unpack("<QQQ", rec[:24])  # Alg. 3: a, then b, then c
    if dtype == F64:
        return struct.unpack("<d", rec)[0]
    if dtype == PAIR:
        return struct.unpack("<Q", rec[:8])[0]
    return rec[:10]  # bytes compare lexicographically as unsigned (R1)


def to_records(arr, dtype):
    D = {U64: 8, F64: 8, PAIR: 16, REC100: 100, U32: 4, QUARTET: 32}[dtype]
    b = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    return [bytes(b[i * D:(i + 1) * D]) for i in range(b.size // D)]


def from_records(recs, dtype):
    if not recs:
        return np.zeros(0, dtype=np.uint8)
    return np.frombuffer(b"".join(recs), dtype=np.uint8).copy()


def battery(dtype, rng):
    """Tiny inputs (length <= 64) per SURVEY 8(c).1 step 3(a)."""
    cases = []
    for n in [0, 1, 2, 3, 5, 8, 16, 31, 33, 64]:
        if dtype in (U64, PAIR):
            keys = [rng.integers(0, 2**64, dtype=np.uint64) for _ in range(n)]
            cases.append(keys)
            cases.append([np.uint64(7)] * n)
            cases.append([np.uint64(i % 2) for i in range(n)])
            cases.append([np.uint64(i) for i in range(n)])
            cases.append([np.uint64(n - i) for i in range(n)])
            cases.append([np.uint64(i % 5) for i in range(n)])
            cases.append([np.uint64(0 if i % 3 else 2**64 - 1) for i in range(n)])
        elif dtype == QUARTET:
            # (a, b, c) triples with many ties in a and in (a, b)
            cases.append([(int(rng.integers(0, 3)), int(rng.integers(0, 3)), int(rng.integers(0, 2**64, dtype=np.uint64)))
                          for _ in range(n)])
            cases.append([(7, 7, 7)] * n)
            cases.append([(i % 2, (i // 2) % 2, i % 3) for i in range(n)])
            cases.append([(0, 0, n - i) for i in range(n)])
            cases.append([(2**64 - 1 if i % 2 else 0, i % 3, 2**64 - 1 - i) for i in range(n)])
        elif dtype == U32:
            cases.append([int(x) for x in rng.integers(0, 2**32, n, dtype=np.uint64)])
            cases.append([7] * n)
            cases.append([i % 2 for i in range(n)])
            cases.append([i for i in range(n)])
            cases.append([n - i for i in range(n)])
            cases.append([0 if i % 3 else 2**32 - 1 for i in range(n)])
        elif dtype == F64:
            special = [-np.inf, np.inf, -1.7976931348623157e308, 1.7976931348623157e308,
                       5e-324, -5e-324, 2.2250738585072014e-308, 0.0, -1.0, 1.0, -0.5, 3.25]
            cases.append(list(rng.standard_normal(n) * 1e3))
            cases.append([2.5] * n)
            cases.append([float(i % 2) - 0.5 for i in range(n)])
            cases.append([float(i) for i in range(n)])
            cases.append([float(-i) for i in range(n)])
            cases.append([special[int(rng.integers(0, len(special)))] for _ in range(n)])
        else:
            recs = []
            for i in range(n):
                r = bytearray(rng.integers(0, 256, 100, dtype=np.uint8).tobytes())
                recs.append(r)
            cases.append(recs)
            # keys equal in bytes 0..8, differing only in byte 9 (values >= 128 too)
            cases.append([bytearray(b"\x05" * 9 + bytes([int(rng.integers(0, 256))])) +
                          bytearray(rng.integers(0, 256, 90, dtype=np.uint8).tobytes())
                          for _ in range(n)])
            # keys differing only in byte 0
            cases.append([bytearray(bytes([int(rng.integers(0, 256))]) + b"\x00" * 9) +
                          bytearray(rng.integers(0, 256, 90, dtype=np.uint8).tobytes())
                          for _ in range(n)])
            # all-zero keys, distinct payloads
            cases.append([bytearray(10) + bytearray(struct.pack("<Q", i) * 11 + b"\x00\x00")
                          for i in range(n)])
    return cases


def case_to_array(case, dtype, rng):
    if dtype == U64:
        return np.array(case, dtype=np.uint64)
    if dtype == U32:
        return np.array(case, dtype=np.uint32)
    if dtype == QUARTET:
        a = np.zeros((len(case), 4), dtype=np.uint64)
        for i, (x, y, z) in enumerate(case):
            a[i, :3] = (x, y, z)
        a[:, 3] = rng.integers(0, 2**64, len(case), dtype=np.uint64)
        return a
    if dtype == F64:
        return np.array(case, dtype=np.float64)
    if dtype == PAIR:
        a = np.zeros((len(case), 2), dtype=np.uint64)
        a[:, 0] = np.array(case, dtype=np.uint64) if case else a[:, 0]
        a[:, 1] = rng.integers(0, 2**64, len(case), dtype=np.uint64)
        return a
    return np.frombuffer(b"".join(bytes(r) for r in case), dtype=np.uint8).copy() if case \
        else np.zeros(0, dtype=np.uint8)


# ----------------------------------------------------------------- mergesort vs brute force
@pytest.mark.parametrize("dtype", [U64, F64, PAIR, REC100, U32, QUARTET])
def test_mergesort_matches_brute_force_and_python_sorted(orc, dtype):
    """output = input in sorted order.  Stable mergesort, stable
    insertion sort and stable Python sorted() must agree byte for byte."""
    rng = np.random.default_rng(100 + dtype)
    for case in battery(dtype, rng):
        a = case_to_array(case, dtype, rng)
        m = orc.sort(a, dtype)
        ins = orc.insertion_sort(a, dtype)
        recs = to_records(a, dtype)
        py = from_records(sorted(recs, key=lambda r: py_key(dtype, r)), dtype)
        assert m.tobytes() == ins.tobytes()
        assert m.tobytes() == py.tobytes()
        assert orc.is_sorted(m, dtype)
        assert orc.multiset_hash(m, dtype) == orc.multiset_hash(a, dtype)


@pytest.mark.parametrize("dtype", [U64, F64, PAIR, REC100, U32, QUARTET])
def test_mergesort_all_sequences_over_three_values(orc, dtype):
    """every permutation of every multiset of size <= 7
    over <= 3 distinct values (= all sequences over {v0,v1,v2})."""
    vals = {U64: [0, 1, 2**63 + 5], F64: [-2.0, 0.0, 3.5], PAIR: [0, 1, 2**63 + 5],
            REC100: [0, 1, 255], U32: [0, 1, 2**31 + 5], QUARTET: [0, 1, 2]}[dtype]
    for n in range(0, 8):
        for seq in itertools.product(range(3), repeat=n):
            if dtype == U64:
                a = np.array([vals[s] for s in seq], dtype=np.uint64)
            elif dtype == U32:
                a = np.array([vals[s] for s in seq], dtype=np.uint32)
            elif dtype == QUARTET:
                # the order lives in c while a and b tie, payload tags in value
                a = np.array([[5, 9, vals[s], i] for i, s in enumerate(seq)], dtype=np.uint64).reshape(-1, 4)
            elif dtype == F64:
                a = np.array([vals[s] for s in seq], dtype=np.float64)
            elif dtype == PAIR:
                a = np.array([[vals[s], i] for i, s in enumerate(seq)], dtype=np.uint64).reshape(-1, 2)
            else:
                a = np.zeros((n, 100), dtype=np.uint8)
                for i, s in enumerate(seq):
                    a[i, 0] = vals[s]  # byte 0 carries the order
                    a[i, 50] = i       # payload tag
            m = orc.sort(a, dtype)
            ins = orc.insertion_sort(a, dtype)
            assert m.tobytes() == ins.tobytes(), (dtype, seq)


# ----------------------------------------------------------------- invariants at size
@pytest.mark.parametrize("dtype", [U64, F64, U32])
def test_mergesort_vs_numpy_sort(orc, dtype):
    """Library cross-check: numpy's sort of the same input."""
    n = 1 << 18
    a = {U64: gen.uniform_u64, F64: gen.exponential_f64, U32: gen.uniform_u32}[dtype](n, 11)
    m = orc.sort(a, dtype)
    assert np.array_equal(m, np.sort(a, kind="stable"))


def test_mergesort_pairs_exact_multiset_pin(orc):
    """pairs with value = i; after sorting, values are a
    permutation of 0..n-1 and g[j] == in[g[j].value]; keys non-decreasing."""
    n = 1 << 16
    a = gen.pairs(n, 4)
    g = orc.sort(a, PAIR)
    vals = g[:, 1].astype(np.int64)
    assert np.array_equal(np.sort(vals), np.arange(n))
    assert np.array_equal(a[vals], g)
    assert np.all(g[1:, 0] >= g[:-1, 0])


def test_mergesort_records_vs_python(orc):
    n = 3000
    a = gen.records100(n, 5)
    g = orc.sort(a, REC100)
    recs = [bytes(r) for r in a]
    py = np.frombuffer(b"".join(sorted(recs, key=lambda r: r[:10])), dtype=np.uint8).reshape(n, 100)
    assert np.array_equal(g, py)


# ----------------------------------------------------------------- closed forms
def test_closed_form_rootdup(orc):
    """RootDup A[i] = i mod floor(sqrt n); at n = r^2 the sorted
    output is out[j] = floor(j / r)."""
    n = 1 << 16
    r = math.isqrt(n)
    g = orc.sort(gen.rootdup_u64(n), U64)
    assert np.array_equal(g, (np.arange(n, dtype=np.uint64) // np.uint64(r)))


def test_closed_form_almost_sorted(orc):
    """AlmostSorted = 0..n-1 with adjacent swaps: sorted output is out[j] = j."""
    n = 1 << 16
    g = orc.sort(gen.almost_sorted_f64(n, 2), F64)
    assert np.array_equal(g, np.arange(n, dtype=np.float64))


def test_closed_form_sorted_reverse_ones(orc):
    n = 1 << 15
    s = gen.sorted_f64(n, 2)
    assert np.array_equal(orc.sort(s, F64), s)
    assert np.array_equal(orc.sort(s[::-1].copy(), F64), s)
    o = gen.ones_u64(n)
    assert np.array_equal(orc.sort(o, U64), o)


@pytest.mark.parametrize("name", ["twodup_u64", "zipf_u64", "rootdup_u64", "eightdup_u64", "zero_u64"])
def test_counting_sort_pin(orc, name):
    """Reduction to counting sort: values are small integers."""
    n = 1 << 17
    a = gen.generate(name, n, 3)
    counts = np.bincount(a.astype(np.int64))
    expect = np.repeat(np.arange(counts.size, dtype=np.uint64), counts)
    assert np.array_equal(orc.sort(a, U64), expect)


# ----------------------------------------------------------------- parity checker
def test_parity_checker_rules(orc):
    """keys identical + equal-key runs as multisets."""
    o = np.array([[1, 10], [2, 20], [2, 21], [2, 22], [5, 50]], dtype=np.uint64)
    g = np.array([[1, 10], [2, 22], [2, 20], [2, 21], [5, 50]], dtype=np.uint64)
    assert orc.parity(g, o, PAIR) == -1          # permuted equal-key run is fine
    bad = g.copy()
    bad[1, 1] = 99                                # payload changed inside a run
    assert orc.parity(bad, o, PAIR) == 1
    bad = g.copy()
    bad[4, 0] = 6                                 # key changed
    assert orc.parity(bad, o, PAIR) == 4
    bad = g.copy()
    bad[0, 1] = 11                                # singleton run payload changed
    assert orc.parity(bad, o, PAIR) == 0
    u = np.array([1, 2, 3], dtype=np.uint64)
    assert orc.parity(u, u.copy(), U64) == -1
    assert orc.parity(np.array([1, 3, 2], dtype=np.uint64), u, U64) == 1


def test_check_input_rejects_nan_and_negative_zero(orc):
    assert orc.check_input(np.array([1.0, 2.0, 0.0]), F64) == -1
    assert orc.check_input(np.array([1.0, np.nan]), F64) == 1
    assert orc.check_input(np.array([1.0, 2.0, -0.0]), F64) == 2


# ----------------------------------------------------------------- classifier / tree
def _u64s(xs):
    return np.array(xs, dtype=np.uint64)


def test_golden_spec_build_tree(orc):
    g = json.load(open(os.path.join(GOLD, "spec_vectors.json")))
    for v in g["build_tree"]:
        tree, spl, l = orc.build_tree(_u64s(v["splitters"]), U64)
        assert l == v["l"], v["cite"]
        assert tree.view(np.uint64).tolist() == v["tree"], v["cite"]
        assert spl.view(np.uint64).tolist() == v["splitter"], v["cite"]


def test_golden_spec_classify(orc):
    g = json.load(open(os.path.join(GOLD, "spec_vectors.json")))
    for v in g["classify"]:
        tree, spl, l = orc.build_tree(_u64s(v["splitters"]), U64)
        for e, want in v["cases"]:
            x = _u64s([e])
            assert orc.classify_linear(spl, l, v["equality"], U64, x) == want, v["cite"]
            assert orc.classify_tree(tree, spl, l, v["equality"], U64, x) == want, v["cite"]


def test_golden_spec_boundaries_and_splitters(orc):
    g = json.load(open(os.path.join(GOLD, "spec_vectors.json")))
    for v in g["boundaries"]:
        E, d = orc.boundaries(v["counts"], v["b"])
        assert E.tolist() == v["E"] and d.tolist() == v["d"], v["cite"]
    for v in g["select_splitters"]:
        sp, eq, kf = orc.select_splitters(_u64s(v["sample"]), v["k"], 256, U64)
        assert sp.view(np.uint64).tolist() == v["splitters"], v["cite"]
        assert eq == v["equality"], v["cite"]
    for v in g["radix_digit"]:
        assert orc.radix_digit(U64, _u64s([v["key"]]), v["shift"], v["bits"]) == v["digit"]


def test_golden_survey_worked_example(orc):
    g = json.load(open(os.path.join(GOLD, "survey_worked_example.json")))
    A = _u64s(g["A"])
    tree, spl, l = orc.build_tree(_u64s(g["splitters"]), U64)
    assert tree.view(np.uint64).tolist() == g["tree"]
    assert spl.view(np.uint64).tolist() == g["splitter"]
    for key, eq in (("no_equality", False), ("equality", True)):
        ids = [orc.classify_tree(tree, spl, l, eq, U64, A[i:i + 1]) for i in range(A.size)]
        assert ids == g[key]["ids"]
        h = orc.histogram(A, U64, spl, l, eq)
        assert h.tolist() == g[key]["counts"]
        E, d = orc.boundaries(h, g["b"])
        assert E.tolist() == g[key]["E"] and d.tolist() == g[key]["d"]
    # the partition of the no-equality case, as multisets
    ids = g["no_equality"]["ids"]
    for j, want in enumerate(g["no_equality"]["buckets"]):
        assert sorted(int(A[i]) for i in range(A.size) if ids[i] == j) == want


def _py_bucket(splitters_padded, e, equality):
    """Independent brute force of P:432-437 via bisect (leaf = #{s_j < e})."""
    import bisect
    s = len(splitters_padded) - 1  # padded list has s+1 entries
    leaf = bisect.bisect_left(splitters_padded[:s], e)
    if not equality:
        return leaf
    return 2 * leaf + 1 - (1 if e < splitters_padded[leaf] else 0)


def test_classifier_random_vs_bisect_and_tree(orc):
    """SPEC S:156 property: 10^4 random (splitter set, element) pairs; the
    literal Alg. 1 walk, the linear definition and a bisect brute force agree;
    classification is monotone; equality buckets hold only equal keys."""
    rng = np.random.default_rng(7)
    for trial in range(200):
        u = int(rng.integers(1, 40))
        sp = np.unique(rng.integers(0, 100, u).astype(np.uint64))
        tree, spl, l = orc.build_tree(sp, U64)
        padded = spl.view(np.uint64).tolist()
        es = rng.integers(0, 110, 50).astype(np.uint64)
        for eq in (False, True):
            prev = None
            for e in np.sort(es):
                x = _u64s([e])
                a = orc.classify_linear(spl, l, eq, U64, x)
                b = orc.classify_tree(tree, spl, l, eq, U64, x)
                c = _py_bucket(padded, int(e), eq)
                assert a == b == c
                if prev is not None:
                    assert a >= prev
                prev = a
                if eq and a % 2 == 1 and a // 2 < (1 << l) - 1:
                    assert int(e) == padded[a // 2]


def test_classifier_f64_and_rec100_use_the_dtype_order(orc):
    rng = np.random.default_rng(8)
    sp = np.sort(rng.standard_normal(7))
    tree, spl, l = orc.build_tree(sp, F64)
    padded = spl.view(np.float64).tolist()
    for e in rng.standard_normal(500) * 2:
        x = np.array([e])
        assert orc.classify_tree(tree, spl, l, True, F64, x) == _py_bucket(padded, float(e), True)
    # REC100: keys are 10-byte strings; bytes >= 128 must order above bytes < 128
    keys = sorted({bytes(rng.integers(0, 256, 10, dtype=np.uint8)) for _ in range(5)})
    recs = np.zeros((len(keys), 100), dtype=np.uint8)
    for i, k in enumerate(keys):
        recs[i, :10] = np.frombuffer(k, dtype=np.uint8)
    tree, spl, l = orc.build_tree(recs, REC100)
    padded = [bytes(spl.reshape(-1, 100)[i, :10]) for i in range((1 << l))]
    for _ in range(300):
        e = np.zeros(100, dtype=np.uint8)
        e[:10] = rng.integers(0, 256, 10, dtype=np.uint8)
        if rng.random() < 0.3:
            e[:10] = np.frombuffer(keys[int(rng.integers(0, len(keys)))], dtype=np.uint8)
        assert orc.classify_tree(tree, spl, l, True, REC100, e) == \
            _py_bucket(padded, bytes(e[:10]), True)


def test_select_splitters_equality_budget(orc):
    """R10 (DESIGN): with equality buckets the u unique splitters must leave
    2*(u+1) <= kidx_max bucket indices.  The u - (kidx_max/2 - 1) surplus
    splitters are dropped one at a time, fewest picks first (ties: the
    smaller), never two neighbours; if that many cannot be dropped, k is
    halved.  Expected splitters are worked out by hand in the comments."""
    m = 256 * 4
    # 200 zeros, then 1..824: picks at 4j+3 give 0 (50 times) and 4i for
    # i = 1..205 (once each): u = 206, 79 too many -> drop i = 1, 3, .., 157
    sample = np.sort(np.concatenate([np.zeros(200, dtype=np.uint64),
                                     np.arange(1, m - 199, dtype=np.uint64)]))
    sp, eq, kf = orc.select_splitters(sample, 256, 256, U64)
    want = [0] + [4 * i for i in range(2, 159, 2)] + [4 * i for i in range(159, 206)]
    assert kf == 256 and eq and sp.view(np.uint64).tolist() == want
    # 128 unique picks (one over the budget): 0 picked 128 times, 1..127 once
    # each -> the first of the lightest, 1, is dropped
    s2 = np.sort(np.concatenate([np.zeros(512, dtype=np.uint64), np.repeat(np.arange(1, 129, dtype=np.uint64), 4)]))
    sp3, eq3, kf3 = orc.select_splitters(s2, 256, 256, U64)
    got = sp3.view(np.uint64).tolist()
    assert eq3 and kf3 == 256 and got == [0] + list(range(2, 128)), got
    # budget 64 (31 equality splitters): k = 256 has u = 206 (at most 103
    # droppable), k = 128 has u = 103 (51 droppable, 72 needed); k = 64 picks
    # 0 (12 times) and 16i - 8 for i = 1..51: drop i = 1, 3, .., 41
    sp4, eq4, kf4 = orc.select_splitters(sample, 256, 64, U64)
    want4 = [0] + [16 * i - 8 for i in range(2, 43, 2)] + [16 * i - 8 for i in range(43, 52)]
    assert kf4 == 64 and eq4 and sp4.view(np.uint64).tolist() == want4, sp4.view(np.uint64).tolist()
    sp2, eq2, kf2 = orc.select_splitters(np.arange(m, dtype=np.uint64), 256, 256, U64)
    assert kf2 == 256 and not eq2 and sp2.size // 8 == 255


def test_radix_digit_quartet(orc):
    """IPS2Ra digit of the 192-bit Quartet key a*2^128 + b*2^64 + c (Alg. 3
    order): compared with Python integers."""
    rng = np.random.default_rng(6)
    for _ in range(200):
        e = rng.integers(0, 2**64, 4, dtype=np.uint64)
        big = (int(e[0]) << 128) | (int(e[1]) << 64) | int(e[2])
        for sh, bits in [(0, 8), (60, 8), (120, 8), (184, 8), (127, 3)]:
            assert orc.radix_digit(QUARTET, e, sh, bits) == (big >> sh) & ((1 << bits) - 1)


def test_radix_digit_u32(orc):
    """IPS2Ra digit of 32-bit keys: bits [shift, shift+bits)."""
    rng = np.random.default_rng(5)
    for x in rng.integers(0, 2**32, 200, dtype=np.uint64):
        a = np.array([x], dtype=np.uint32)
        for sh, bits in [(0, 8), (24, 8), (13, 7), (31, 1)]:
            assert orc.radix_digit(U32, a, sh, bits) == (int(x) >> sh) & ((1 << bits) - 1)


def test_radix_digit_orders(orc):
    """P:1688 extractor: the full 64/80-bit digit sequence orders like the
    dtype's comparator (f64 via the oracle's own IEEE argument)."""
    rng = np.random.default_rng(9)
    xs = np.concatenate([rng.standard_normal(300) * 1e5, [0.0, -np.inf, np.inf, 5e-324, -5e-324]])
    keyed = [((orc.radix_digit(F64, np.array([x]), 32, 32) << 32) |
              orc.radix_digit(F64, np.array([x]), 0, 32), x) for x in xs]
    assert [x for _, x in sorted(keyed)] == sorted(xs.tolist())
    for _ in range(200):
        r = np.zeros(100, dtype=np.uint8)
        r[:10] = rng.integers(0, 256, 10, dtype=np.uint8)
        big = int.from_bytes(bytes(r[:10]), "big")
        sh = int(rng.integers(0, 72))
        assert orc.radix_digit(REC100, r, sh, 8) == (big >> sh) & 255


def test_sample_index_range_and_uniformity(orc):
    """R8 generator: indices fall in [begin, begin+size) and are uniform."""
    begin, size = 1000, 97
    hits = np.zeros(size)
    for j in range(20000):
        i = orc.sample_index(5, 1, begin, size, j)
        assert begin <= i < begin + size
        hits[i - begin] += 1
    exp = 20000 / size
    chi2 = float(((hits - exp) ** 2 / exp).sum())
    assert chi2 < 200  # 96 dof; mean 96, 5-sigma ~ 165
    assert orc.sample_index(5, 1, begin, size, 3) == orc.sample_index(5, 1, begin, size, 3)
    assert orc.sample_index(5, 1, begin, size, 3) != orc.sample_index(5, 2, begin, size, 3) or \
        orc.sample_index(5, 1, begin, size, 4) != orc.sample_index(5, 2, begin, size, 4)


def test_sample_tree_subroracle_is_consistent(orc):
    """K1 sub-oracle end to end on a duplicate-heavy task: the tree it builds
    classifies the task consistently with the bisect brute force."""
    a = gen.rootdup_u64(1 << 14)
    st = orc.sample_tree(a, U64, 0, a.size, seed=1, level=0, k=64, alpha=4, kidx_max=256)
    padded = st["splitter"].view(np.uint64).tolist()
    for x in a[:500]:
        assert orc.classify_tree(st["tree"], st["splitter"], st["l"], st["equality"], U64,
                                 np.array([x])) == _py_bucket(padded, int(x), st["equality"])


# ----------------------------------------------------------------- R8 pin
M64 = (1 << 64) - 1


def _py_mix(z):
    """SplitMix64 finaliser (Steele, Lea, Flood), written out with Python ints."""
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _py_sample_index(seed, level, begin, size, j):
    """DESIGN R8 transcribed independently of oracle.c:
    base = mix(seed + g(level+1)) ^ mix(begin + g(size+1)), u_j = mix(base + g(j+1)),
    index = begin + floor(u_j * size / 2^64)."""
    g = 0x9E3779B97F4A7C15
    base = _py_mix((seed + g * (level + 1)) & M64) ^ _py_mix((begin + g * (size + 1)) & M64)
    u = _py_mix((base + g * (j + 1)) & M64)
    return begin + ((u * size) >> 64)


def test_sample_index_matches_r8_transcription(orc):
    """orc_sample_index equals an independent Python transcription of R8 on
    every argument corner (large seeds, levels, 2^32-sized tasks, j wrap)."""
    cases = [(0, 0, 0, 1, 0), (1, 0, 0, 2, 0), (42, 0, 0, 1 << 30, 5), (0x1F4A2C7, 1, 123456, 4194304, 16383),
             (M64, 7, (1 << 40) + 3, (1 << 32) - 1, (1 << 20) + 1), (5, 1, 1000, 97, 3), (5, 2, 1000, 97, 3)]
    rng = np.random.default_rng(11)
    for _ in range(300):
        cases.append((int(rng.integers(0, 1 << 63)) * 2 + 1, int(rng.integers(0, 64)), int(rng.integers(0, 1 << 40)),
                      int(rng.integers(1, 1 << 34)), int(rng.integers(0, 1 << 20))))
    for c in cases:
        assert orc.sample_index(*c) == _py_sample_index(*c), c


# ----------------------------------------------------------------- checkers reject
@pytest.mark.parametrize("dtype", [U64, F64, PAIR, REC100, U32, QUARTET])
def test_multiset_hash_and_is_sorted_reject_changes(orc, dtype):
    """The invariant checkers are not vacuous: a changed byte changes the
    multiset hash, a swapped pair of distinct keys is not sorted, and the
    parity checker reports the first differing element."""
    D = {U64: 8, F64: 8, PAIR: 16, REC100: 100, U32: 4, QUARTET: 32}[dtype]
    rng = np.random.default_rng(dtype + 3)
    n = 257
    a = rng.integers(0, 256, n * D, dtype=np.uint8)
    if dtype == F64:  # finite, non-negative doubles (no NaN / -0.0, R2)
        a = rng.random(n).view(np.uint8)
    s = orc.sort(a, dtype)
    assert orc.is_sorted(s, dtype)
    h = orc.multiset_hash(a, dtype)
    assert orc.multiset_hash(s, dtype) == h
    for pos in [0, D - 1, 17 * D + 3, n * D - 1]:
        b = a.copy()
        b[pos] ^= 0x10
        assert orc.multiset_hash(b, dtype) != h, pos
    # a record duplicated over another changes the multiset
    b = a.copy()
    b[5 * D:6 * D] = b[9 * D:10 * D]
    assert orc.multiset_hash(b, dtype) != h
    # swap two adjacent elements of the sorted output with distinct keys
    E = s.reshape(n, D).copy()
    for i in range(n - 1):
        if orc.less(dtype, E[i], E[i + 1]):
            E[[i, i + 1]] = E[[i + 1, i]]
            break
    bad = E.reshape(-1)
    assert not orc.is_sorted(bad, dtype)
    assert orc.parity(bad, s, dtype) == i
    # a payload change inside an equal-key run is a multiset error for parity
    if dtype in (PAIR, REC100, QUARTET):
        P = s.reshape(n, D).copy()
        P[n // 2, D - 1] ^= 1
        assert orc.parity(P.reshape(-1), s, dtype) != -1


def test_log_digit_pins(orc):
    """orc_log_digit (DESIGN R33) against what its definition fixes, none of it
    through the oracle's own formula: the identity below 2^(M+1); brute force
    over every offset below 2^14 that the mapping is monotone, hits every slot
    (steps of 0 or 1), and gives every octave [2^e, 2^(e+1)), e > M, exactly
    2^M slots of 2^(e-M) offsets each; hand-computed values; and the slot
    count of a range, 2^M (bitlen(R) - M + 1) slots up to the octave of R."""
    for M in range(1, 8):
        prev = -1
        per_slot = {}
        for d in range(1 << 14):
            q = orc.log_digit(d, M)
            if d < (2 << M):
                assert q == d
            assert q - prev in (0, 1)
            prev = q
            per_slot[q] = per_slot.get(q, 0) + 1
        for e in range(M + 1, 14):
            slots = sorted({orc.log_digit(d, M) for d in range(1 << e, 2 << e)})
            assert len(slots) == 1 << M
            assert all(per_slot[q] == 1 << (e - M) for q in slots)
    # by hand, M = 3: d = 16..31 is octave 4 (slot width 2): 16 -> 16, 17 -> 16,
    # 30 -> 23; octave 5 (width 4) starts at slot 24: 32 -> 24, 63 -> 31;
    # d = 2^40 opens octave 40: 8 * (40 - 3 + 1) = 304
    assert [orc.log_digit(d, 3) for d in (15, 16, 17, 30, 31, 32, 35, 36, 63, 64)] == [15, 16, 16, 23, 23, 24, 24, 25, 31, 32]
    assert orc.log_digit(1 << 40, 3) == 304
    assert orc.log_digit((1 << 41) - 1, 3) == 311
    # M = 1: two slots per octave; 2^63 opens the last octave: 2 * (63 - 1 + 1) = 126
    assert orc.log_digit(1 << 63, 1) == 126 and orc.log_digit((1 << 64) - 1, 1) == 127
