"""Soak run of the CUDA path (opt-in: IPS4O_SOAK_SECONDS=<seconds>, skipped
otherwise so that the default `-m gpu` run keeps its length).

The block permutation and the device-side recursion (Alg. 2,
P:1119-1163) synchronise CTAs through atomics, flags and tail launches whose
interleaving differs from run to run; compute-sanitizer is closed on the GPU
pool (profiles/r2_sanitizer_closed.txt).  This test therefore repeats the
randomized differential family of test_gpu_parity.py far past its 240 fixed
cases (oracle parity + guard bands), and repeats large sorts (2^26 .. 2^30
elements, every key-only type, both algorithms, several distributions)
checking each against the input's sorted order as a library sort on the
device computes it (torch.sort of the order-preserving signed image; test
infrastructure only) — bit-exact, the problem statement P:328-331.
"""
import os
import time

import numpy as np
import pytest

import synth_inputs as gen
from gpu_util import F64, U32, U64
from test_gpu_parity import check, ips, make, random_case  # noqa: F401  (ips: fixture)

pytestmark = pytest.mark.gpu

SOAK_S = float(os.environ.get("IPS4O_SOAK_SECONDS", "0"))
START = int(os.environ.get("IPS4O_SOAK_START", "240"))  # first random case / seed offset of a run
needs_soak = pytest.mark.skipif(SOAK_S <= 0, reason="opt-in: set IPS4O_SOAK_SECONDS")


@needs_soak
def test_soak_random_cases(ips, orc):
    """Random cases START, START + 1, ... (default 240) for half of the soak time."""
    import torch

    t_end = time.time() + SOAK_S / 2
    i = START
    while time.time() < t_end:
        dtype, n, kind, opts, off = random_case(i)
        a = make(dtype, n, 7000 + i, kind)
        b = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
        G = 4096
        buf = torch.full((G + off + b.size + G,), 0xA5, dtype=torch.uint8, device="cuda")
        lo, hi = G + off, G + off + b.size
        buf[lo:hi].copy_(torch.from_numpy(b))
        ips.sort_ex(buf[lo:hi], dtype, **opts)
        torch.cuda.synchronize()
        assert ips.device_status(0) == 0, (i, dtype, n, kind, opts)
        assert bool((buf[:lo] == 0xA5).all()) and bool((buf[hi:] == 0xA5).all()), (i, dtype, n, kind, opts)
        g = buf[lo:hi].cpu().numpy().view(a.dtype).reshape(a.shape)
        check(orc, a, g, dtype)
        i += 1
    print(f"soak: random cases {START}..{i - 1} pass", flush=True)


def _ordered_i64(t, dtype):
    """Order-preserving signed 64-bit image of the keys on the device
    (test-side check only; the product's own key maps live in csrc/)."""
    import torch

    if dtype == U32:
        return t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    x = t.view(torch.int64)
    if dtype == U64:
        return x ^ (-(1 << 63))
    # F64 (no NaNs in the generators): negative doubles reverse their order
    return torch.where(x < 0, x ^ 0x7FFFFFFFFFFFFFFF, x)


BIG = [
    (U64, "uniform_u64"), (F64, "exponential_f64"), (U32, "uniform_u32"), (U64, "zipf_u64"),
    (U64, "twodup_u64"), (F64, "almost_sorted_f64"), (U64, "rootdup_u64"), (U64, "eightdup_u64"),
]


@needs_soak
def test_soak_large_sorts(ips):
    """Large sorts for the other half of the soak time: sizes 2^26 .. 2^30
    (+ a ragged tail), both algorithms, compared element by element with a
    library sort of the same device data."""
    import torch

    t_end = time.time() + SOAK_S / 2
    it = 0
    sh = START % 7  # another run pairs sizes and distributions differently
    while time.time() < t_end:
        dtype, dist = BIG[it % len(BIG)]
        lg = [30, 26, 28, 27, 29][(it + sh) % 5]
        n = (1 << lg) - (it * 977) % 4099
        a = getattr(gen, dist)(n, 260 + START + it)
        t = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1)).cuda()
        want = torch.sort(_ordered_i64(t, dtype)).values
        for rep in range(4):  # the same input again (twice per algorithm): the interleavings differ
            w = t.clone()
            st = ips.sort_ex(w, dtype, algo=(it + rep) % 2)
            torch.cuda.synchronize()
            assert ips.device_status(0) == 0, (it, dist, n)
            assert torch.equal(_ordered_i64(w, dtype), want), (it, rep, dist, n, st.get("levels"))
            del w
        print(f"soak: {dist} n={n} x4 ok", flush=True)
        del t, want
        it += 1
    print(f"soak: {it} large inputs x 4 sorts pass", flush=True)


def _mix_sum(x64):
    """Two wrapping 64-bit sums of mixed keys (multiset fingerprints)."""
    a = x64 * (-7046029254386353131)  # 0x9E3779B97F4A7C15 as int64, wraps
    a = a ^ (a >> 29)
    return int((a * (-4658895280553007687)).sum().item()), int((x64 * x64 + x64).sum().item())


@needs_soak
@pytest.mark.parametrize("dtype", [U32, U64])
def test_near_maximum_n(ips, dtype):
    """The largest n the ABI accepts is 2^32 - 1 (ips4o.h): a sort of
    n = 2^32 - 4097 elements (16 GiB of U32, 32 GiB of U64), checked by
    properties that hold at any size — non-decreasing, and the multiset kept
    (two independent wrapping fingerprints, taken chunk by chunk before and
    after).  The input is a 2^28-element seeded stream repeated 16 times, each
    copy xored with its own constant (built on the device, test side)."""
    import torch

    n = (1 << 32) - 4097
    tdt = torch.int32 if dtype == U32 else torch.int64
    base = gen.uniform_u32(1 << 28, 77) if dtype == U32 else gen.uniform_u64(1 << 28, 77)
    hb = torch.from_numpy(base.view(np.int32 if dtype == U32 else np.int64)).cuda()
    t = torch.empty(n, dtype=tdt, device="cuda")
    C = 1 << 28
    for c in range(16):
        m = min(C, n - c * C)
        t[c * C:c * C + m] = hb[:m] ^ (c * 0x01234567 if dtype == U32 else c * 0x0123456789ABCDE)
    del hb

    def prints(v):
        f0 = f1 = 0
        for c in range(0, n, C):
            x = v[c:c + C]
            x = (x.to(torch.int64) & 0xFFFFFFFF) if dtype == U32 else x
            a, b = _mix_sum(x)
            f0, f1 = (f0 + a) & (2**64 - 1), (f1 + b) & (2**64 - 1)
        return f0, f1

    before = prints(t)
    st = ips.sort_ex(t.view(torch.uint8), dtype)
    torch.cuda.synchronize()
    assert ips.device_status(0) == 0
    assert prints(t) == before, "multiset changed"
    for c in range(0, n, C):
        x = t[c:min(n, c + C + 1)]
        x = (x.to(torch.int64) & 0xFFFFFFFF) if dtype == U32 else (x ^ (-(1 << 63)))
        assert bool((x[1:] >= x[:-1]).all()), f"not sorted in chunk {c // C}"
    print(f"near-max n={n} dtype {dtype}: levels {st['levels']} tasks {st['tasks_per_level']}", flush=True)
