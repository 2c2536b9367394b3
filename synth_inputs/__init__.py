"""Seeded synthetic inputs in the paper's distributions.

This module serves BOTH the oracle tests and the CUDA path's tests/bench.  It
holds none of the method's arithmetic: no sorting, no classification, no
partitioning -- only counter-based random numbers and the closed-form
generators.  Recipe:

* RNG: SplitMix64 used counter-style, x_i = mix(seed + (i+1)*GAMMA).
* Uniform u64 ........ A[i] = x_i
* Uniform f64 ........ (x_i >> 11) * 2^-53 in [0, 1)
* Exponential f64 .... 0.0 - log(((x_i >> 11) + 1) * 2^-53)  (lambda = 1; +0.0, never -0.0)
* AlmostSorted f64 ... A[i] = i, then for s < floor(sqrt n): j = x_s mod (n-1),
                       swap A[j], A[j+1] in sequence          (BJ)
* Sorted f64 ......... A[i] = (i + (x_i >> 11) * 2^-53) / n  (a sorted Uniform draw,
                       strictly increasing, built without sorting)
* ReverseSorted f64 .. Sorted reversed
* RootDup u64 ........ A[i] = i mod floor(sqrt n)
* TwoDup u64 ......... A[i] = (i^2 + n/2) mod n              (reading R15)
* Zipf u64 ........... rank r in [1, 2^20] with P(r) ~ 1/r (s = 1), by inverse CDF
* Ones u64 ........... A[i] = 1
* Pair ............... {key = x_i, value = i}
* 100B ............... record i = first 100 bytes of x_{13i} .. x_{13i+12}
                       (little-endian); key = bytes 0..9
"""
from __future__ import annotations

import math

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
CHUNK = 1 << 24

SEEDS = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5, "head": 42}


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def splitmix(seed: int, start: int, count: int) -> np.ndarray:
    """x_i for i in [start, start+count): mix(seed + (i+1)*GAMMA)."""
    out = np.empty(count, dtype=np.uint64)
    s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    for c0 in range(0, count, CHUNK):
        c1 = min(count, c0 + CHUNK)
        i = np.arange(start + c0 + 1, start + c1 + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            out[c0:c1] = _mix(s + i * GAMMA)
    return out


def uniform_u64(n: int, seed: int) -> np.ndarray:
    return splitmix(seed, 0, n)


def _unit(x: np.ndarray) -> np.ndarray:
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_f64(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        out[c0:c1] = _unit(splitmix(seed, c0, c1 - c0))
    return out


def exponential_f64(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        u = ((splitmix(seed, c0, c1 - c0) >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
        out[c0:c1] = 0.0 - np.log(u)
    return out


def almost_sorted_f64(n: int, seed: int) -> np.ndarray:
    a = np.arange(n, dtype=np.float64)
    if n < 2:
        return a
    swaps = math.isqrt(n)
    js = (splitmix(seed, 0, swaps) % np.uint64(n - 1)).astype(np.int64)
    for j in js.tolist():
        a[j], a[j + 1] = a[j + 1], a[j]
    return a


def sorted_f64(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        frac = _unit(splitmix(seed, c0, c1 - c0))
        out[c0:c1] = (np.arange(c0, c1, dtype=np.float64) + frac) / float(n)
    return out


def reverse_sorted_f64(n: int, seed: int) -> np.ndarray:
    return sorted_f64(n, seed)[::-1].copy()


def rootdup_u64(n: int, seed: int = 0) -> np.ndarray:
    r = max(1, math.isqrt(n))
    return (np.arange(n, dtype=np.uint64) % np.uint64(r)).astype(np.uint64)


def twodup_u64(n: int, seed: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    nn = np.uint64(max(n, 1))
    half = np.uint64(n // 2)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        i = np.arange(c0, c1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            out[c0:c1] = (i * i + half) % nn
    return out


ZIPF_VALUES = 1 << 20


def zipf_u64(n: int, seed: int, values: int = ZIPF_VALUES) -> np.ndarray:
    w = 1.0 / np.arange(1, values + 1, dtype=np.float64)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    out = np.empty(n, dtype=np.uint64)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        u = _unit(splitmix(seed, c0, c1 - c0))
        r = np.searchsorted(cdf, u, side="right") + 1
        out[c0:c1] = np.minimum(r, values).astype(np.uint64)
    return out


def ones_u64(n: int, seed: int = 0) -> np.ndarray:
    return np.ones(n, dtype=np.uint64)


def zero_u64(n: int, seed: int = 0) -> np.ndarray:
    """Zero: just zeros."""
    return np.zeros(n, dtype=np.uint64)


def eightdup_u64(n: int, seed: int = 0) -> np.ndarray:
    """EightDup: A[i] = (i^8 + n/2) mod n, i^8 mod n by repeated
    squaring mod n (every square < 2^60 for n <= 2^30)."""
    out = np.empty(n, dtype=np.uint64)
    nn = np.uint64(max(n, 1))
    half = np.uint64(n // 2)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        x = np.arange(c0, c1, dtype=np.uint64) % nn
        for _ in range(3):
            x = (x * x) % nn
        out[c0:c1] = (x + half) % nn
    return out


def uniform_u32(n: int, seed: int) -> np.ndarray:
    """32-bit unsigned keys: the high halves of the SplitMix64 stream."""
    out = np.empty(n, dtype=np.uint32)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        out[c0:c1] = (splitmix(seed, c0, c1 - c0) >> np.uint64(32)).astype(np.uint32)
    return out


def pairs(n: int, seed: int) -> np.ndarray:
    """(n, 2) uint64: column 0 = key, column 1 = value = i."""
    out = np.empty((n, 2), dtype=np.uint64)
    out[:, 0] = splitmix(seed, 0, n)
    out[:, 1] = np.arange(n, dtype=np.uint64)
    return out


def quartets(n: int, seed: int) -> np.ndarray:
    """(n, 4) uint64 Quartet elements {a, b, c, value=i}.  a takes
    only 2^12 values and b 2^20, so the lexicographic order is decided by b
    and by c often (Alg. 3)."""
    out = np.empty((n, 4), dtype=np.uint64)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        w = splitmix(seed, 3 * c0, 3 * (c1 - c0)).reshape(c1 - c0, 3)
        out[c0:c1, 0] = w[:, 0] >> np.uint64(52)
        out[c0:c1, 1] = w[:, 1] >> np.uint64(44)
        out[c0:c1, 2] = w[:, 2]
        out[c0:c1, 3] = np.arange(c0, c1, dtype=np.uint64)
    return out


def records100(n: int, seed: int) -> np.ndarray:
    """(n, 100) uint8 records; key = bytes 0..9."""
    out = np.empty((n, 100), dtype=np.uint8)
    step = max(1, CHUNK // 13)
    for c0 in range(0, n, step):
        c1 = min(n, c0 + step)
        words = splitmix(seed, 13 * c0, 13 * (c1 - c0)).reshape(c1 - c0, 13)
        out[c0:c1] = words.view(np.uint8).reshape(c1 - c0, 104)[:, :100]
    return out


# name -> (dtype name, generator)
DISTRIBUTIONS = {
    "uniform_u64": ("u64", uniform_u64),
    "uniform_f64": ("f64", uniform_f64),
    "exponential_f64": ("f64", exponential_f64),
    "almost_sorted_f64": ("f64", almost_sorted_f64),
    "sorted_f64": ("f64", sorted_f64),
    "reverse_sorted_f64": ("f64", reverse_sorted_f64),
    "rootdup_u64": ("u64", rootdup_u64),
    "twodup_u64": ("u64", twodup_u64),
    "zipf_u64": ("u64", zipf_u64),
    "ones_u64": ("u64", ones_u64),
    "zero_u64": ("u64", zero_u64),
    "eightdup_u64": ("u64", eightdup_u64),
    "uniform_u32": ("u32", uniform_u32),
    "quartets": ("quartet", quartets),
    "pairs": ("pair", pairs),
    "records100": ("rec100", records100),
}

# BASELINE.json configs (index -> list of (distribution, n, seed))
CONFIGS = {
    0: [("uniform_u64", 1 << 20, 1)],
    1: [("uniform_f64", 1 << 28, 2), ("exponential_f64", 1 << 28, 2),
        ("almost_sorted_f64", 1 << 28, 2), ("sorted_f64", 1 << 28, 2),
        ("reverse_sorted_f64", 1 << 28, 2)],
    2: [("rootdup_u64", 1 << 30, 3), ("twodup_u64", 1 << 30, 3),
        ("zipf_u64", 1 << 30, 3), ("ones_u64", 1 << 30, 3)],
    3: [("pairs", 1 << 28, 4)],
    4: [("records100", 1 << 24, 5)],
}
HEADLINE = ("uniform_u64", 1 << 30, 42)


def generate(name: str, n: int, seed: int) -> np.ndarray:
    return DISTRIBUTIONS[name][1](n, seed)
