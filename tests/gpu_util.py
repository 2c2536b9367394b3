"""Helpers for the GPU tests: move numpy arrays through the C ABI and back."""
import numpy as np

U64, F64, PAIR, REC100, U32, QUARTET = 0, 1, 2, 3, 4, 5
NAMES = {U64: "u64", F64: "f64", PAIR: "pair", REC100: "rec100", U32: "u32", QUARTET: "quartet"}
ELEM = {U64: 8, F64: 8, PAIR: 16, REC100: 100, U32: 4, QUARTET: 32}
KEYB = {U64: 8, F64: 8, PAIR: 8, REC100: 16, U32: 4, QUARTET: 24}


def to_dev(a: np.ndarray):
    import torch

    b = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    t = torch.empty(b.size, dtype=torch.uint8, device="cuda")
    t.copy_(torch.from_numpy(b))
    return t


def from_dev(t, like: np.ndarray) -> np.ndarray:
    import torch

    torch.cuda.synchronize()
    return t.cpu().numpy().view(like.dtype).reshape(like.shape)


def gpu_sort(a: np.ndarray, dtype: int, **opts):
    import paper_2009_13569_b200 as p

    t = to_dev(a)
    st = p.sort_ex(t, dtype, **opts)
    return from_dev(t, a), st


def key_bytes_of(a: np.ndarray, dtype: int) -> np.ndarray:
    """(n, key_bytes) raw keys in the ABI's raw key form (8 B or 10+6 B)."""
    E = np.ascontiguousarray(a).view(np.uint8).reshape(-1, ELEM[dtype])
    if dtype == REC100:
        out = np.zeros((E.shape[0], 16), dtype=np.uint8)
        out[:, :10] = E[:, :10]
        return out
    return E[:, :KEYB[dtype]].copy()


def splitters_as_elements(raw: np.ndarray, dtype: int, count: int) -> np.ndarray:
    """Turn raw key bytes from ips4o_step_info into oracle elements."""
    D = ELEM[dtype]
    kb = KEYB[dtype]
    keys = raw.reshape(-1, kb)[:count]
    out = np.zeros((count, D), dtype=np.uint8)
    if dtype == REC100:
        out[:, :10] = keys[:, :10]
    else:
        out[:, :kb] = keys
    return out.reshape(-1)
