"""Multi-GPU samplesort (paper_2009_13569_b200.distributed).

CPU (gloo, world sizes 2 and 3): the exchange logic of ``sample_sort`` -- the
sample all-gather, empty shards, the size and element all-to-alls -- with the
local steps done by CPU stand-ins built on the oracle (DESIGN R8 sample
indices, oracle sort, the bucket rule of P:392-394).  The concatenated slices
must equal the oracle's sort of the union.

GPU: the three library steps (ips4o_sample, ips4o_select_splitters,
ips4o_partition_splitters) against the oracle, and the whole algorithm with
p shards on one GPU and the exchange done by slicing (one process; no ranks
waiting on each other)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

U64, PAIR = 0, 2
D = {U64: 8, PAIR: 16}


def _keys(a, dtype):
    return a if dtype == U64 else a[:, 0]


def _view(t, dtype):
    a = t.numpy().view(np.uint64)
    return a if dtype == U64 else a.reshape(-1, 2)


class OracleSteps:
    """CPU stand-ins for the library's local steps (test infrastructure)."""

    def __init__(self):
        import oracle

        self.orc = oracle

    def sample(self, t, dtype, m, seed):
        a = _view(t, dtype)
        n = a.shape[0]
        idx = [self.orc.sample_index(seed, 0, 0, n, j) for j in range(m)]
        return torch.from_numpy(np.ascontiguousarray(a[idx]).view(np.uint8).reshape(-1).copy())

    def select_splitters(self, samples, dtype, parts):
        s = self.orc.sort(_view(samples, dtype), dtype)
        total = s.shape[0]
        pick = [((j + 1) * total) // parts - 1 for j in range(parts - 1)]
        return torch.from_numpy(np.ascontiguousarray(s[pick]).view(np.uint8).reshape(-1).copy())

    def partition(self, t, dtype, splitters, nspl):
        a = _view(t, dtype)
        S = _keys(_view(splitters, dtype), dtype)[:nspl]
        r = np.searchsorted(S, _keys(a, dtype), side="left")  # #{j : S_j < e}: S_{r-1} < e <= S_r
        order = np.argsort(r, kind="stable")
        a[...] = a[order].copy()
        cnt = np.bincount(r, minlength=nspl + 1)
        return [0] + np.cumsum(cnt).tolist()

    def sort(self, t, dtype):
        a = _view(t, dtype)
        a[...] = self.orc.sort(np.ascontiguousarray(a), dtype)


def _shard(rank, world, dtype, n, kind):
    rng = np.random.default_rng(100 + rank)
    if kind == "empty0" and rank == 0:
        n = 0
    if kind == "dups":
        k = rng.integers(0, 5, n).astype(np.uint64)
    else:
        k = rng.integers(0, 2**64, n, dtype=np.uint64)
    if dtype == U64:
        return k
    return np.stack([k, np.arange(n, dtype=np.uint64) + (rank << 40)], axis=1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dtype, n, kind, q):
    import torch.distributed as dist

    from paper_2009_13569_b200 import distributed as dd

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = _shard(rank, world, dtype, n, kind)
    t = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1).copy())
    out, info = dd.sample_sort(t, dtype, steps=OracleSteps(), samples_per_rank=64)
    q.put((rank, out.numpy().tobytes(), info["send"], info["recv"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dtype,n,kind", [(2, U64, 5000, "uniform"), (3, U64, 4001, "dups"),
                                                (3, PAIR, 3000, "empty0"), (2, PAIR, 2500, "dups")])
def test_sample_sort_gloo(world, dtype, n, kind):
    import oracle

    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dtype, n, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    sends = np.array([r[2] for r in res])
    recvs = np.array([r[3] for r in res])
    assert np.array_equal(sends.T, recvs)  # what r sends to s is what s receives from r
    got = np.concatenate([np.frombuffer(r[1], dtype=np.uint64) for r in res])
    union = np.concatenate([_shard(r, world, dtype, n, kind).reshape(-1) for r in range(world)])
    if dtype == PAIR:
        got, union = got.reshape(-1, 2), union.reshape(-1, 2)
    want = oracle.sort(np.ascontiguousarray(union), dtype)
    assert oracle.parity(np.ascontiguousarray(got), want, dtype) == -1
    # each slice holds the keys of one range: slices are ordered and non-overlapping
    slices = [_keys(np.frombuffer(r[1], dtype=np.uint64).reshape(-1, 1 if dtype == U64 else 2), dtype).reshape(-1)
              for r in res]
    for a, b in zip(slices, slices[1:]):
        if a.size and b.size:
            assert a.max() <= b.min()


# ------------------------------------------------------------------ GPU: the library's steps
@pytest.fixture(scope="module")
def ips():
    import paper_2009_13569_b200 as p

    p.load()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [U64, PAIR])
def test_native_sample_matches_r8(ips, dtype):
    import oracle

    n, m, seed = 100003, 777, 0xABCDEF
    a = _shard(0, 1, dtype, n, "uniform")
    t = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1).copy()).cuda()
    out = torch.empty(m * D[dtype], dtype=torch.uint8, device="cuda")
    ips.sample(t, dtype, m, seed, out)
    torch.cuda.synchronize()
    idx = [oracle.sample_index(seed, 0, 0, n, j) for j in range(m)]
    assert np.array_equal(out.cpu().numpy(), np.ascontiguousarray(a[idx]).view(np.uint8).reshape(-1))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [U64, PAIR])
@pytest.mark.parametrize("parts", [2, 5, 64])
def test_native_select_splitters(ips, dtype, parts):
    import oracle

    a = _shard(1, 1, dtype, 4096 + 17, "uniform")
    t = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1).copy()).cuda()
    out = torch.empty((parts - 1) * D[dtype], dtype=torch.uint8, device="cuda")
    ips.select_splitters(t, dtype, parts, out)
    torch.cuda.synchronize()
    s = oracle.sort(a, dtype)
    total = s.shape[0]
    want = s[[((j + 1) * total) // parts - 1 for j in range(parts - 1)]]
    got = out.cpu().numpy().view(np.uint64).reshape(want.shape)
    assert np.array_equal(_keys(got, dtype), _keys(want, dtype))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [U64, PAIR])
@pytest.mark.parametrize("n,nspl,kind", [(1 << 20, 7, "uniform"), (300001, 63, "uniform"), (200000, 3, "dups"),
                                         (5000, 127, "uniform"), (1, 4, "uniform"), (0, 2, "uniform")])
def test_native_partition_splitters(ips, dtype, n, nspl, kind):
    """Range r = [bounds[r], bounds[r+1]) holds exactly the elements e with
    S_{r-1} < e <= S_r and the multiset is unchanged."""
    import oracle

    a = _shard(2, 1, dtype, n, kind)
    rng = np.random.default_rng(7)
    keys = np.sort(rng.integers(0, 2**64, nspl, dtype=np.uint64)) if kind != "dups" else \
        np.array([1, 1, 3][:nspl], dtype=np.uint64)
    spl = keys if dtype == U64 else np.stack([keys, np.zeros_like(keys)], axis=1)
    t = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1).copy()).cuda()
    st = torch.from_numpy(np.ascontiguousarray(spl).view(np.uint8).reshape(-1).copy()).cuda()
    b = ips.partition_splitters(t, dtype, st, nspl)
    g = t.cpu().numpy().view(np.uint64)
    g = g if dtype == U64 else g.reshape(-1, 2)
    assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
    r = np.searchsorted(keys, _keys(a, dtype), side="left")
    assert np.array_equal(np.diff(b), np.bincount(r, minlength=nspl + 1))
    for j in range(nspl + 1):
        seg = _keys(g[b[j]:b[j + 1]], dtype)
        if seg.size:
            assert (j == 0 or seg.min() > keys[j - 1]) and (j == nspl or seg.max() <= keys[j])
    if n > 1:
        assert oracle.parity(oracle.sort(np.ascontiguousarray(g), dtype), oracle.sort(a, dtype), dtype) == -1


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [U64, PAIR])
@pytest.mark.parametrize("p,kind", [(4, "uniform"), (3, "dups"), (8, "uniform")])
def test_native_steps_composed(ips, dtype, p, kind):
    """The whole samplesort with p shards on one GPU: the library's steps, the
    exchange done by slicing in one process."""
    import oracle
    from paper_2009_13569_b200.distributed import NativeSteps, default_samples_per_rank

    S = NativeSteps()
    shards = [_shard(r, p, dtype, 200000 + 777 * r, kind) for r in range(p)]
    ts = [torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1).copy()).cuda() for a in shards]
    m = default_samples_per_rank(sum(a.shape[0] for a in shards), p)
    smp = torch.cat([S.sample(t, dtype, m, 1000 + r) for r, t in enumerate(ts)])
    spl = S.select_splitters(smp, dtype, p)
    bounds = [S.partition(t, dtype, spl, p - 1) for t in ts]
    E = D[dtype]
    outs = []
    for r in range(p):
        out = torch.cat([ts[s][bounds[s][r] * E:bounds[s][r + 1] * E] for s in range(p)])
        if out.numel() > E:
            S.sort(out, dtype)
        outs.append(out)
    torch.cuda.synchronize()
    got = torch.cat(outs).cpu().numpy().view(np.uint64)
    union = np.concatenate([a.reshape(-1) for a in shards])
    if dtype == PAIR:
        got, union = got.reshape(-1, 2), union.reshape(-1, 2)
    assert oracle.parity(np.ascontiguousarray(got), oracle.sort(np.ascontiguousarray(union), dtype), dtype) == -1
    if kind == "uniform":  # balanced within a loose bound
        sizes = [o.numel() // E for o in outs]
        assert max(sizes) < 2.0 * sum(sizes) / p
