"""Multi-GPU samplesort: the distributed form of the partitioning step
(SURVEY 8(e), row NEXT-4).  The paper uses IPS4o as the local step of
distributed-memory sorting; the splitter rule is its own
(random sample, equidistant picks).  One process per GPU under
torch.distributed (NCCL over NVLink/NVSwitch); every step on the data runs in
the library's kernels, the exchanges are NCCL collectives:

  1. ``ips4o_sample``: each rank draws ``m`` samples of its shard (DESIGN R8
     draw, a seed per rank);
  2. all-gather of the samples (and of the shard sizes: empty shards
     contribute none);
  3. ``ips4o_select_splitters``: every rank sorts the same global sample and
     picks the same p - 1 splitters at the equidistant ranks;
  4. ``ips4o_partition_splitters``: one in-place partitioning step of the
     shard into p ranges, range r = {e : S_{r-1} < e <= S_r};
  5. all-to-all of the range sizes, then of the ranges themselves;
  6. ``ips4o_sort`` of the received elements.

Rank r returns the r-th slice of the globally sorted sequence; the slices of
ranks 0..p-1 concatenated are the sorted union of the shards.  This is not
globally in place: the receive buffer is new (the exchange needs one).

``steps`` selects who executes steps 1, 3, 4 and 6.  The default is the
library (CUDA tensors).  The tests pass CPU stand-ins built on the oracle to
check the exchange logic with the gloo backend on CPU; nothing here imports
the oracle.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import ELEM_BYTES, partition_splitters, sample, select_splitters, sort


class NativeSteps:
    """Steps 1, 3, 4, 6 on the GPU through the C ABI (uint8 CUDA tensors)."""

    def sample(self, t, dtype: int, m: int, seed: int):
        out = torch.empty(m * ELEM_BYTES[dtype], dtype=torch.uint8, device=t.device)
        sample(t, dtype, m, seed, out)
        return out

    def select_splitters(self, samples, dtype: int, parts: int):
        out = torch.empty((parts - 1) * ELEM_BYTES[dtype], dtype=torch.uint8, device=samples.device)
        select_splitters(samples, dtype, parts, out)
        return out

    def partition(self, t, dtype: int, splitters, nspl: int) -> list:
        return partition_splitters(t, dtype, splitters, nspl)

    def sort(self, t, dtype: int) -> None:
        sort(t, dtype)


def default_samples_per_rank(n_total: int, p: int) -> int:
    """m samples per rank: alpha * p with alpha = max(16, ceil(0.2 log2 N))
    (the paper's oversampling, with a floor for small N), so the
    global sample holds alpha samples per range."""
    alpha = max(16, math.ceil(0.2 * math.log2(max(n_total, 2))))
    return alpha * p


def sample_sort(t, dtype: int, group=None, samples_per_rank: int = 0, seed: int = 0x5EED, steps=None):
    """Sort the union of the ranks' shards.  ``t`` is this rank's shard as a
    contiguous uint8 tensor of n*D bytes (CUDA for NCCL; CPU with gloo and CPU
    ``steps``).  It is partitioned in place (step 4).  Returns
    ``(out, info)``: ``out`` (uint8, this rank's sorted slice) and a dict with
    the splitter count, the send/receive element counts and the bounds."""
    steps = steps or NativeSteps()
    D = ELEM_BYTES[dtype]
    if t.dtype != torch.uint8 or t.dim() != 1 or t.numel() % D:
        raise ValueError("expected a flat uint8 tensor of whole elements")
    p = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = t.numel() // D
    dev = t.device
    if p == 1:
        steps.sort(t, dtype)
        return t, {"parts": 1, "send": [n], "recv": [n], "bounds": [0, n]}
    # shard sizes (every rank learns N and which shards are empty)
    sizes = torch.tensor([n], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(p)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [int(x.item()) for x in all_sizes]
    n_total = sum(all_sizes)
    if n_total == 0:
        return t[:0].clone(), {"parts": p, "send": [0] * p, "recv": [0] * p, "bounds": [0] * (p + 1)}
    m = samples_per_rank or default_samples_per_rank(n_total, p)
    # 1-2. samples, gathered (an empty shard sends a placeholder block that is dropped)
    rank_seed = (seed + 0x9E3779B97F4A7C15 * (rank + 1)) % (1 << 64)
    mine = steps.sample(t, dtype, m, rank_seed) if n > 0 else torch.zeros(m * D, dtype=torch.uint8, device=dev)
    blocks = [torch.empty(m * D, dtype=torch.uint8, device=dev) for _ in range(p)]
    dist.all_gather(blocks, mine, group=group)
    gathered = torch.cat([b for b, s in zip(blocks, all_sizes) if s > 0])
    # 3. the same p - 1 splitters on every rank
    spl = steps.select_splitters(gathered, dtype, p)
    # 4. the shard's ranges
    bounds = steps.partition(t, dtype, spl, p - 1) if n > 0 else [0] * (p + 1)
    send = [bounds[r + 1] - bounds[r] for r in range(p)]
    # 5. sizes, then the elements
    send_t = torch.tensor(send, dtype=torch.int64, device=dev)
    recv_t = torch.empty(p, dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv_t, send_t, group=group)
    recv = [int(x) for x in recv_t.tolist()]
    out = torch.empty(sum(recv) * D, dtype=torch.uint8, device=dev)
    dist.all_to_all_single(out, t, output_split_sizes=[c * D for c in recv],
                           input_split_sizes=[c * D for c in send], group=group)
    # 6. the received ranges sorted locally
    if sum(recv) > 1:
        steps.sort(out, dtype)
    return out, {"parts": p, "send": send, "recv": recv, "bounds": bounds, "samples_per_rank": m}
