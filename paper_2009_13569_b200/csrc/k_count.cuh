// k_count.cuh -- count-first finish of narrow-range tasks (key-only types).
//
// The paper's future work ("first determine exact bucket sizes
// ... then one could integrate the classification phase and the permutation
// phase") in the one case where it needs no buffers at all: a task of a
// key-only type (U64, F64, U32) whose key range [lo, hi] holds at most
// CNT_RANGE_MAX values.  Counting the keys per value (one read pass) gives
// the exact size of every "bucket" = key value, and the sorted task is written
// from the counts alone (one write pass): 2nD instead of the 4nD of a
// partitioning level plus the 2nD of the base case.  Key-only: an element is
// its key, so writing value lo + v count_v times reproduces the multiset
// exactly.  The scheduler (K6) routes such children larger than the base case
// here (smaller ones are counted by the one-CTA base case itself); duplicate-
// heavy inputs make them (RootDup's level-1 buckets hold ~128 key values).
//
// Three kernels after the round's cleanup (the tasks' elements are then in
// place): K9a splits the tasks into chunks and clears their counters, K9b
// counts per chunk in shared memory and adds the non-zero counts to the
// task's counters, K9c writes each chunk of positions from the prefix of the
// counts.  Chunks are taken from a work counter, so every CTA stays busy
// whatever the task sizes.
#pragma once
#include "common.cuh"

namespace ips4o {

constexpr int CNT_THREADS = 512;
constexpr u32 CNT_RANGE_MAX = 4096;     // key values of a count task (hi - lo + 1)
constexpr u64 CNT_CHUNK = 1ull << 18;   // elements per work item
constexpr u32 CNT_POOL = 1u << 20;      // task counters per round (u32)
constexpr int CNT_SETUP_THREADS = 1024;

// K9a: exclusive prefix of the tasks' chunk counts (pre[n] = total); clears
// the counters of every task and the two work counters.  One CTA.
__global__ void __launch_bounds__(CNT_SETUP_THREADS) count_setup_kernel(LevelArgs A) {
  __shared__ u32 s_ws[CNT_SETUP_THREADS / 32 + 1];
  const u32 nt = min(A.counters[9], A.count_cap);
  if (nt == 0) return;
  KTIMER(A.tslot, KS_NARROW);
  const int tid = threadIdx.x;
  u32 carry = 0;
  for (u32 b0 = 0; b0 < nt; b0 += CNT_SETUP_THREADS) {
    const u32 i = b0 + tid;
    const u32 c = i < nt ? (u32)((A.count_tasks[i].size + CNT_CHUNK - 1) / CNT_CHUNK) : 0u;
    u32 tot;
    const u32 ex = block_exclusive_scan<CNT_SETUP_THREADS>(c, s_ws, &tot);
    if (i < nt) A.count_pre[i] = carry + ex;
    carry += tot;
  }
  if (tid == 0) {
    A.count_pre[nt] = carry;
    A.count_work[0] = 0;
    A.count_work[1] = 0;
  }
  const u32 used = min(A.counters[10], CNT_POOL);
  for (u32 v = tid; v < used; v += CNT_SETUP_THREADS) A.count_hist[v] = 0;
}

// Work item `it` -> (task, first element of its chunk).
__device__ __forceinline__ u32 count_task_of(const u32 *pre, u32 nt, u32 it) {
  u32 a = 0, b = nt - 1;  // largest t with pre[t] <= it
  while (a < b) {
    const u32 m = (a + b + 1) >> 1;
    if (pre[m] <= it) a = m;
    else b = m - 1;
  }
  return a;
}

// K9b: counts per key value.  Equal keys of a warp are counted with one
// shared-memory atomic (few-valued tasks have long runs of equal keys).
template <int DT>
__global__ void __launch_bounds__(CNT_THREADS) count_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  constexpr int D = Tr::D;
  __shared__ u32 s_cnt[CNT_RANGE_MAX];
  __shared__ u32 s_it;
  const u32 nt = min(A.counters[9], A.count_cap);
  if (nt == 0) return;
  KTIMER(A.tslot, KS_NARROW);
  const u32 total = A.count_pre[nt];
  const int tid = threadIdx.x, lane = tid & 31;
  for (;;) {
    if (tid == 0) s_it = atomicAdd(&A.count_work[0], 1u);
    __syncthreads();
    const u32 it = s_it;
    if (it >= total) break;
    const u32 t = count_task_of(A.count_pre, nt, it);
    const TaskDesc T = A.count_tasks[t];
    const Key lo = key_from_words<Key>(T.lo), hi = key_from_words<Key>(T.hi);
    const u32 R = (u32)(hi - lo) + 1;
    const u64 c0 = (u64)(it - A.count_pre[t]) * CNT_CHUNK;
    const u64 c1 = c0 + CNT_CHUNK < T.size ? c0 + CNT_CHUNK : T.size;
    for (u32 v = tid; v < R; v += CNT_THREADS) s_cnt[v] = 0;
    __syncthreads();
    const char *g = A.base + T.begin * (u64)D;
    // whole warps over the chunk, CU elements per thread in flight; a warp
    // whose 32 keys are one value adds them with one atomic (runs of equal
    // keys), else one atomic per lane (inactive lanes count nothing)
    constexpr int CU = 8;
    for (u64 i0 = c0 + (u64)(tid - lane) * CU; i0 < c1; i0 += (u64)CNT_THREADS * CU) {
      u32 v[CU];
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const u64 i = i0 + (u64)u * 32 + lane;
        v[u] = i < c1 ? (u32)(Tr::key(g + i * D) - lo) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const u32 v0 = __shfl_sync(0xffffffffu, v[u], 0);
        if (__all_sync(0xffffffffu, v[u] == v0)) {
          if (lane == 0 && v0 != 0xFFFFFFFFu && IPS4O_GUARD(v0 < R, A.err)) atomicAdd(&s_cnt[v0], 32u);
        } else if (v[u] != 0xFFFFFFFFu && IPS4O_GUARD(v[u] < R, A.err)) {
          atomicAdd(&s_cnt[v[u]], 1u);
        }
      }
    }
    __syncthreads();
    u32 *gc = A.count_hist + A.count_off[t];
    for (u32 v = tid; v < R; v += CNT_THREADS)
      if (s_cnt[v]) atomicAdd(&gc[v], s_cnt[v]);
    __syncthreads();  // s_cnt and s_it are reused
  }
}

// K9c: writes the chunk's positions: position p of the task holds lo + v for
// the largest v with start_v <= p (starts = exclusive prefix of the counts).
// A warp takes 256 consecutive positions (coalesced stores); two lanes bound
// the values of its first and last position; one value (long runs) is written
// at once, otherwise each position searches between the bounds.
template <int DT>
__global__ void __launch_bounds__(CNT_THREADS) count_write_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  constexpr int D = Tr::D;
  __shared__ u32 s_st[CNT_RANGE_MAX];
  __shared__ u32 s_ws[CNT_THREADS / 32 + 1];
  __shared__ u32 s_it;
  const u32 nt = min(A.counters[9], A.count_cap);
  if (nt == 0) return;
  KTIMER(A.tslot, KS_NARROW);
  const u32 total = A.count_pre[nt];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int VPT = CNT_RANGE_MAX / CNT_THREADS;
  for (;;) {
    if (tid == 0) s_it = atomicAdd(&A.count_work[1], 1u);
    __syncthreads();
    const u32 it = s_it;
    if (it >= total) break;
    const u32 t = count_task_of(A.count_pre, nt, it);
    const TaskDesc T = A.count_tasks[t];
    const Key lo = key_from_words<Key>(T.lo), hi = key_from_words<Key>(T.hi);
    const u32 R = (u32)(hi - lo) + 1;
    const u64 c0 = (u64)(it - A.count_pre[t]) * CNT_CHUNK;
    const u64 c1 = c0 + CNT_CHUNK < T.size ? c0 + CNT_CHUNK : T.size;
    // starts of the values: thread t scans values [t*VPT, (t+1)*VPT)
    const u32 *gc = A.count_hist + A.count_off[t];
    u32 h[VPT], sum = 0;
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const u32 v = (u32)tid * VPT + q;
      h[q] = v < R ? gc[v] : 0u;
      sum += h[q];
    }
    u32 all;
    u32 st = block_exclusive_scan<CNT_THREADS>(sum, s_ws, &all);
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const u32 v = (u32)tid * VPT + q;
      if (v < R) s_st[v] = st;
      st += h[q];
    }
    __syncthreads();
    if (IPS4O_GUARD(all == T.size, A.err)) {
      auto last_le = [&](u32 p, u32 a, u32 b) -> u32 {  // largest v in [a, b] with start_v <= p
        while (a < b) {
          const u32 m = (a + b + 1) >> 1;
          if (s_st[m] <= p) a = m;
          else b = m - 1;
        }
        return a;
      };
      char *g = A.base + T.begin * (u64)D;
      auto put = [&](u64 p, u32 v) {
        const Key k = lo + (Key)v;
        if constexpr (DT == DT_F64) reinterpret_cast<u64 *>(g)[p] = key_to_f64((u64)k);
        else if constexpr (DT == DT_U32) reinterpret_cast<u32 *>(g)[p] = (u32)k;
        else reinterpret_cast<u64 *>(g)[p] = (u64)k;
      };
      // a warp takes WU * 32 consecutive positions; if its first and last
      // position hold the same value (long runs) every lane writes it,
      // otherwise each position searches between the two bounds
      constexpr int WU = 8;
      for (u64 p0 = c0 + (u64)wid * 32 * WU; p0 < c1; p0 += (u64)CNT_THREADS * WU) {
        const u64 plast = p0 + 32 * WU - 1 < c1 ? p0 + 32 * WU - 1 : c1 - 1;
        u32 bd = 0;
        if (lane < 2) bd = last_le((u32)(lane == 0 ? p0 : plast), 0u, R - 1);
        const u32 va = __shfl_sync(0xffffffffu, bd, 0), vb = __shfl_sync(0xffffffffu, bd, 1);
#pragma unroll
        for (int u = 0; u < WU; ++u) {
          const u64 p = p0 + (u64)u * 32 + lane;
          if (p < c1) put(p, va == vb ? va : last_le((u32)p, va, vb));
        }
      }
    }
    __syncthreads();  // s_st and s_it are reused
  }
}

}  // namespace ips4o
