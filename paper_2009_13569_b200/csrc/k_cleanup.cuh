// k_cleanup.cuh -- K5 cleanup and K6 the recursion scheduler
// (Alg. 2, adapted to device task lists).
#pragma once
#include "common.cuh"
#include "k_count.cuh"
#include "k_basecase.cuh"
#include "k_classify.cuh"

namespace ips4o {

// ------------------------------------------------------------------ K5a
// Phase a (one warp per bucket): save the elements of bucket j that its last
// block wrote past E_{j+1} into bucket j+1's head ("the head of
// b_{i+1}") -- logical positions [E_{j+1}, w_j*b) -- and, for the bucket that
// used the overflow block, copy the in-array part of that block to its
// final place [p*b, E_{j+1}).  Phase b then only writes holes.
constexpr int CLN_WARPS = 8;

// Grid: one CTA per (task, group of CLN_WARPS buckets), flattened into x
// (gridDim.y would cap the tasks of a level at 65535).
template <int DT> __host__ __device__ constexpr u32 cleanup_groups() {
  return (u32)((Traits<DT>::KIDX + CLN_WARPS - 1) / CLN_WARPS);
}

template <int DT>
__global__ void __launch_bounds__(CLN_WARPS * 32) cleanup_save_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Unit = typename Tr::Unit;
  constexpr int D = Tr::D, B = Tr::B;
  constexpr int UPE = D / (int)sizeof(Unit);
  if (A.go && *A.go == 0) return;  // round 0 of an easy input (k_plan.cuh)
  KTIMER(A.tslot, KS_CSAVE);
  const u32 ti = blockIdx.x / cleanup_groups<DT>();
  const LevelTask &L = A.tasks[ti];
  const int j = (int)(blockIdx.x % cleanup_groups<DT>()) * CLN_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= (int)L.K) return;
  const u64 bo = L.bucket_off;
  const u64 size = L.t.size;
  const u64 pblk = (size % B) ? size / B : ~0ull;
  const u32 ovb = A.ovf_used[ti];
  const char *ovf = A.overflow + (size_t)ti * B * D;
  char *gtask = A.base + L.t.begin * (u64)D;
  const u64 W = (A.wr[(bo + j) * WR_STRIDE] >> 32) * (u64)B;  // logical end of bucket j's blocks
  const u64 E1 = A.E[bo + j + 1];
  const u64 d0 = (A.E[bo + j] + B - 1) / B * B;
  const u64 o0 = E1 > d0 ? E1 : d0;  // bucket j's blocks cover [d0, W)
  auto logical = [&](u64 x) -> const Unit * {
    if (ovb == (u32)j && x >= pblk * B) return reinterpret_cast<const Unit *>(ovf + (x - pblk * B) * D);
    return reinterpret_cast<const Unit *>(gtask + x * D);
  };
  if (W > o0) {
    const u64 o = W - o0;  // < b
    if (!IPS4O_GUARD(o < (u64)B, A.err)) return;
    Unit *dst = reinterpret_cast<Unit *>(A.overlap + (bo + j) * (u64)B * D);
    for (u64 u = lane; u < o * UPE; u += 32) {
      u64 e = u / UPE, w = u % UPE;
      dst[u] = logical(o0 + e)[w];
    }
  }
  if (lane == 0) {
    // invariant of the cleanup: #holes = overlap + partial buffers (+ the
    // overflow block, placed below); a violation is reported, never silent
    const u64 hd = d0 < E1 ? d0 : E1;
    const u64 tl = W > hd ? W : hd;
    const u64 nholes = (hd - A.E[bo + j]) + (tl < E1 ? E1 - tl : 0);
    const u64 o = W > o0 ? W - o0 : 0;
    if (nholes != o + A.ptot[bo + j]) atomicOr(A.err, (u32)ERR_CLEANUP);
  }
  if (ovb == (u32)j) {
    const u64 p0 = pblk * B;
    const u64 hi = E1 < size ? E1 : size;
    for (u64 u = lane; p0 + u / UPE < hi; u += 32) {
      u64 e = u / UPE, w = u % UPE;
      reinterpret_cast<Unit *>(gtask + (p0 + e) * D)[w] = reinterpret_cast<const Unit *>(ovf + e * D)[w];
    }
  }
}

// ------------------------------------------------------------------ K5b
// Phase b: fill the holes of every bucket j -- its head [E_j, min(d_j,
// E_{j+1})) and its tail [w_j*b, E_{j+1}) -- with the saved overlap of bucket
// j and the partial buffers of every stripe of the task (the
// misplaced elements are in the head of b_{i+1}, in the partially filled
// buffers, or in the overflow block).  Hole h of bucket j (heads first) takes
// overlap element h for h < o, then the partial buffers in stripe order:
// stripe s's buffer fills holes [o + pcum_s, o + pcum_s + pfill_s).  One CTA
// per (stripe, task), a warp per bucket, coalesced copies of each buffer;
// the CTA of stripe 0 also places the overlaps.  Grid: the level's stripes.
constexpr int FILL_THREADS = 256;

template <int DT>
__global__ void __launch_bounds__(FILL_THREADS) cleanup_fill_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Unit = typename Tr::Unit;
  constexpr int D = Tr::D, B = Tr::B;
  constexpr int UPE = D / (int)sizeof(Unit);
  constexpr int NW = FILL_THREADS / 32;
  if (A.go && *A.go == 0) return;  // round 0 of an easy input (k_plan.cuh)
  KTIMER(A.tslot, KS_CFILL);
  const u32 ti = A.stripe_task[blockIdx.x];
  const LevelTask &L = A.tasks[ti];
  const u32 s = blockIdx.x - L.stripe_first;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u64 bo = L.bucket_off;
  char *gtask = A.base + L.t.begin * (u64)D;
  for (int j = wid; j < (int)L.K; j += NW) {
    const u64 slot = L.sbk_off + (u64)s * L.kidx + j;
    const u32 f = A.pfill[slot];
    const u64 E0 = A.E[bo + j], E1 = A.E[bo + j + 1];
    const u64 d0 = (E0 + B - 1) / B * B;
    const u64 W = (A.wr[(bo + j) * WR_STRIDE] >> 32) * (u64)B;
    const u64 hd = d0 < E1 ? d0 : E1;  // head hole [E0, hd)
    const u64 tl = W > hd ? W : hd;    // tail hole [tl, E1)
    const u64 nhead = hd - E0;
    const u64 o0 = E1 > d0 ? E1 : d0;
    const u64 o = W > o0 ? W - o0 : 0;  // saved overlap elements
    auto hole = [&](u64 h) -> u64 { return h < nhead ? E0 + h : tl + (h - nhead); };
    if (s == 0 && o) {
      const Unit *src = reinterpret_cast<const Unit *>(A.overlap + (bo + j) * (u64)B * D);
      for (u64 u = lane; u < o * UPE; u += 32) {
        const u64 e = u / UPE, w = u % UPE;
        if (IPS4O_GUARD(hole(e) < E1 && hole(e) >= E0, A.err)) reinterpret_cast<Unit *>(gtask + hole(e) * D)[w] = src[u];
      }
    }
    if (f == 0) continue;
    const u64 h0 = o + A.pcum[slot];
    const Unit *src = reinterpret_cast<const Unit *>(A.partials + slot * (u64)B * D);
    for (u32 u = lane; u < f * UPE; u += 32) {
      const u32 e = u / UPE, w = u % UPE;
      if (IPS4O_GUARD(hole(h0 + e) < E1 && hole(h0 + e) >= E0, A.err))
        reinterpret_cast<Unit *>(gtask + hole(h0 + e) * D)[w] = src[u];
    }
  }
}

// ------------------------------------------------------------------ K6
// Scheduler: turn the buckets of every task into child tasks.
// Equality buckets (odd index 2i+1, i < s) are terminal; buckets
// of at most one element are done; buckets of at most M elements (the
// one-CTA base-case capacity, the GPU analogue of "at most 2 n_0")
// go to the base-case list; the rest are appended to the pending list of the
// next round.  Child key bounds come from the splitters (TREE) or the digit
// (DIGIT).  Runs inside the boundaries kernel (K3a), by all threads of the
// task's CTA, once E is known: nothing it reads changes after K3a.
template <int DT, int ALGO>
__device__ void schedule_task(const LevelArgs &A, u32 ti, const u64 *sE) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  constexpr int KI = Tr::KIDX;
  const LevelTask &L = A.tasks[ti];
  const int K = (int)L.K;
  const Key plo = key_from_words<Key>(L.t.lo), phi = key_from_words<Key>(L.t.hi);
  const bool loose = (L.t.flags & TF_LOOSE) != 0;
  const Key *gt = reinterpret_cast<const Key *>(A.trees) + (size_t)ti * 2 * KI;
  const Key *spl = gt + KI;
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const u64 e0 = sE[j], e1 = sE[j + 1];
    const u64 sz = e1 - e0;
    if (sz == 0) continue;
    Key lo = plo, hi = phi;
    bool terminal = false;
    if (ALGO == ALGO_TREE) {
      const int s = (1 << L.l) - 1;
      if (L.equality) {
        const int i = j >> 1;
        if ((j & 1) && i < s) {
          lo = hi = spl[i];
          terminal = true;
        } else {
          // keys in (s_{i-1}, s_i) for i < s, or (s_{s-1}, +inf) for i = s
          if (i > 0) lo = spl[i - 1] + 1;
          if (i < s) hi = spl[i] - 1;
        }
      } else {
        // keys in (s_{j-1}, s_j]
        if (j > 0) lo = spl[j - 1] + 1;
        if (j < s) hi = spl[j];
      }
    } else if (sizeof(Key) == 8 && L.lut_log) {
      // logarithmic digit (R33): slot j covers the offsets [start(j), start(j+1))
      // from the task's lower bound
      if constexpr (sizeof(Key) == 8) {
        lo = plo + (Key)lut_slot_start((u32)j, 0, (int)L.lut_log);
        hi = plo + (Key)lut_slot_start((u32)j + 1, 0, (int)L.lut_log) - 1;
        if (hi < lo) hi = phi;  // (wrapped past 2^64: the last slots)
      }
    } else {
      const int bits = (int)L.l;
      const int sb = L.shift + bits;
      const Key top = sb >= (int)(8 * sizeof(Key)) ? (Key)0 : (plo >> sb) << sb;
      const Key dlo = top | ((Key)(u32)j << L.shift);
      const Key dhi = dlo | ((((Key)1) << L.shift) - 1);
      lo = dlo;
      hi = dhi;
      terminal = (L.shift == 0);  // a single key value per digit
    }
    if (lo < plo) lo = plo;
    if (hi > phi) hi = phi;
    if (lo >= hi) terminal = true;  // one distinct key (or an empty range)
    if (terminal || sz <= 1) {
      if (sz > 1) atomicAdd(reinterpret_cast<unsigned long long *>(&A.counters[2]), (unsigned long long)sz);
      continue;
    }
    if (sz == L.t.size && lo == plo && hi == phi && ALGO == ALGO_TREE) {
      // a child identical to its parent would be partitioned again forever
      // (cannot happen with >= 3 splitters, k_max >= 4); report, never loop
      atomicOr(A.err, (u32)ERR_NO_PROGRESS);
      continue;
    }
    TaskDesc c;
    c.begin = L.t.begin + e0;
    c.size = sz;
    key_to_words<Key>(lo, c.lo);
    key_to_words<Key>(hi, c.hi);
    c.level = L.t.level + 1;
    // a bound taken from a loose parent bound stays loose (TF_LOOSE)
    c.flags = loose && (lo == plo || hi == phi) ? (u32)TF_LOOSE : 0u;
    // DIGIT: a digit that kept most of the task splits bits the keys do not
    // use (sparse keys); measure the child's exact range first (DESIGN R27)
    if (ALGO == ALGO_DIGIT && 2 * sz > L.t.size) c.flags |= TF_MEASURE;
    if constexpr (BaseItem<DT>::KEY_ONLY) {
      // a narrow key range larger than the base case: counted and written
      // from the counts in this round (k_count.cuh, count-first)
      if (sz > 65535 && sz > A.base_split_elems && A.count_cap && hi - lo < (Key)CNT_RANGE_MAX) {
        const u32 R = (u32)(hi - lo) + 1;
        const u32 off = atomicAdd(&A.counters[10], R);
        if (off + R <= CNT_POOL) {
          const u32 slot = atomicAdd(&A.counters[9], 1u);
          if (slot < A.count_cap) {
            A.count_tasks[slot] = c;
            A.count_off[slot] = off;
            atomicAdd(reinterpret_cast<unsigned long long *>(&A.counters[6]), (unsigned long long)sz);
            continue;
          }
        }
      }
    }
    u32 *cnt;
    TaskDesc *list;
    u32 cap;
    if (sz <= A.base_cap_elems) {
      cnt = &A.counters[1], list = A.base_tasks, cap = A.base_cap_tasks;
      atomicAdd(reinterpret_cast<unsigned long long *>(&A.counters[6]), (unsigned long long)sz);
    } else if (sz <= A.base_split_elems ||
               (BaseItem<DT>::KEY_ONLY && sz <= 65535 && hi - lo < (Key)basecase_count_range<DT>())) {
      // up to twice the capacity: the base case's two-pass split (K7s); a
      // narrow key range of a key-only type: counted exactly (any size)
      cnt = &A.counters[8], list = A.split_tasks, cap = A.base_cap_tasks;
      atomicAdd(reinterpret_cast<unsigned long long *>(&A.counters[6]), (unsigned long long)sz);
    } else {
      cnt = A.next_count, list = A.next_tasks, cap = A.next_cap;
    }
    const u32 slot = atomicAdd(cnt, 1u);
    if (slot < cap) list[slot] = c;
    else atomicOr(A.err, (u32)ERR_LIST_OVERFLOW);
  }
}

}  // namespace ips4o
