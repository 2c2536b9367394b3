// k_classify.cuh -- K2: classification with block buffers (P:739-780,
// Figs. 4/5 P:745-760).  One CTA per stripe.  The CTA streams its stripe
// through shared-memory tiles (cp.async double buffering), classifies each
// element with the branchless tree (Alg. 1, batched per thread like
// the paper's unrolled loop) or the IPS2Ra digit, appends it to one of K
// shared-memory buffer blocks of b elements, and writes every full block back
// to the front of its own stripe (there is always room because at
// least b more elements were read than written).  Per-bucket counts come for
// free.  At the end the partially filled buffers are spilled to
// scratch (they are the "partial buffers" of the cleanup).
//
// Tile-synchronous form (SURVEY 7/H2 option B): per tile, bucket ranks come
// from shared-memory atomics, a CTA-wide scan over the K buckets yields the
// blocks each bucket emits, and warps write whole blocks with coalesced
// stores.  Elements of an emitted block come from the bucket's buffer (older
// elements) followed by tile elements (gathered through an index list).
#pragma once
#include "common.cuh"

namespace ips4o {

template <class Key>
__device__ __forceinline__ u32 tree_bucket(const Key *tree, const Key *spl, int l, int eq, Key e) {
  u32 i = 1;
  for (int r = 0; r < l; ++r) i = 2 * i + (tree[i] < e ? 1u : 0u);
  u32 leaf = i - (1u << l);
  if (!eq) return leaf;
  return 2 * leaf + 1 - (e < spl[leaf] ? 1u : 0u);
}

// Alg. 1: one tree level across all IPT elements before the next level.
template <class Key, int IPT>
__device__ __forceinline__ void tree_bucket_batch(const Key *tree, const Key *spl, int l, int eq,
                                                  const Key (&e)[IPT], u32 (&b)[IPT]) {
#pragma unroll
  for (int k = 0; k < IPT; ++k) b[k] = 1;
  for (int r = 0; r < l; ++r) {
#pragma unroll
    for (int k = 0; k < IPT; ++k) b[k] = 2 * b[k] + (tree[b[k]] < e[k] ? 1u : 0u);
  }
  const u32 half = 1u << l;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    u32 leaf = b[k] - half;
    b[k] = eq ? 2 * leaf + 1 - (e[k] < spl[leaf] ? 1u : 0u) : leaf;
  }
}

// The read-done bytes of the permutation (K4) for this stripe's block
// positions start at 0; each stripe clears its own (no separate memset).
template <int B>
__device__ __forceinline__ void clear_read_flags(const LevelArgs &A, const LevelTask &L, u64 s0, u64 s1) {
  unsigned char *f = A.rdone + L.blk_off;
  const u64 b0 = s0 / B, b1 = (s1 + B - 1) / B;
  for (u64 x = b0 + threadIdx.x; x < b1; x += blockDim.x) f[x] = 0;
}

template <int DT>
struct ClsSmem {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  static constexpr int D = Tr::D, B = Tr::B, KI = Tr::KIDX, T = Tr::CLS_TILE, NT = Tr::CLS_THREADS;
  static constexpr int TILE_BYTES = ((T * D + 16) + 15) / 16 * 16;
  static constexpr size_t off_buf = 0;
  static constexpr size_t off_tiles = off_buf + (size_t)KI * B * D;
  static constexpr size_t off_tree = (off_tiles + 2 * TILE_BYTES + 15) / 16 * 16;
  static constexpr size_t off_u32 = off_tree + 2 * KI * sizeof(Key);
  // u32 arrays: fill, tcnt, cnt, boff, eoff, nb  (KI each) + ws (NT/32 + 1)
  static constexpr size_t off_idx = off_u32 + (6 * KI + NT / 32 + 1) * 4;
  static constexpr size_t bytes = (off_idx + T * 2 + 15) / 16 * 16;
};

template <int DT, int ALGO>
__global__ void __launch_bounds__(Traits<DT>::CLS_THREADS, 1) classify_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  using Unit = typename Tr::Unit;
  using S = ClsSmem<DT>;
  constexpr int D = Tr::D, B = Tr::B, KI = Tr::KIDX, T = Tr::CLS_TILE, NT = Tr::CLS_THREADS;
  constexpr int IPT = T / NT;
  constexpr int UPE = D / (int)sizeof(Unit);  // units per element
  constexpr int NWARPS = NT / 32;
  static_assert(T % NT == 0, "tile must be a multiple of the CTA size");
  static_assert(KI <= NT, "one thread per bucket in the scans");
  static_assert(T < 65536 && T / B + KI < 65536, "16-bit scan packing");

  extern __shared__ __align__(16) char smem[];
  char *s_buf = smem + S::off_buf;
  char *s_tiles = smem + S::off_tiles;
  Key *s_tree = reinterpret_cast<Key *>(smem + S::off_tree);
  Key *s_spl = s_tree + KI;
  u32 *s_fill = reinterpret_cast<u32 *>(smem + S::off_u32);
  u32 *s_tcnt = s_fill + KI;
  u32 *s_cnt = s_tcnt + KI;
  u32 *s_boff = s_cnt + KI;
  u32 *s_eoff = s_boff + KI;
  u32 *s_nb = s_eoff + KI;
  u32 *s_ws = s_nb + KI;
  unsigned short *s_idx = reinterpret_cast<unsigned short *>(smem + S::off_idx);

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (A.go && *A.go == 0) return;  // round 0 of an easy input (k_plan.cuh)
  KTIMER(A.tslot, KS_CLASSIFY);
  const u32 stripe = blockIdx.x;
  const u32 ti = A.stripe_task[stripe];
  const LevelTask &L = A.tasks[ti];
  const int K = (int)L.K, l = (int)L.l, eq = (int)L.equality, shift = L.shift;
  const u32 dmask = L.K - 1;
  const u64 size = L.t.size;
  const u64 s0 = (u64)(stripe - L.stripe_first) * L.stripe_elems;
  const u64 s1 = (s0 + L.stripe_elems < size) ? s0 + L.stripe_elems : size;
  char *gtask = A.base + L.t.begin * (u64)D;
  clear_read_flags<B>(A, L, s0, s1);

  if (ALGO == ALGO_TREE) {
    const Key *gt = reinterpret_cast<const Key *>(A.trees) + (size_t)ti * 2 * KI;
    const int leaves = 1 << l;
    for (int i = tid; i < leaves; i += NT) {
      s_tree[i] = gt[i];
      s_spl[i] = gt[KI + i];
    }
  }
  for (int j = tid; j < KI; j += NT) {
    s_fill[j] = 0;
    s_tcnt[j] = 0;
    s_cnt[j] = 0;
  }

  const u64 n = s1 > s0 ? s1 - s0 : 0;
  const u64 ntiles = (n + T - 1) / T;
  u64 front = 0;  // blocks flushed so far (relative to the stripe start)

  if (ntiles > 0) {
    u64 c0 = n < (u64)T ? n : (u64)T;
    tile_load_async(s_tiles, gtask + s0 * D, c0 * D, tid, NT);
  }
  cp_async_commit();

  for (u64 t = 0; t < ntiles; ++t) {
    const int stage = (int)(t & 1);
    const u64 e0 = s0 + t * T;  // first element of this tile (task-relative)
    const int cnt = (int)((s1 - e0) < (u64)T ? (s1 - e0) : (u64)T);
    if (t + 1 < ntiles) {
      const u64 e1 = e0 + T;
      const u64 c1 = (s1 - e1) < (u64)T ? (s1 - e1) : (u64)T;
      tile_load_async(s_tiles + (1 - stage) * S::TILE_BYTES, gtask + e1 * D, c1 * D, tid, NT);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const char *tp = s_tiles + stage * S::TILE_BYTES + (int)(((uintptr_t)(gtask + e0 * D)) & 15);

    // ---- classify (Alg. 1 batched over IPT elements per thread)
    Key key[IPT];
    u32 bkt[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      int i = tid + k * NT;
      key[k] = i < cnt ? Tr::key(tp + (size_t)i * D) : (Key)0;
    }
    if (ALGO == ALGO_TREE) {
      tree_bucket_batch<Key, IPT>(s_tree, s_spl, l, eq, key, bkt);
    } else {
#pragma unroll
      for (int k = 0; k < IPT; ++k) bkt[k] = digit_of(key[k], shift, dmask);
    }
    u32 rank[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      int i = tid + k * NT;
      rank[k] = i < cnt ? atomicAdd(&s_tcnt[bkt[k]], 1u) : 0u;
    }
    __syncthreads();

    // ---- per-bucket plan: blocks to emit (nb) and tile elements they take (em)
    u32 tc = 0, tot = 0, nb = 0, em = 0;
    if (tid < KI) {
      tc = s_tcnt[tid];
      tot = s_fill[tid] + tc;
      nb = tot / B;
      em = nb ? nb * B - s_fill[tid] : 0;
    }
    u32 total;
    u32 pre = block_exclusive_scan<NT>((nb << 16) | em, s_ws, &total);
    if (tid < KI) {
      s_boff[tid] = pre >> 16;
      s_eoff[tid] = pre & 0xFFFFu;
      s_nb[tid] = nb;
      s_cnt[tid] += tc;
    }
    const u32 nblocks = total >> 16;
    __syncthreads();

    // ---- stage the tile elements of emitted blocks (index list)
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      int i = tid + k * NT;
      if (i < cnt) {
        u32 j = bkt[k];
        u32 v = s_fill[j] + rank[k];
        if (v < s_nb[j] * B) s_idx[s_eoff[j] + rank[k]] = (unsigned short)i;
      }
    }
    __syncthreads();

    // ---- emit full blocks to the stripe's write front (coalesced per warp)
    for (u32 g = wid; g < nblocks; g += NWARPS) {
      // bucket j = last index with boff[j] <= g (it has nb > 0)
      int lo = 0, hi = KI;  // find first index with boff > g
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (s_boff[mid] <= g) lo = mid + 1;
        else hi = mid;
      }
      const int j = lo - 1;
      const u32 q = g - s_boff[j];
      const u32 bf = s_fill[j];
      const u32 eo = s_eoff[j];
      Unit *dst = reinterpret_cast<Unit *>(gtask + (s0 + (front + s_boff[j] + q) * B) * D);
      if (!IPS4O_GUARD(s0 + (front + s_boff[j] + q + 1) * B <= s1, A.err)) continue;
      if (lane == 0) A.bid[L.blk_off + s0 / B + front + s_boff[j] + q] = (unsigned short)j;
      for (int u = lane; u < B * UPE; u += 32) {
        const int e = u / UPE, w = u - e * UPE;
        const u32 v = q * B + e;
        const char *src = v < bf ? s_buf + ((size_t)j * B + v) * D
                                 : tp + (size_t)s_idx[eo + v - bf] * D;
        dst[u] = reinterpret_cast<const Unit *>(src)[w];
      }
    }
    front += nblocks;
    __syncthreads();

    // ---- remaining tile elements go to the (now free) buffer slots
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      int i = tid + k * NT;
      if (i < cnt) {
        u32 j = bkt[k];
        u32 v = s_fill[j] + rank[k];
        u32 cut = s_nb[j] * B;
        if (v >= cut) {
          const Unit *src = reinterpret_cast<const Unit *>(tp + (size_t)i * D);
          Unit *dst = reinterpret_cast<Unit *>(s_buf + ((size_t)j * B + (v - cut)) * D);
#pragma unroll
          for (int w = 0; w < UPE; ++w) dst[w] = src[w];
        }
      }
    }
    __syncthreads();
    if (tid < KI) {
      s_fill[tid] = tot - nb * B;
      s_tcnt[tid] = 0;
    }
    // the next iteration's __syncthreads orders these updates
  }
  __syncthreads();

  // ---- outputs: counts, partial fill, full blocks, partial buffers
  const u64 sbase = L.sbk_off + (u64)(stripe - L.stripe_first) * L.kidx;
  for (int j = tid; j < (int)L.kidx; j += NT) {
    A.counts[sbase + j] = s_cnt[j];
    A.pfill[sbase + j] = s_fill[j];
  }
  if (tid == 0) A.fullblocks[stripe] = (u32)front;
  for (int j = wid; j < K; j += NWARPS) {
    const int f = (int)s_fill[j];
    const Unit *src = reinterpret_cast<const Unit *>(s_buf + (size_t)j * B * D);
    Unit *dst = reinterpret_cast<Unit *>(A.partials + (sbase + j) * (u64)B * D);
    for (int u = lane; u < f * UPE; u += 32) dst[u] = src[u];
  }
}

}  // namespace ips4o

namespace ips4o {

template <int DT>
__device__ __forceinline__ typename Traits<DT>::Key elem_key(const typename Traits<DT>::Unit &x) {
  if constexpr (DT == DT_PAIR) {
    return ((u64)x.y << 32) | (u64)x.x;
  } else if constexpr (DT == DT_U32) {
    return (u64)x;
  } else if constexpr (DT == DT_F64) {
    return f64_to_key(x);
  } else {
    return x;
  }
}

// ------------------------------------------------------------------ K2 v2, 8/16-byte elements
// Tile-synchronous classification with block buffers, three barriers per tile.
// 1024 threads; each owns IPT elements of a T-element tile in registers (the
// next tile is loaded while the current one is processed).  Per tile:
//   classify (LUT of starting leaves + short search) and rank by
//   shared atomics  | A |  the previous tile's leftovers enter the freed
//   buffers; one scan over the k' buckets plans, per bucket j, nb_j full
//   blocks: block 0 is buffer j completed by the first B - fill_j tile
//   elements, blocks 1..nb_j-1 are whole runs of tile elements staged
//   contiguously; the remaining elements are leftovers  | B |  scatter: every
//   element is stored once, into buffer j, its staged block, or kept in
//   registers as a leftover  | C |  warps copy the emitted blocks to the
//   stripe's write front.  Leftovers are written into buffer j
//   after the next tile's barrier A, once the copies have read buffer j.
#ifndef IPS4O_CLS_STCS
#define IPS4O_CLS_STCS 1  // emitted blocks (8-byte units) stored with the streaming (evict-first) hint: 2^30 u64 classify 9.94 -> 9.84 ms
#endif
#ifndef IPS4O_CLS_LDCS
#define IPS4O_CLS_LDCS 0  // tile loads with the streaming hint (measured: +0.2 ms)
#endif
template <class Unit> __device__ __forceinline__ void cls_store(Unit *p, const Unit &v) {
#if IPS4O_CLS_STCS
  if constexpr (sizeof(Unit) == 8) {
    __stcs(reinterpret_cast<unsigned long long *>(p), *reinterpret_cast<const unsigned long long *>(&v));
    return;
  }
#endif
  *p = v;
}
template <class Unit> __device__ __forceinline__ Unit cls_load(const Unit *p) {
#if IPS4O_CLS_LDCS
  if constexpr (sizeof(Unit) == 8) {
    const unsigned long long w = __ldcs(reinterpret_cast<const unsigned long long *>(p));
    return *reinterpret_cast<const Unit *>(&w);
  }
#endif
  return *p;
}
#ifndef IPS4O_CLS_PF
#define IPS4O_CLS_PF 2  // L2 prefetch distance in tiles
#endif
template <int DT> struct ClsV2 {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
#ifndef IPS4O_CLS_NT
#define IPS4O_CLS_NT 1024
#endif
  static constexpr int NT = IPS4O_CLS_NT;
  static constexpr int T = Tr::D <= 8 ? 4096 : 2048;
  static constexpr int IPT = T / NT;
  static constexpr int D = Tr::D, B = Tr::B, KI = Tr::KIDX;
  static constexpr int BUFS = B + (Tr::D <= 8 ? 1 : 0);  // buffer stride in elements (bank skew)
  static constexpr size_t off_buf = 0;
  static constexpr size_t off_stage = ((size_t)KI * BUFS * D + 15) / 16 * 16;
  static constexpr size_t off_tree = off_stage + (size_t)T * D;
  static constexpr size_t off_u32 = off_tree + 2 * KI * sizeof(Key);
  // u32 arrays: tcnt, cnt, plan (KI each), ws (32); then the block -> (bucket, index) map
  static constexpr size_t off_blkb = off_u32 + (3 * KI + 32) * 4;
  static constexpr int MAXBLK = T / B + KI;
  static constexpr int LUT_BITS = 14;  // 16-bit entries
  static constexpr size_t off_lut = (off_blkb + (size_t)MAXBLK * 2 + 15) / 16 * 16;
  static constexpr size_t bytes = off_lut + ((size_t)2 << LUT_BITS);
};

template <int DT, int ALGO>
__global__ void __launch_bounds__(ClsV2<DT>::NT, 1) classify_v2_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  using Unit = typename Tr::Unit;  // one element
  using S = ClsV2<DT>;
  constexpr int NT = S::NT, T = S::T, IPT = S::IPT, B = Tr::B, KI = Tr::KIDX, BUFS = S::BUFS;
  constexpr int NWARPS = NT / 32;
  constexpr u32 NONE = 0xFFFFFFFFu;
  static_assert(Tr::D == sizeof(Unit), "one unit per element");
  static_assert(KI % 32 == 0 && KI <= NT && B <= 255 && (T / B + 1) * B < 8192 && T / B < 2048, "plan packing");
  constexpr u32 STG0 = (u32)(S::off_stage / sizeof(Unit));  // stage start, in elements from s_buf

  extern __shared__ __align__(16) char smem[];
  Unit *s_buf = reinterpret_cast<Unit *>(smem + S::off_buf);
  Unit *s_stage = reinterpret_cast<Unit *>(smem + S::off_stage);
  Key *s_tree = reinterpret_cast<Key *>(smem + S::off_tree);
  Key *s_spl = s_tree + KI;
  u32 *s_tcnt = reinterpret_cast<u32 *>(smem + S::off_u32);
  u32 *s_cnt = s_tcnt + KI;
  u32 *s_plan = s_cnt + KI;
  u32 *s_ws = s_plan + KI;
  unsigned short *s_blkb = reinterpret_cast<unsigned short *>(smem + S::off_blkb);
  unsigned short *s_lut = reinterpret_cast<unsigned short *>(smem + S::off_lut);

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (A.go && *A.go == 0) return;  // round 0 of an easy input (k_plan.cuh)
  KTIMER(A.tslot, KS_CLASSIFY);
  const u32 stripe = blockIdx.x;
  const u32 ti = A.stripe_task[stripe];
  const LevelTask &L = A.tasks[ti];
  const int K = (int)L.K, l = (int)L.l, eq = (int)L.equality, shift = L.shift;
  const u32 dmask = L.K - 1;
  const u64 size = L.t.size;
  const u64 s0 = (u64)(stripe - L.stripe_first) * L.stripe_elems;
  const u64 s1 = (s0 + L.stripe_elems < size) ? s0 + L.stripe_elems : size;
  Unit *gtask = reinterpret_cast<Unit *>(A.base + L.t.begin * (u64)Tr::D);
  clear_read_flags<B>(A, L, s0, s1);

  if (ALGO == ALGO_TREE) {
    const Key *gt = reinterpret_cast<const Key *>(A.trees) + (size_t)ti * 2 * KI;
    for (int i = tid; i < (1 << l); i += NT) {
      s_tree[i] = gt[i];
      s_spl[i] = gt[KI + i];
    }
  }
  for (int j = tid; j < KI; j += NT) {
    s_tcnt[j] = 0;
    s_cnt[j] = 0;
  }
  if (tid == 0) s_ws[KI / 32] = 0;  // block allocator of the first tile
  u32 myfill = 0;  // tid < KI: elements buffered for bucket tid

  // Lookup table of starting leaves, built once per task by K1
  // (build_lut): copied into shared memory, 32 B per thread.
  const Key tlo = key_from_words<Key>(L.t.lo);
  Key llo = tlo;
  int ls = 0;
  u32 nlut_used = 1;
  bool span_task = false;
  int lut_log = 0;
  const int dig_log = ALGO == ALGO_DIGIT ? (int)L.lut_log : 0;  // IPS2Ra: logarithmic digit (R33)
  const int nspl = (1 << l) - 1;
  constexpr u32 FIN = LUT_FIN;
  static_assert(KI <= 512, "bucket and splitter indices fit 9 bits");
  static_assert(S::LUT_BITS == LUT_BITS, "table size");
  if (ALGO == ALGO_TREE) {
    llo = key_from_words<Key>(L.lut_lo);
    ls = (int)L.lut_ls;
    nlut_used = L.lut_n;
    span_task = L.lut_span != 0;
    lut_log = (int)L.lut_log;
    const uint4 *src = reinterpret_cast<const uint4 *>(A.luts + L.lut_off);
    for (u32 q = tid; q < (2u << L.lut_bits) / 16; q += NT) reinterpret_cast<uint4 *>(s_lut)[q] = src[q];
  }

  const u64 n = s1 > s0 ? s1 - s0 : 0;
  unsigned short *const bidp = A.bid + L.blk_off + s0 / B;  // block buckets of this stripe (K4)
  const u64 ntiles = (n + T - 1) / T;
  u64 front = 0;
  Unit x[IPT], y[IPT], xl[IPT];
  u32 sl[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    sl[k] = NONE;
    const u64 i = s0 + tid + (u64)k * NT;
    if (i < s1) x[k] = gtask[i];
  }
  __syncthreads();

  for (u64 t = 0; t < ntiles; ++t) {
    const u64 e0 = s0 + t * T;
    const int cnt = (int)((s1 - e0) < (u64)T ? (s1 - e0) : (u64)T);
    if (wid == 0 && t + IPS4O_CLS_PF < ntiles) {
      const u64 p0 = e0 + IPS4O_CLS_PF * (u64)T;
      const u64 p1 = p0 + T < s1 ? p0 + T : s1;
      prefetch_l2(gtask + p0, (p1 - p0) * sizeof(Unit), lane, 2);
    }
    if (t + 1 < ntiles) {
      if (cnt == T && e0 + 2 * (u64)T <= s1) {
#pragma unroll
        for (int k = 0; k < IPT; ++k) y[k] = cls_load(gtask + e0 + T + tid + (u64)k * NT);
      } else {
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          const u64 i = e0 + T + tid + (u64)k * NT;
          if (i < s1) y[k] = gtask[i];
        }
      }
    }
    // ---- classify + rank (Alg. 1 batched over IPT elements; LUT start)
    u32 bkt[IPT], rank[IPT];
    {
      Key key[IPT];
#pragma unroll
      for (int k = 0; k < IPT; ++k) key[k] = elem_key<DT>(x[k]);
      if (ALGO == ALGO_TREE) {
        u32 ent[IPT];
        if (lut_log) {
          // logarithmic slots (lut_slot_of): keys below llo only outside span_task
#pragma unroll
          for (int k = 0; k < IPT; ++k) {
            const Key dk = key[k] - llo;
            const u32 q = (!span_task && key[k] < llo) ? 0u : min(lut_slot_of((u64)dk, 0, lut_log), nlut_used - 1);
            ent[k] = s_lut[q];
          }
        } else if (span_task) {
          // keys lie in [tlo, thi]; the clamp only guards the unused lanes of
          // a partial tile
#pragma unroll
          for (int k = 0; k < IPT; ++k) ent[k] = s_lut[min((u32)((key[k] - llo) >> ls), nlut_used - 1)];
        } else {
#pragma unroll
          for (int k = 0; k < IPT; ++k) {
            const Key dk = key[k] - llo;
            ent[k] = s_lut[key[k] < llo ? 0u : ((dk >> ls) < (Key)nlut_used ? (u32)(dk >> ls) : nlut_used - 1)];
          }
        }
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          if (ent[k] & FIN) {
            bkt[k] = ent[k] & 0x3FFu;
          } else {  // the slot holds splitters: lower bound among them
            const u32 a0 = ent[k] & 0x1FFu, c = ent[k] >> 9;
            const Key sv = s_spl[a0];
            if (c == 1) {
              // one splitter s_a0 in the slot; the next one lies above it
              if (sv < key[k]) {
                const u32 a1 = a0 + 1;
                bkt[k] = eq ? 2 * a1 + (a1 == (u32)nspl ? 1u : 0u) : a1;
              } else {
                bkt[k] = eq ? 2 * a0 + 1 - (key[k] < sv ? 1u : 0u) : a0;
              }
            } else {
              u32 a = a0, b = c == 63 ? (u32)nspl : a0 + c;
              while (a < b) {
                const u32 mid = (a + b) >> 1;
                if (s_spl[mid] < key[k]) a = mid + 1;
                else b = mid;
              }
              bkt[k] = eq ? 2 * a + 1 - (key[k] < s_spl[a] ? 1u : 0u) : a;
            }
          }
        }
      } else {
        if constexpr (sizeof(Key) == 8) {
          if (dig_log) {
            // sample-adaptive extractor (k_sample.cuh digit_adapt, DESIGN R33):
            // logarithmic slots of the offset from the task's lower bound;
            // the clamp only guards the unused lanes of a partial tile
#pragma unroll
            for (int k = 0; k < IPT; ++k) bkt[k] = min(lut_slot_of((u64)(key[k] - tlo), 0, dig_log), dmask);
          } else {
#pragma unroll
            for (int k = 0; k < IPT; ++k) bkt[k] = digit_of(key[k], shift, dmask);
          }
        } else {
#pragma unroll
          for (int k = 0; k < IPT; ++k) bkt[k] = digit_of(key[k], shift, dmask);
        }
      }
    }
    if (cnt == T) {
      // a warp whose 32 elements share one bucket (presorted or
      // duplicate-heavy runs: RootDup, AlmostSorted) takes its ranks with one
      // atomic instead of 32 same-address ones (tested on the first element
      // of the thread; the other elements of such a tile are tested too)
      if (__all_sync(0xffffffffu, bkt[0] == __shfl_sync(0xffffffffu, bkt[0], 0))) {
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          const u32 b0 = __shfl_sync(0xffffffffu, bkt[k], 0);
          if (__all_sync(0xffffffffu, bkt[k] == b0)) {
            u32 r0 = 0;
            if (lane == 0) r0 = atomicAdd(&s_tcnt[b0], 32u);
            rank[k] = __shfl_sync(0xffffffffu, r0, 0) + (u32)lane;
          } else {
            rank[k] = atomicAdd(&s_tcnt[bkt[k]], 1u);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < IPT; ++k) rank[k] = atomicAdd(&s_tcnt[bkt[k]], 1u);
      }
    } else {
#pragma unroll
      for (int k = 0; k < IPT; ++k) rank[k] = (tid + k * NT < cnt) ? atomicAdd(&s_tcnt[bkt[k]], 1u) : 0u;
    }
    __syncthreads();  // A: ranks final; the previous tile's blocks have been copied out

    // ---- the previous tile's leftovers enter their buffers
#pragma unroll
    for (int k = 0; k < IPT; ++k)
      if (sl[k] != NONE && IPS4O_GUARD(sl[k] < (u32)(KI * BUFS), A.err)) s_buf[sl[k]] = xl[k];

    // ---- plan: nb blocks per bucket.  The buckets that emit blocks take
    //      their block indices and staged runs with ONE atomic on the packed
    //      total (nb | staged blocks << 16): the order of a tile's blocks in
    //      the stripe is free (their buckets are recorded per block, K4 reads
    //      them), so no scan and no second barrier is needed.
    if (tid < KI) {
      // s_tcnt[j] started the tile at bucket j's buffer fill, so the rank
      // atomics returned each element's position v in the bucket's stream
      const u32 tot = s_tcnt[tid];
      s_cnt[tid] += tot - myfill;
      const u32 nb = tot / B;
      u32 pl = 0;
      if (nb) {
        const u32 pre = atomicAdd(&s_ws[KI / 32], nb | ((nb - 1) << 16));
        const u32 boff = pre & 0xFFFFu, soff = pre >> 16;
        pl = ((nb * B) << 8) | (soff << 21);
        for (u32 q = 0; q < nb; ++q) s_blkb[boff + q] = (unsigned short)(tid | (q << 9));
      }
      s_plan[tid] = pl;
      myfill = tot - nb * B;
      s_tcnt[tid] = myfill;  // the next tile's ranks start at the new fill
    }
    __syncthreads();  // B: plan visible
    const u32 nblocks = s_ws[KI / 32] & 0xFFFFu;

    // ---- scatter: buffer j, a staged block, or a leftover.  The staged
    //      runs of bucket j start at element STG0 + soff_j*B and element v
    //      (v >= B) of the bucket's tile run lands at STG0 + soff_j*B + v - B:
    //      one address formula, no per-element branches.
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const bool valid = cnt == T || tid + k * NT < cnt;
      const u32 j = valid ? bkt[k] : 0u;
      const u32 v = rank[k];
      // only elements past the buffer read the plan (about a quarter)
      const u32 pl = v >= (u32)B ? s_plan[j] : 0u;
      const u32 cut = (pl >> 8) & 0x1FFFu;
      const u32 pos = v < (u32)B ? j * BUFS + v : STG0 + (pl >> 21) * B + v - B;
      const bool keep = v < cut || v < (u32)B;
      if (valid && keep && IPS4O_GUARD(pos < STG0 + (u32)T, A.err)) s_buf[pos] = x[k];
      sl[k] = (valid && !keep) ? j * BUFS + (v - cut) : NONE;
      xl[k] = x[k];
    }
    __syncthreads();  // C: blocks complete (everyone has read the totals)
    if (tid == 0) s_ws[KI / 32] = 0;  // the next tile's block allocator

    // ---- copy the emitted blocks to the stripe's write front; bucket j's
    //      blocks are [boff_j, boff_j + nb_j): block 0 from buffer j, the
    //      rest from the stage.  One warp per block.
    {
#ifndef IPS4O_CLS_COPY_WARP
#define IPS4O_CLS_COPY_WARP 0
#endif
#if IPS4O_CLS_COPY_WARP
      for (u32 g = wid; g < nblocks; g += NWARPS) {  // a block per warp: 2 x 256 contiguous bytes
        const u32 jq = s_blkb[g];
        const u32 j = jq & 0x1FFu, q = jq >> 9;
        const Unit *src = q == 0 ? s_buf + j * BUFS : s_stage + ((s_plan[j] >> 21) + q - 1) * B;
        Unit *dst = gtask + s0 + (front + g) * B;
        if (!IPS4O_GUARD(s0 + (front + g + 1) * B <= s1, A.err)) continue;  // blocks stay in the stripe
#pragma unroll
        for (int e = 0; e < B / 32; ++e) dst[lane + 32 * e] = src[lane + 32 * e];
      }
#else
      const u32 half = (u32)lane >> 4, hl = (u32)lane & 15u;
      for (u32 g = 2 * wid + half; g < nblocks; g += 2 * NWARPS) {  // a block per half-warp
        const u32 jq = s_blkb[g];
        const u32 j = jq & 0x1FFu, q = jq >> 9;
        const Unit *src = q == 0 ? s_buf + j * BUFS : s_stage + ((s_plan[j] >> 21) + q - 1) * B;
        Unit *dst = gtask + s0 + (front + g) * B;
        if (!IPS4O_GUARD(s0 + (front + g + 1) * B <= s1, A.err)) continue;  // blocks stay in the stripe
#pragma unroll
        for (int e = 0; e < B / 16; ++e) cls_store(dst + hl + 16 * e, src[hl + 16 * e]);
      }
#endif
      // the buckets of the emitted blocks, for K4 (coalesced 2-byte stores by
      // the last warp; warp 0 issues the prefetches)
      if (wid == NWARPS - 1) {
#pragma unroll 1
        for (u32 g = lane; g < nblocks; g += 32) bidp[front + g] = (unsigned short)(s_blkb[g] & 0x1FFu);
      }
    }
    front += nblocks;
#pragma unroll
    for (int k = 0; k < IPT; ++k) x[k] = y[k];
  }
  __syncthreads();  // the last copies have read the buffers
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    if (sl[k] != NONE && IPS4O_GUARD(sl[k] < (u32)(KI * BUFS), A.err)) s_buf[sl[k]] = xl[k];
  __syncthreads();

  // ---- outputs: counts, partial fill, full blocks, partial buffers
  const u64 sbase = L.sbk_off + (u64)(stripe - L.stripe_first) * L.kidx;
  if (tid < KI) s_plan[tid] = myfill;
  __syncthreads();
  for (int j = tid; j < (int)L.kidx; j += NT) {
    A.counts[sbase + j] = s_cnt[j];
    A.pfill[sbase + j] = s_plan[j];
  }
  if (tid == 0) A.fullblocks[stripe] = (u32)front;
  for (int j = wid; j < K; j += NWARPS) {
    const int f = (int)s_plan[j];
    Unit *dst = reinterpret_cast<Unit *>(A.partials + (sbase + j) * (u64)B * Tr::D);
    for (int u = lane; u < f; u += 32) dst[u] = s_buf[j * BUFS + u];
  }
}

}  // namespace ips4o
