// k_permute.cuh -- K3 bucket boundaries + stripe-boundary fix (P:785-801,
// P:827-839) and K4 the atomic block permutation (Figs. 6-8).
#pragma once
#include "common.cuh"
#include "k_classify.cuh"

namespace ips4o {

// ------------------------------------------------------------------ K3a
// One CTA per task.  Aggregates the per-stripe counts, computes
// the exact boundaries E (prefix sum), the block-rounded delimiters
// d_j = ceil(E_j / b) * b, the full blocks per bucket, and initialises
// the packed (w, r) words: w_j = d_j / b, r_j = w_j + f_j - 1.
constexpr int BND_THREADS = 256;

template <int DT>
__global__ void __launch_bounds__(BND_THREADS) boundaries_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  constexpr int KI = Tr::KIDX, B = Tr::B;
  static_assert(KI <= BND_THREADS, "one thread per bucket");
  __shared__ u32 ws[BND_THREADS / 32 + 1];
  const u32 ti = blockIdx.x;
  LevelTask &L = A.tasks[ti];
  const int K = (int)L.K;
  const int j = threadIdx.x;
  u32 c = 0, f = 0;
  if (j < K) {
    for (u32 s = 0; s < L.nstripes; ++s) {
      const u64 slot = L.sbk_off + (u64)s * L.kidx + j;
      u32 cs = A.counts[slot];
      c += cs;
      f += (cs - A.pfill[slot]) / B;
    }
  }
  u32 total;
  u32 pre = block_exclusive_scan<BND_THREADS>(c, ws, &total);
  const u64 bo = L.bucket_off;
  if (j < K) {
    A.E[bo + j] = pre;
    A.fblk[bo + j] = f;
    u64 w = ((u64)pre + B - 1) / B;
    i64 r = (i64)w + (i64)f - 1;
    A.wr[(bo + j) * WR_STRIDE] = (w << 32) | (u64)(r + (i64)RBIAS);
    A.wr[(bo + j) * WR_STRIDE + 4] = 0;  // readers
  }
  if (j == 0) {
    A.E[bo + K] = L.t.size;
    A.ovf_used[ti] = 0xFFFFFFFFu;
  }
}

// ------------------------------------------------------------------ K3b
// Stripe-boundary fix, one CTA per stripe.  After classification
// every stripe holds F_c full blocks followed by empty blocks.  For each bucket
// j whose full-block prefix [d_j/b, d_j/b + f_j) reaches into this stripe's
// empty tail, the CTA fills those holes with the LAST full blocks of bucket j
// ("moves the last full block in the bucket into the first empty
// block"), skipping as many as holes of bucket j in preceding stripes
// (P:836-838).  Afterwards every bucket region is "full blocks, then empty".
constexpr int FIX_THREADS = 256;

template <int DT>
__global__ void __launch_bounds__(FIX_THREADS) stripe_fix_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Unit = typename Tr::Unit;
  constexpr int D = Tr::D, B = Tr::B;
  constexpr int NU = B * D / (int)sizeof(Unit);
  constexpr int NWARPS = FIX_THREADS / 32;
  extern __shared__ __align__(16) u32 s_cum[];  // [nstripes of task + 1]
  __shared__ u32 ws[FIX_THREADS / 32 + 1];
  const u32 stripe = blockIdx.x;
  const u32 ti = A.stripe_task[stripe];
  const LevelTask &L = A.tasks[ti];
  const u32 c = stripe - L.stripe_first;
  const u64 SB = L.stripe_elems / B;                // block slots per stripe
  const u64 nblk_total = (L.t.size + B - 1) / B;     // incl. a partial last block
  const u64 c_lo = (u64)c * SB;
  const u64 c_hi = (c_lo + SB < nblk_total) ? c_lo + SB : nblk_total;
  const u64 F = A.fullblocks[stripe];
  const u64 e0 = c_lo + F;  // empty tail [e0, c_hi)
  if (e0 >= c_hi) return;
  const int K = (int)L.K;
  const u64 bo = L.bucket_off;
  char *gtask = A.base + L.t.begin * (u64)D;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  // first bucket whose prefix end d_j/b + f_j exceeds e0 (prefix ends are
  // non-decreasing because bucket j's full blocks fit its region)
  int jlo = 0, jhi = K;
  while (jlo < jhi) {
    int mid = (jlo + jhi) >> 1;
    u64 pe = (A.E[bo + mid] + B - 1) / B + A.fblk[bo + mid];
    if (pe <= e0) jlo = mid + 1;
    else jhi = mid;
  }
  for (int j = jlo; j < K; ++j) {
    const u64 r0 = (A.E[bo + j] + B - 1) / B;       // region start (blocks)
    const u64 r1 = (A.E[bo + j + 1] + B - 1) / B;   // region end
    const u64 pe = r0 + A.fblk[bo + j];             // prefix end
    if (r0 >= c_hi) break;
    const u64 h0 = e0 > r0 ? e0 : r0;
    const u64 h1 = c_hi < pe ? c_hi : pe;
    if (h0 >= h1) continue;                          // no holes of j here
    // stripes overlapping region [r0, r1)
    const u64 ca = r0 / SB, cb = (r1 - 1) / SB;
    const u32 nst = (u32)(cb - ca + 1);
    // full positions of stripe cc within the region: [max(cc*SB, r0), min(cc*SB+F_cc, r1))
    // (1) holes of bucket j before h0: (h0 - r0) - #full positions in [r0, h0)
    // (2) sources (full positions >= pe) per stripe, cumulated from the LAST stripe
    u32 before = 0;
    for (u32 base = 0; base < nst; base += FIX_THREADS) {
      u32 idx = base + threadIdx.x;
      u32 srcs = 0, fb = 0;
      if (idx < nst) {
        u64 cc = ca + idx;
        u64 f0 = cc * SB > r0 ? cc * SB : r0;
        u64 fe = cc * SB + A.fullblocks[L.stripe_first + cc];
        u64 f1 = fe < r1 ? fe : r1;
        if (f1 > f0) {
          u64 x1 = f1 < h0 ? f1 : h0;
          fb = x1 > f0 ? (u32)(x1 - f0) : 0;           // full positions in [r0, h0)
          u64 s0_ = f0 > pe ? f0 : pe;
          srcs = f1 > s0_ ? (u32)(f1 - s0_) : 0;       // full positions in [pe, r1)
        }
      }
      // store sources reversed so that a forward scan cumulates from the end
      if (idx < nst) s_cum[nst - 1 - idx] = srcs;
      u32 tot;
      block_exclusive_scan<FIX_THREADS>(fb, ws, &tot);
      before += tot;
    }
    __syncthreads();
    // exclusive scan of s_cum[0..nst) in place (chunked)
    u32 carry = 0;
    for (u32 base = 0; base < nst; base += FIX_THREADS) {
      u32 idx = base + threadIdx.x;
      u32 v = idx < nst ? s_cum[idx] : 0;
      u32 tot;
      u32 p = block_exclusive_scan<FIX_THREADS>(v, ws, &tot);
      if (idx < nst) s_cum[idx] = carry + p;
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) s_cum[nst] = carry;
    __syncthreads();
    const u64 skip = (h0 - r0) - before;
    const u64 nholes = h1 - h0;
    // move: hole h0+i  <-  source number skip+i counted from the end
    for (u64 i = wid; i < nholes; i += NWARPS) {
      const u32 g = (u32)(skip + i);
      // reversed stripe index rr with s_cum[rr] <= g < s_cum[rr+1]
      int lo = 0, hi = (int)nst;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (s_cum[mid] <= g) lo = mid + 1;
        else hi = mid;
      }
      const int rr = lo - 1;
      const u64 cc = ca + (nst - 1 - rr);
      u64 fe = cc * SB + A.fullblocks[L.stripe_first + cc];
      u64 f1 = fe < r1 ? fe : r1;
      const u64 src = f1 - 1 - (g - s_cum[rr]);
      const u64 dstb = h0 + i;
      const Unit *s = reinterpret_cast<const Unit *>(gtask + src * B * D);
      Unit *d = reinterpret_cast<Unit *>(gtask + dstb * B * D);
      for (int u = lane; u < NU; u += 32) d[u] = s[u];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ K4
// Block permutation.  Agents are warps; each holds its two swap
// buffers in registers.  Per bucket a packed 64-bit word (w, r+RBIAS)
// is read and modified with one atomic and a reader
// counter implements "threads are only allowed to write to empty blocks if no
// other threads are currently reading from the bucket".
constexpr int PERM_WARPS = 8;
constexpr int PERM_THREADS = PERM_WARPS * 32;

template <int DT, int ALGO>
__device__ __forceinline__ u32 classify_one(const typename Traits<DT>::Key *tree,
                                            const typename Traits<DT>::Key *spl, int l, int eq,
                                            int shift, u32 dmask, const char *e) {
  using Key = typename Traits<DT>::Key;
  Key k = Traits<DT>::key(e);
  if (ALGO == ALGO_TREE) return tree_bucket<Key>(tree, spl, l, eq, k);
  return digit_of(k, shift, dmask);
}

template <int DT, int ALGO>
__global__ void __launch_bounds__(PERM_THREADS) permute_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  using Unit = typename Tr::Unit;
  constexpr int D = Tr::D, B = Tr::B, KI = Tr::KIDX;
  constexpr int NU = B * D / (int)sizeof(Unit);
  constexpr int NPL = (NU + 31) / 32;
  __shared__ Key s_tree[KI], s_spl[KI];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 cta = blockIdx.x;
  const u32 ti = A.perm_task[cta];
  const LevelTask &L = A.tasks[ti];
  const int K = (int)L.K, l = (int)L.l, eq = (int)L.equality, shift = L.shift;
  const u32 dmask = L.K - 1;
  if (ALGO == ALGO_TREE) {
    const Key *gt = reinterpret_cast<const Key *>(A.trees) + (size_t)ti * 2 * KI;
    for (int i = threadIdx.x; i < (1 << l); i += PERM_THREADS) {
      s_tree[i] = gt[i];
      s_spl[i] = gt[KI + i];
    }
  }
  __syncthreads();
  if (K <= 1) return;
  char *gtask = A.base + L.t.begin * (u64)D;
  const u64 size = L.t.size;
  const u64 pblk = (size % B) ? size / B : ~0ull;  // partial last block -> overflow
  char *ovf = A.overflow + (size_t)ti * B * D;
  u64 *wr = A.wr + L.bucket_off * WR_STRIDE;
  const u32 agent = (cta - L.perm_first) * PERM_WARPS + wid;
  const u32 nagents = L.nperm * PERM_WARPS;
  int p = (int)(((u64)agent * (u64)K) / nagents);  // P:847 starting points spread

  auto blk_ptr = [&](u64 x) -> Unit * {
    return reinterpret_cast<Unit *>(x == pblk ? ovf : gtask + x * (u64)B * D);
  };
  auto load_blk = [&](u64 x, Unit(&r)[NPL]) {
    const Unit *s = blk_ptr(x);
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      int u = lane + 32 * i;
      if (u < NU) r[i] = s[u];
    }
  };
  auto store_blk = [&](u64 x, const Unit(&r)[NPL]) {
    Unit *d = blk_ptr(x);
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      int u = lane + 32 * i;
      if (u < NU) d[u] = r[i];
    }
  };
  auto first_bucket = [&](u64 x) -> u32 {
    u32 b = 0;
    if (lane == 0) b = classify_one<DT, ALGO>(s_tree, s_spl, l, eq, shift, dmask, (const char *)blk_ptr(x));
    return __shfl_sync(0xffffffffu, b, 0);
  };

  Unit buf0[NPL], buf1[NPL];
  int misses = 0;  // consecutive primary buckets without unprocessed blocks
  for (;;) {
    // ---- fetch an unprocessed block from the primary bucket
    u64 x = ~0ull;
    while (misses < K) {
      u64 got = 0;
      if (lane == 0) {
        u64 cur = ld_relaxed_u64(&wr[(u64)p * WR_STRIDE]);
        i64 w = (i64)(cur >> 32), r = (i64)(cur & 0xFFFFFFFFull) - (i64)RBIAS;
        if (r >= w) {
          atomicAdd(&wr[(u64)p * WR_STRIDE + 4], 1ull);
          __threadfence();
          u64 old = atomicAdd(&wr[(u64)p * WR_STRIDE], ~0ull);  // r -= 1
          w = (i64)(old >> 32);
          r = (i64)(old & 0xFFFFFFFFull) - (i64)RBIAS;
          if (r >= w) got = 1ull << 63 | (u64)r;
          else atomicAdd(&wr[(u64)p * WR_STRIDE + 4], ~0ull);
        }
      }
      got = __shfl_sync(0xffffffffu, got, 0);
      if (got) {
        x = got & ~(1ull << 63);
        break;
      }
      p = p + 1 == K ? 0 : p + 1;
      ++misses;
    }
    if (x == ~0ull) break;  // a whole cycle without work: done
    misses = 0;
    load_blk(x, buf0);
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(&wr[(u64)p * WR_STRIDE + 4], ~0ull);  // reader done
    u32 dest;
    {
      // the key sits in the first KEY_UNITS units, i.e. on lanes 0..KEY_UNITS-1
      Unit ku[Tr::KEY_UNITS];
      if constexpr (Tr::KEY_UNITS == 1) {
        ku[0] = buf0[0];
      } else {
#pragma unroll
        for (int q = 0; q < Tr::KEY_UNITS; ++q) ku[q] = __shfl_sync(0xffffffffu, buf0[0], q);
      }
      u32 b = 0;
      if (lane == 0) {
        Key k = Tr::key(reinterpret_cast<const char *>(ku));
        b = ALGO == ALGO_TREE ? tree_bucket<Key>(s_tree, s_spl, l, eq, k) : digit_of(k, shift, dmask);
      }
      dest = __shfl_sync(0xffffffffu, b, 0);
    }
    // ---- place buf0 into dest, swapping as long as dest has unprocessed blocks
    for (;;) {
      u64 old = 0;
      if (lane == 0) old = atomicAdd(&wr[(u64)dest * WR_STRIDE], 1ull << 32);  // w += 1
      old = __shfl_sync(0xffffffffu, old, 0);
      const i64 w = (i64)(old >> 32), r = (i64)(old & 0xFFFFFFFFull) - (i64)RBIAS;
      if (w <= r) {
        // unprocessed block at w: skip it if it is already in place
        u32 b2 = first_bucket((u64)w);
        if (b2 == dest) continue;
        load_blk((u64)w, buf1);
        store_blk((u64)w, buf0);
#pragma unroll
        for (int i = 0; i < NPL; ++i) buf0[i] = buf1[i];
        dest = b2;
        continue;
      }
      // empty block at w: wait until nobody reads from dest
      if (lane == 0) {
        while (ld_acquire_u64(&wr[(u64)dest * WR_STRIDE + 4]) != 0) __nanosleep(64);
      }
      __syncwarp();
      store_blk((u64)w, buf0);
      if ((u64)w == pblk && lane == 0) A.ovf_used[ti] = dest;
      break;
    }
  }
}

}  // namespace ips4o
