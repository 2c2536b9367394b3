// k_permute.cuh -- K3 bucket boundaries + stripe-boundary fix (P:785-801,
// P:827-839) and K4 the atomic block permutation (Figs. 6-8).
#pragma once
#include "common.cuh"
#include "k_classify.cuh"
#include "k_cleanup.cuh"

namespace ips4o {

// ------------------------------------------------------------------ K3a
// One CTA per task.  Aggregates the per-stripe counts, computes
// the exact boundaries E (prefix sum), the block-rounded delimiters
// d_j = ceil(E_j / b) * b, the full blocks per bucket, and initialises
// the packed (w, r) words: w_j = d_j / b, r_j = w_j + f_j - 1.
// Then the same CTA schedules the task's buckets (K6, schedule_task).
constexpr int BND_THREADS = 1024;

template <int DT, int ALGO>
__global__ void __launch_bounds__(BND_THREADS) boundaries_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  constexpr int KI = Tr::KIDX, B = Tr::B;
  if (A.go && *A.go == 0) return;  // round 0 of an easy input (k_plan.cuh)
  KTIMER(A.tslot, KS_BOUND);
  constexpr int QB = BND_THREADS / KI;  // threads per bucket, each over a share of the stripes
  static_assert(KI * QB == BND_THREADS, "whole threads per bucket");
  __shared__ u32 ws[BND_THREADS / 32 + 1];
  __shared__ u64 s_E[KI + 1];
  __shared__ u32 s_pq[QB][KI];
  const u32 ti = blockIdx.x;
  LevelTask &L = A.tasks[ti];
  const int K = (int)L.K;
  const int j = threadIdx.x % KI, qb = threadIdx.x / KI;
  // prefix of the stripes' full-block counts (for F(x) below)
  u32 carry = 0;
  for (u32 b0 = 0; b0 < L.nstripes; b0 += BND_THREADS) {
    u32 idx = b0 + threadIdx.x;
    u32 v = idx < L.nstripes ? A.fullblocks[L.stripe_first + idx] : 0;
    u32 tot;
    u32 p = block_exclusive_scan<BND_THREADS>(v, ws, &tot);
    if (idx < L.nstripes) A.fcum[L.stripe_first + idx] = carry + p;
    carry += tot;
  }
  // per bucket: total count over the stripes and the exclusive
  // prefix over the stripes of the partial-buffer fills (cleanup, K5b);
  // QB threads per bucket, each over a contiguous share of the stripes
  const u32 ns = L.nstripes;
  const u32 s_lo = (u32)(((u64)ns * qb) / QB), s_hi = (u32)(((u64)ns * (qb + 1)) / QB);
  u32 c = 0, pc = 0;
  if (j < K) {
    for (u32 s = s_lo; s < s_hi; ++s) {
      const u64 slot = L.sbk_off + (u64)s * L.kidx + j;
      c += A.counts[slot];
      pc += A.pfill[slot];
    }
    s_pq[qb][j] = pc;
  }
  __syncthreads();
  if (j < K) {
    u32 run = 0;
    for (int q = 0; q < qb; ++q) run += s_pq[q][j];
    for (u32 s = s_lo; s < s_hi; ++s) {
      const u64 slot = L.sbk_off + (u64)s * L.kidx + j;
      A.pcum[slot] = run;
      run += A.pfill[slot];
    }
    if (qb == QB - 1) A.ptot[L.bucket_off + j] = run;
  }
  __syncthreads();
  s_pq[qb][j] = j < K ? c : 0u;  // reuse: per-share counts
  __syncthreads();
  if (qb == 0) {
    c = 0;
    for (int q = 0; q < QB; ++q) c += s_pq[q][j];
  }
  u32 total;
  u32 pre = block_exclusive_scan<BND_THREADS>(qb == 0 && j < K ? c : 0u, ws, &total);
  if (qb == 0 && j < K) s_E[j] = pre;
  if (threadIdx.x == 0) s_E[K] = L.t.size;
  __syncthreads();
  const u64 bo = L.bucket_off;
  if (qb == 0 && j < K) {
    // region j = blocks [ceil(E_j/b), ceil(E_{j+1}/b)); fr = full positions in it
    const u64 SB = L.stripe_elems / B;
    const u64 r0 = (s_E[j] + B - 1) / B, r1 = (s_E[j + 1] + B - 1) / B;
    auto F = [&](u64 x) -> u64 {  // full block positions in [0, x)
      u64 cc = x / SB;
      if (cc >= L.nstripes) return carry;
      u64 fb = A.fullblocks[L.stripe_first + cc];
      u64 in = x - cc * SB;
      return A.fcum[L.stripe_first + cc] + (in < fb ? in : fb);
    };
    const u64 fr = F(r1) - F(r0);
    A.E[bo + j] = s_E[j];
    A.fblk[bo + j] = (u32)fr;
    const i64 r = (i64)r0 + (i64)fr - 1;
    A.wr[(bo + j) * WR_STRIDE] = (r0 << 32) | (u64)(r + (i64)RBIAS);
    A.wr[(bo + j) * WR_STRIDE + 1] = r0 + fr;  // prefix end (formerly full positions)
  }
  if (threadIdx.x == 0) {
    A.E[bo + K] = L.t.size;
    A.ovf_used[ti] = 0xFFFFFFFFu;
  }
  if (!A.capture) {
    __syncthreads();
    schedule_task<DT, ALGO>(A, ti, s_E);
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
  if (A.go && *A.go == 0) return;  // round 0 of an easy input (k_plan.cuh)
  KTIMER(A.tslot, KS_FIX);
  using Unit = typename Tr::Unit;
  constexpr int D = Tr::D, B = Tr::B;
  constexpr int NU = B * D / (int)sizeof(Unit);
  constexpr int NWARPS = FIX_THREADS / 32;
  const u32 stripe = blockIdx.x;
  const u32 ti = A.stripe_task[stripe];
  const LevelTask &L = A.tasks[ti];
  const u32 c = stripe - L.stripe_first;
  const u64 SB = L.stripe_elems / B;                // block slots per stripe
  const u64 nblk_total = (L.t.size + B - 1) / B;     // incl. a partial last block
  const u64 c_lo = (u64)c * SB;
  const u64 c_hi = (c_lo + SB < nblk_total) ? c_lo + SB : nblk_total;
  const u64 Fc = A.fullblocks[stripe];
  const u64 e0 = c_lo + Fc;  // empty tail [e0, c_hi)
  if (e0 >= c_hi) return;
  const int K = (int)L.K;
  const u64 bo = L.bucket_off;
  char *gtask = A.base + L.t.begin * (u64)D;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 sf = L.stripe_first, nst = L.nstripes;
  const u64 ftot = A.fcum[sf + nst - 1] + A.fullblocks[sf + nst - 1];
  auto F = [&](u64 x) -> u64 {  // full block positions in [0, x) after classification
    u64 cc = x / SB;
    if (cc >= nst) return ftot;
    u64 fb = A.fullblocks[sf + cc];
    u64 in = x - cc * SB;
    return A.fcum[sf + cc] + (in < fb ? in : fb);
  };
  auto select = [&](u64 q) -> u64 {  // position of the full block of rank q
    u32 lo = 0, hi = nst;  // last stripe with fcum <= q
    while (hi - lo > 1) {
      u32 mid = (lo + hi) >> 1;
      if (A.fcum[sf + mid] <= q) lo = mid;
      else hi = mid;
    }
    return (u64)lo * SB + (q - A.fcum[sf + lo]);
  };

  // first bucket whose prefix end r0_j + fr_j exceeds e0 (prefix ends are
  // non-decreasing: region j's full positions fit region j)
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
    // holes of region j before h0 belong to preceding stripes
    const u64 skip = (h0 - r0) - (F(h0) - F(r0));
    const u64 Fr1 = F(r1);
    const u64 nholes = h1 - h0;
    // hole h0+i <- the (skip+i)-th full block of region j counted from its end,
    // i.e. the full block of task-wide rank Fr1 - 1 - (skip+i)
    for (u64 i = wid; i < nholes; i += NWARPS) {
      const u64 q = Fr1 - 1 - (skip + i);
      const u64 src = select(q);
      const u64 dstb = h0 + i;
      if (!IPS4O_GUARD(src < nblk_total && dstb < nblk_total && (dstb + 1) * B <= L.t.size, A.err)) continue;
      const Unit *s = reinterpret_cast<const Unit *>(gtask + src * B * D);
      Unit *d = reinterpret_cast<Unit *>(gtask + dstb * B * D);
      for (int u = lane; u < NU; u += 32) d[u] = s[u];
      if (lane == 0) A.bid[L.blk_off + dstb] = A.bid[L.blk_off + src];
    }
  }
}

// ------------------------------------------------------------------ K4
// Block permutation.  Agents are warps; each holds its two swap
// buffers in registers.  Per bucket a packed 64-bit word (w, r+RBIAS)
// is read and modified with ONE atomic, which gives every agent a consistent
// view of both pointers.
//
// Reader tracking: a writer may fill an empty block only after the
// agent that read that block (when w and r crossed) has finished reading it.
// The paper counts readers per bucket; here every block position carries a
// "read done" byte that the reader sets with a release store after its loads
// completed, and a writer that targets a formerly full position waits on that
// byte with acquire loads.  Same guarantee, no shared counters, no fences
// (DESIGN "Permutation on the GPU").
//
// The bucket of a block is not recomputed from its first key: K2 records it
// per block position when it flushes the block (K3 moves it with the block),
// so an agent learns where a swapped-out block goes from a 2-byte load that
// returns long before the block, and issues the next atomic while the block
// is still in flight.
#ifndef IPS4O_PERM_WARPS
#define IPS4O_PERM_WARPS 8
#endif
constexpr int PERM_WARPS = IPS4O_PERM_WARPS;
#ifndef IPS4O_PERM_MINB
#define IPS4O_PERM_MINB 8  // full occupancy: 32 registers (a few bytes spill)
#endif
#ifndef IPS4O_PERM_HOP_WINDOW
#define IPS4O_PERM_HOP_WINDOW 64
#endif
constexpr u32 PERM_HOP_WINDOW = IPS4O_PERM_HOP_WINDOW;  // tasks an idle agent may look ahead
#ifndef IPS4O_PERM_TREE_PACE_NS
#define IPS4O_PERM_TREE_PACE_NS 0
#endif
#ifndef IPS4O_PERM_DIGIT_PACE_NS
#define IPS4O_PERM_DIGIT_PACE_NS 100
#endif
constexpr int PERM_DIGIT_PACE_NS = IPS4O_PERM_DIGIT_PACE_NS;

#ifdef IPS4O_PERM_CLOCKS
// debug: per-warp cycles spent in fetch (incl. misses), swap atomics, swap
// loads, empty-write waits, and number of swap steps
__device__ unsigned long long g_perm_clk[6];
#define PCLK_DECL long long pc_t0_ = 0, pc_acc_[6] = {0, 0, 0, 0, 0, 0};
#define PCLK_START() pc_t0_ = clock64()
#define PCLK_ADD(i) pc_acc_[i] += clock64() - pc_t0_
#define PCLK_CNT(i) pc_acc_[i] += 1
#define PCLK_FLUSH() \
  if (lane == 0)     \
    for (int q_ = 0; q_ < 6; ++q_) atomicAdd(&g_perm_clk[q_], (unsigned long long)pc_acc_[q_]);
#else
#define PCLK_DECL
#define PCLK_START()
#define PCLK_ADD(i)
#define PCLK_CNT(i)
#define PCLK_FLUSH()
#endif

#ifdef IPS4O_PERM_STATS
// debug counters: fetch attempts, fetches, misses, swaps, skips, empty writes,
// waits (empty writes that polled rdone), poll iterations
__device__ unsigned long long g_perm_stats[8];
#define PSTAT(i, v) atomicAdd(&g_perm_stats[i], (unsigned long long)(v))
#else
#define PSTAT(i, v)
#endif
constexpr int PERM_THREADS = PERM_WARPS * 32;

__device__ __forceinline__ void st_release_u8(unsigned char *p, unsigned v) {
  asm volatile("st.release.gpu.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u8(const unsigned char *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u8 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <class Unit> __device__ __forceinline__ Unit ld_cg_unit(const Unit *p);
template <> __device__ __forceinline__ u64 ld_cg_unit<u64>(const u64 *p) {
  u64 v;
  asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ u32 ld_cg_unit<u32>(const u32 *p) {
  u32 v;
  asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ uint4 ld_cg_unit<uint4>(const uint4 *p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <class Unit> __device__ __forceinline__ Unit shfl_unit(const Unit &u, int src) {
  return __shfl_sync(0xffffffffu, u, src);
}
template <> __device__ __forceinline__ uint4 shfl_unit<uint4>(const uint4 &u, int src) {
  return make_uint4(__shfl_sync(0xffffffffu, u.x, src), __shfl_sync(0xffffffffu, u.y, src),
                    __shfl_sync(0xffffffffu, u.z, src), __shfl_sync(0xffffffffu, u.w, src));
}

template <class Unit> __device__ __forceinline__ u32 fold32(const Unit &u);
template <> __device__ __forceinline__ u32 fold32<u64>(const u64 &u) { return (u32)u ^ (u32)(u >> 32); }
template <> __device__ __forceinline__ u32 fold32<u32>(const u32 &u) { return u; }
template <> __device__ __forceinline__ u32 fold32<uint4>(const uint4 &u) { return u.x ^ u.y ^ u.z ^ u.w; }

__device__ __forceinline__ u32 ld_relaxed_u32(const u32 *p) {
  u32 v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Agents (warps) start on the task of their CTA (agents per task in
// proportion to its size) and, once no block of it can be fetched
// any more, move on to the next unfinished task of the level, so that the
// level ends when the last block is placed rather than when the slowest task's
// own agents are done.  The protocol per task is unchanged; it does not care
// which agents take part.
template <int DT, int ALGO>
__global__ void __launch_bounds__(PERM_THREADS, IPS4O_PERM_MINB) permute_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  using Unit = typename Tr::Unit;
  constexpr int D = Tr::D, B = Tr::B, KI = Tr::KIDX;
  constexpr int NU = B * D / (int)sizeof(Unit);
  constexpr int NPL = (NU + 31) / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (A.go && *A.go == 0) return;  // round 0 of an easy input (k_plan.cuh)
  KTIMER(A.tslot, KS_PERM);
  const u32 home = A.perm_task[blockIdx.x];
  if (A.dbg_one_agent && wid != 0) return;
  const u32 agent = (blockIdx.x - A.tasks[home].perm_first) * PERM_WARPS + wid;
  PCLK_DECL

  u32 ti = home;
  for (u32 hop = 0; hop < A.ntasks; ++hop) {
    if (hop > 0) {
      if (A.dbg_one_agent) break;
      // next unfinished task among the following PERM_HOP_WINDOW tasks (32
      // done flags per probe; a bounded window keeps levels with thousands of
      // small tasks from scanning all of them)
      u32 nxt = ~0u;
      const u32 lim = A.ntasks < PERM_HOP_WINDOW + 1 ? A.ntasks : PERM_HOP_WINDOW + 1;
      for (u32 base = 1; base < lim && nxt == ~0u; base += 32) {
        u32 q = ti + base + lane;
        q = q >= A.ntasks ? q - A.ntasks : q;
        const bool open = base + lane < lim && ld_relaxed_u32(&A.task_done[q]) == 0;
        const unsigned m = __ballot_sync(0xffffffffu, open);
        if (m) nxt = __shfl_sync(0xffffffffu, q, __ffs(m) - 1);
      }
      if (nxt == ~0u) break;
      hop += (nxt >= ti ? nxt - ti : nxt + A.ntasks - ti) - 1;
      ti = nxt;
    }
    const LevelTask &L = A.tasks[ti];
    const int K = (int)L.K, shift = L.shift;
    const u32 dmask = L.K - 1;
    if (K <= 1) {
      if (lane == 0) atomicExch(&A.task_done[ti], 1u);
      continue;
    }
    const bool local = ti == home;
    char *gtask = A.base + L.t.begin * (u64)D;
    const u64 size = L.t.size;
    const u64 pblk = (size % B) ? size / B : ~0ull;  // partial last block -> overflow
    char *ovf = A.overflow + (size_t)ti * B * D;
    u64 *wr = A.wr + L.bucket_off * WR_STRIDE;
    unsigned char *rdone = A.rdone + L.blk_off;
    const unsigned short *bid = A.bid + L.blk_off;  // bucket of each full block (K2/K3)
    const u32 nagents = A.dbg_one_agent ? 1 : L.nperm * PERM_WARPS;
    // P:847 starting points spread over the buckets
    int p = local ? (int)(((u64)agent * (u64)K) / nagents) : (int)((agent * 97u + blockIdx.x) % (u32)K);

    auto blk_ptr = [&](u64 x) -> Unit * {
      return reinterpret_cast<Unit *>(x == pblk ? ovf : gtask + x * (u64)B * D);
    };
    // all loads of a block are issued back to back (volatile: the compiler
    // may not sink the later ones past the bucket test that needs the first)
    auto load_blk = [&](u64 x, Unit(&r)[NPL]) {
      const Unit *src = blk_ptr(x);
#pragma unroll
      for (int i = 0; i < NPL; ++i) {
        int u = lane + 32 * i;
        if (u < NU) r[i] = ld_cg_unit(src + u);
      }
    };
    auto store_blk = [&](u64 x, const Unit(&r)[NPL]) {
      if (!IPS4O_GUARD(x < (size + B - 1) / B, A.err)) return;  // block positions of the task
      Unit *d = blk_ptr(x);
#pragma unroll
      for (int i = 0; i < NPL; ++i) {
        int u = lane + 32 * i;
        if (u < NU) d[u] = r[i];
      }
    };
    // Pacing: with nothing between a block's arrival and the next atomic,
    // agents of the digit path return to the hot (w, r) words so fast that
    // same-address atomics queue up at L2 and every step slows ~10x
    // (measured: 7100-cycle atomics vs ~650 with a ~100 ns gap).
    // The digit path therefore takes a block's bucket from its first key
    // once the block has arrived (one shift), and sleeps briefly.
    auto bucket = [&](u32 bv, const Unit(&r)[NPL]) -> u32 {
      if constexpr (ALGO == ALGO_DIGIT) {
        Unit ku[Tr::KEY_UNITS];
        if constexpr (Tr::KEY_UNITS == 1) {
          ku[0] = r[0];
        } else {
#pragma unroll
          for (int q = 0; q < Tr::KEY_UNITS; ++q) ku[q] = shfl_unit(r[0], q);
        }
        if (lane == 0) {
          const Key kx = Tr::key(reinterpret_cast<const char *>(ku));
          bv = digit_of(kx, shift, dmask);
          if constexpr (sizeof(Key) == 8) {
            if (L.lut_log) bv = min(lut_slot_of((u64)(kx - key_from_words<Key>(L.t.lo)), 0, (int)L.lut_log), dmask);
          }
          __nanosleep(PERM_DIGIT_PACE_NS);
        }
      } else {
#if IPS4O_PERM_TREE_PACE_NS > 0
        if (lane == 0) __nanosleep(IPS4O_PERM_TREE_PACE_NS);  // tuning experiment
#endif
      }
      return __shfl_sync(0xffffffffu, bv, 0);
    };
    // Place the block held in `hold` (bucket dest): w += 1 on dest; an
    // unprocessed block at w is swapped out into `spare` (its bucket comes
    // from the block-bucket array, so the next atomic is issued while the
    // block itself is still in flight) unless it already belongs to dest
    // (P:902-903); an empty block at w is written once its reader is done
    // (P:898).  Returns 0 = placed, 1 = swapped (spare now holds
    // the block to place, dest its bucket), 2 = skipped (hold unchanged).
    auto place = [&](Unit(&hold)[NPL], Unit(&spare)[NPL], u32 &dest) -> int {
      u64 old = 0;
      PCLK_START();
      if (lane == 0) old = atomicAdd(&wr[(u64)dest * WR_STRIDE], 1ull << 32);  // w += 1
      old = __shfl_sync(0xffffffffu, old, 0);
      PCLK_ADD(1);
      PCLK_CNT(4);
      const i64 w = (i64)(old >> 32), r = (i64)(old & 0xFFFFFFFFull) - (i64)RBIAS;
      if (w <= r) {
        PCLK_START();
        const u32 bv = ALGO == ALGO_TREE && lane == 0 ? (u32)__ldg(bid + w) : 0u;
        load_blk((u64)w, spare);
        const u32 b2 = bucket(bv, spare);
        PCLK_ADD(2);
        if (b2 == dest) {
          if (lane == 0) PSTAT(4, 1);
          return 2;
        }
        if (lane == 0) PSTAT(3, 1);
        store_blk((u64)w, hold);  // the loads of block w precede this store (same lanes, same addresses)
        dest = b2;
        return 1;
      }
      PCLK_START();
      if (lane == 0) {
        const u64 pe = wr[(u64)dest * WR_STRIDE + 1];  // prefix end of region dest
        PSTAT(5, 1);
        if ((u64)w < pe) {
          PSTAT(6, 1);
          while (ld_acquire_u8(rdone + w) == 0) {
            PSTAT(7, 1);
            __nanosleep(32);
          }
        }
        if ((u64)w == pblk) A.ovf_used[ti] = dest;
      }
      __syncwarp();
      PCLK_ADD(3);
      store_blk((u64)w, hold);
      return 0;
    };

    Unit buf0[NPL], buf1[NPL];
    for (;;) {
      // ---- fetch an unprocessed block: the primary bucket p
      //      first; when it has none, the 32 lanes probe 32 buckets at a time
      u64 x = ~0ull;
      PCLK_START();
      for (;;) {
        u64 got = 0;
        if (lane == 0) {
          u64 cur = ld_relaxed_u64(&wr[(u64)p * WR_STRIDE]);
          i64 w = (i64)(cur >> 32), r = (i64)(cur & 0xFFFFFFFFull) - (i64)RBIAS;
          if (r >= w) {
            PSTAT(0, 1);
            u64 old = atomicAdd(&wr[(u64)p * WR_STRIDE], ~0ull);  // r -= 1
            w = (i64)(old >> 32);
            r = (i64)(old & 0xFFFFFFFFull) - (i64)RBIAS;
            if (r >= w) got = 1ull << 63 | (u64)r;
          }
        }
        got = __shfl_sync(0xffffffffu, got, 0);
        if (got) {
          x = got & ~(1ull << 63);
          if (lane == 0) PSTAT(1, 1);
          break;
        }
        if (lane == 0) PSTAT(2, 1);
        // r and w only move towards each other: a bucket seen without work
        // stays without work, so one sweep without any means the task is done
        int found = -1;
        for (int base = 0; base < K && found < 0; base += 32) {
          int q = p + base + lane;
          q = q >= K ? q - K : q;
          bool has = false;
          if (base + lane < K) {
            const u64 cur = ld_relaxed_u64(&wr[(u64)q * WR_STRIDE]);
            has = (i64)(cur & 0xFFFFFFFFull) - (i64)RBIAS >= (i64)(cur >> 32);
          }
          const unsigned m = __ballot_sync(0xffffffffu, has);
          if (m) found = __shfl_sync(0xffffffffu, q, __ffs(m) - 1);
        }
        if (found < 0) break;
        p = found;
      }
      if (x == ~0ull) break;
      PCLK_ADD(0);
      const u32 bx = ALGO == ALGO_TREE && lane == 0 ? (u32)__ldg(bid + x) : 0u;
      load_blk(x, buf0);
      u32 dest = bucket(bx, buf0);
      {
        // every lane's loads have returned once the reduction has its
        // operands; then publish "block x read" (release) for a writer
        u32 v = 0;
#pragma unroll
        for (int i = 0; i < NPL; ++i) v ^= fold32<Unit>(buf0[i]);
        v = __reduce_xor_sync(0xffffffffu, v);
        asm volatile("" ::"r"(v));  // keep the dependency on every lane's loads
        if (lane == 0) st_release_u8(rdone + x, 1u);
      }
      // ---- place it, swapping while dest has unprocessed blocks; the two
      //      register buffers alternate roles (no copies between them)
      bool in1 = false;
      for (;;) {
        const int st = in1 ? place(buf1, buf0, dest) : place(buf0, buf1, dest);
        if (st == 0) break;
        if (st == 1) in1 = !in1;
      }
    }
    if (lane == 0) atomicExch(&A.task_done[ti], 1u);
  }
  PCLK_FLUSH()
}

}  // namespace ips4o
