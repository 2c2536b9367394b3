// k_plan.cuh -- a7: the recursion scheduler runs on the device (Alg. 2,
// P:1119-1163; task groups P:969-990).  The host enqueues ONE kernel per sort
// (entry_kernel) and returns; every further launch is made from the device
// with CUDA dynamic parallelism (tail launches, which run in launch order
// after the launching grid completes): the entry kernel decides the easy
// inputs, the planner lays out each level ("round") in a fixed
// scratch arena, launches the level's kernels K1..K7 with exact grid sizes
// and, last, itself for the next round.  The caller's stream sees one
// stream-ordered piece of work (capturable into a CUDA graph); no host
// synchronisation, no host round trip per level (DESIGN "Device planner").
//
// Bounded scratch: a round takes the longest prefix of the pending task list
// whose level plan fits the arena (capacity fixed by the host from the root
// level); the rest is deferred to the next round, before the new children.
#pragma once
#include "common.cuh"
#include "k_basecase.cuh"
#include "k_classify.cuh"
#include "k_cleanup.cuh"
#include "k_count.cuh"
#include "k_misc.cuh"
#include "k_permute.cuh"
#include "k_sample.cuh"

namespace ips4o {

constexpr int MAX_ROUNDS = 64;      // rounds recorded in the statistics / timing slots
constexpr int PLAN_THREADS = 1024;  // the planner is one CTA
constexpr int MAX_PRE_PARTS = 4096;
constexpr int PRE_PARTS_PER_SM = 4;

__host__ __device__ __forceinline__ u64 cdiv(u64 a, u64 b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ u64 rup(u64 a, u64 b) { return cdiv(a, b) * b; }
__host__ __device__ __forceinline__ u64 npow2(u64 x) {
  u64 p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Configuration of one sort (host -> entry kernel, by value).
struct SortCfg {
  char *base;          // the caller's array
  u64 n;
  u64 seed;
  u64 base_cap;        // base-case capacity M in use
  u64 base_split;      // buckets up to this size go to the base case (2M when it can split)
  int algo, k_max, alpha_min, max_levels;
  int skip_prepass, skip_basecase, timing, capture, dbg_one_agent;
  int host_levels;     // profiling mode (IPS4O_HOST_LEVELS=1): the host launches every round
  int sms;             // SMs of the device
  int spm;             // classification stripes per SM
  u32 g_perm;          // permutation CTAs per level (SMs x occupancy)
  char *scratch;       // the call's scratch: SortCtl, then the two task lists, then the arena
  u64 list_cap;        // tasks per pending list
  u64 arena_off, arena_cap;
  u32 *status;         // persistent per-device status word (ips4o_device_status)
  const char *ext_spl; // ips4o_partition_splitters: given splitters (device, ext_n elements)
  int ext_n;
};

// Device-side state of one sort (at the start of the scratch).
struct SortCtl {
  SortCfg cfg;
  TaskDesc *list[2];   // pending task lists (ping-pong by round)
  u32 count[2];
  u32 cur;             // list of the round being planned
  u32 round;
  u32 error;           // ERR_* flags
  u32 easy;            // 0 none, 1 sorted, 2 reverse-sorted, 3 all equal
  u32 levels;
  u32 go;              // round 0 (launched by the host) runs: the input is not an easy input
  u32 need_prepass;    // the entry kernel could not prove a non-easy input: the full pre-pass runs
  u32 pad0;
  u64 launches;        // kernels launched by this sort (host + device)
  u64 arena_peak;      // largest level plan placed in the arena
  u64 base_tasks;      // base-case sorts (folded per round)
  u64 deferred;        // tasks deferred to a later round (arena full)
  u32 counters[16];    // [1] base count, [8] split count (per round); [2..3] equal elems, [6..7] base elems
  PrepassOut pre;
  u64 tasks_per_round[MAX_ROUNDS], elems_per_round[MAX_ROUNDS];
  LevelArgs A;         // the last planned round (read back by the partition-step test hook)
  unsigned long long tslot[MAX_ROUNDS][KS_COUNT][2];
  PrepassPart parts[MAX_PRE_PARTS];
};

// ------------------------------------------------------------------ plan arithmetic (host + device)
// The host sizes the arena with the same functions the device planner uses.
template <int DT> __host__ __device__ u64 level_stripe_elems(const SortCfg &c, u64 N) {
  using Tr = Traits<DT>;
  const u64 target = (u64)c.sms * (u64)c.spm;
  u64 se = rup(cdiv(N, target), (u64)Tr::B);
  const u64 mn = rup((u64)Tr::CLS_TILE * 2, (u64)Tr::B);
  return se > mn ? se : mn;
}

struct TaskShape {
  u32 kr, kidx, m, ns, np, mparts, lut_bits, lut_slots;
  u64 se_t, nblk;
};

template <int DT> __host__ __device__ TaskShape task_shape(const SortCfg &c, u64 size, u32 flags, u64 se, u64 N) {
  using Tr = Traits<DT>;
  constexpr int KI = Tr::KIDX, B = Tr::B;
  TaskShape s;
  const u64 M = c.base_cap;
  // bucket count: expected child <= M/2 (DESIGN "Adaptive k"), P:983-990 analogue
  u64 kr = npow2(cdiv(2 * size, M > 0 ? M : 1));
  kr = kr < 2 ? 2 : kr;
  kr = kr > (u64)c.k_max ? (u64)c.k_max : kr;
  if (c.ext_n > 0) kr = (u64)c.k_max;  // given splitters: every bucket index available
  s.kr = (u32)kr;
  const u64 kx = c.algo == ALGO_TREE ? 2 * kr : kr;
  s.kidx = (u32)(kx < (u64)KI ? kx : (u64)KI);
  // oversampling alpha = max(ceil(0.2 log2 n'), alpha_min) (DESIGN R7)
  u64 alpha = (u64)ceil(0.2 * log2((double)(size > 2 ? size : 2)));
  alpha = alpha > (u64)c.alpha_min ? alpha : (u64)c.alpha_min;
  const u64 smax = (u64)sample_max<DT>();
  if (alpha * kr > smax) alpha = smax / kr > 1 ? smax / kr : 1;
  s.m = (u32)(alpha * kr);
  // stripes: task-relative, multiples of b
  u64 ns = cdiv(size, se);
  ns = ns < 1 ? 1 : ns;
  const u64 se_t = rup(cdiv(size, ns), (u64)B);
  s.se_t = se_t;
  s.ns = (u32)cdiv(size, se_t);
  // permutation agents in proportion to the task size (P:974-977 analogue)
  u64 np = (2 * size * (u64)c.g_perm + N) / (2 * (N > 0 ? N : 1));
  const u64 npmax = cdiv(size / B, (u64)PERM_WARPS * 2);
  np = np < npmax ? np : npmax;
  np = np < 1 ? 1 : np;
  if (c.dbg_one_agent) np = 1;
  s.np = (u32)np;
  s.nblk = cdiv(size, (u64)B) + 1;
  u64 mp = 0;
  if (flags & TF_MEASURE) {
    mp = cdiv(size, MEAS_PART_ELEMS);
    mp = mp < 1 ? 1 : mp;
    mp = mp > MEAS_MAXPARTS ? MEAS_MAXPARTS : mp;
  }
  s.mparts = (u32)mp;
  // lookup table of starting leaves (TREE, 4/8/16-byte keys): ~64 slots per
  // bucket index, at most LUT_SLOTS
  u32 lb = 6;
  while ((1u << (lb - 6)) < s.kidx) ++lb;
  s.lut_bits = lb < (u32)LUT_BITS ? lb : (u32)LUT_BITS;
  s.lut_slots = (Tr::D <= 16 && c.algo == ALGO_TREE) ? (1u << s.lut_bits) : 0u;
  return s;
}

struct PlanTotals {
  u64 T, S, NP, nbk, nsbk, nblk, child, mparts, mtasks, luts;
  u64 max_m, bc_grid, bc_cap;
};

__host__ __device__ __forceinline__ void add_shape(PlanTotals &P, const TaskShape &s) {
  P.T += 1;
  P.S += s.ns;
  P.NP += s.np;
  P.nbk += s.kidx + 1;
  P.nsbk += (u64)s.ns * s.kidx;
  P.nblk += s.nblk;
  P.child += s.kidx;
  P.mparts += s.mparts;
  P.mtasks += s.mparts ? 1 : 0;
  P.luts += s.lut_slots;
  P.max_m = P.max_m > s.m ? P.max_m : s.m;
}

// Level arena layout: offsets from the arena start (base = 0 to size it).
template <int DT> __host__ __device__ u64 layout(LevelArgs &A, char *base, const PlanTotals &P) {
  using Tr = Traits<DT>;
  constexpr int KI = Tr::KIDX, B = Tr::B, D = Tr::D;
  using Key = typename Tr::Key;
  u64 used = 0;
  auto take = [&](u64 bytes) -> char * {
    const u64 off = rup(used, 256);
    used = off + bytes;
    return base + off;
  };
  A.tasks = reinterpret_cast<LevelTask *>(take(P.T * sizeof(LevelTask)));
  A.stripe_task = reinterpret_cast<const u32 *>(take(P.S * 4));
  A.perm_task = reinterpret_cast<const u32 *>(take(P.NP * 4));
  A.trees = take(P.T * 2 * KI * sizeof(Key));
  A.luts = reinterpret_cast<unsigned short *>(take(P.luts * 2));
  A.counts = reinterpret_cast<u32 *>(take(P.nsbk * 4));
  A.pfill = reinterpret_cast<u32 *>(take(P.nsbk * 4));
  A.pcum = reinterpret_cast<u32 *>(take(P.nsbk * 4));
  A.ptot = reinterpret_cast<u32 *>(take(P.nbk * 4));
  A.fullblocks = reinterpret_cast<u32 *>(take(P.S * 4));
  A.fcum = reinterpret_cast<u32 *>(take(P.S * 4));
  A.partials = take(P.nsbk * (u64)B * D);
  A.E = reinterpret_cast<u64 *>(take(P.nbk * 8));
  A.fblk = reinterpret_cast<u32 *>(take(P.nbk * 4));
  A.wr = reinterpret_cast<u64 *>(take(P.nbk * WR_STRIDE * 8));
  A.overlap = take(P.nbk * (u64)B * D);
  A.overflow = take(P.T * (u64)B * D);
  A.ovf_used = reinterpret_cast<u32 *>(take(P.T * 4));
  A.rdone = reinterpret_cast<unsigned char *>(take(P.nblk));
  A.bid = reinterpret_cast<unsigned short *>(take(P.nblk * 2));
  A.task_done = reinterpret_cast<u32 *>(take(P.T * 4));
  A.measure_part = reinterpret_cast<const u32 *>(take(P.mparts * 8));
  A.measure_task = reinterpret_cast<const u32 *>(take(P.mtasks * 12));
  A.measure_out = take(P.mparts * sizeof(PrepassPart));
  A.bc_scratch = BaseItem<DT>::SPLIT ? take(P.bc_grid * P.bc_cap * sizeof(typename BaseItem<DT>::Item)) : nullptr;
  A.base_tasks = reinterpret_cast<TaskDesc *>(take(P.child * sizeof(TaskDesc)));
  A.split_tasks = BaseItem<DT>::SPLIT ? reinterpret_cast<TaskDesc *>(take(P.child * sizeof(TaskDesc))) : nullptr;
  if (BaseItem<DT>::KEY_ONLY) {  // count-first tasks (k_count.cuh): at most one per child
    A.count_cap = (u32)P.child;
    A.count_tasks = reinterpret_cast<TaskDesc *>(take(P.child * sizeof(TaskDesc)));
    A.count_off = reinterpret_cast<u32 *>(take(P.child * 4));
    A.count_pre = reinterpret_cast<u32 *>(take((P.child + 1) * 4));
    A.count_work = reinterpret_cast<u32 *>(take(2 * 4));
    A.count_hist = reinterpret_cast<u32 *>(take((u64)CNT_POOL * 4));
  }
  return rup(used, 256);
}

template <int DT> __host__ __device__ u64 plan_bytes(PlanTotals P, const SortCfg &c) {
  LevelArgs A;
  P.bc_grid = P.child < (u64)c.sms ? (P.child > 0 ? P.child : 1) : (u64)c.sms;
  P.bc_cap = c.base_cap;
  return layout<DT>(A, nullptr, P);
}

// The arguments of round r's kernels (host and device build the same ones:
// round 0 is launched by the host, later rounds by the device planner).
template <int DT, int ALGO>
__host__ __device__ LevelArgs level_args(SortCtl *ctl, const SortCfg &c, const PlanTotals &tot, u32 r, u32 cur,
                                         u64 *used_out) {
  LevelArgs A;
  memset(&A, 0, sizeof A);
  PlanTotals Pt = tot;
  Pt.bc_grid = tot.child < (u64)c.sms ? (tot.child > 0 ? tot.child : 1) : (u64)c.sms;
  Pt.bc_cap = c.base_cap;
  const u64 used = layout<DT>(A, c.scratch + c.arena_off, Pt);
  if (used_out) *used_out = used;
  TaskDesc *lists = reinterpret_cast<TaskDesc *>(c.scratch + rup(sizeof(SortCtl), 256));
  A.base = c.base;
  A.ntasks = (u32)tot.T;
  A.nstripes = (u32)tot.S;
  A.nperm = (u32)tot.NP;
  A.algo = ALGO;
  A.seed = c.seed;
  A.base_cap_elems = c.base_cap;
  A.base_split_elems = c.base_split;
  A.dbg_one_agent = c.dbg_one_agent ? 1 : 0;
  A.sample_p = (u32)npow2(tot.max_m > (u64)SORT_THREADS ? tot.max_m : (u64)SORT_THREADS);
  A.counters = ctl->counters;
  A.err = &ctl->error;
  A.tslot = c.timing ? &ctl->tslot[r < MAX_ROUNDS ? r : MAX_ROUNDS - 1][0][0] : nullptr;
  A.next_tasks = lists + (cur ^ 1) * c.list_cap;
  A.next_count = &ctl->count[cur ^ 1];
  A.next_cap = (u32)c.list_cap;
  A.base_cap_tasks = (u32)tot.child;
  A.capture = c.capture ? 1 : 0;
  A.bc_grid = (u32)Pt.bc_grid;
  A.ctl = ctl;
  A.go = r == 0 ? &ctl->go : nullptr;
  A.nmparts = (u32)tot.mparts;
  A.nmtasks = (u32)tot.mtasks;
  A.count_grid = (u32)c.sms * 4;
  if (c.capture || c.skip_basecase) A.count_cap = 0;  // (no count-first finish: K6 keeps such tasks)
  A.ext_spl = r == 0 ? c.ext_spl : nullptr;
  A.ext_n = r == 0 ? (u32)c.ext_n : 0u;
  u32 stg = 0;
  if (ALGO == ALGO_DIGIT && tot.mtasks > 0) stg |= (1u << ST_MEAS) | (1u << ST_MEASRED);
  for (int x = ST_SAMPLE; x <= ST_CFILL; ++x) stg |= 1u << x;
  if (!c.capture && !c.skip_basecase) {
    if (BaseItem<DT>::KEY_ONLY) stg |= (1u << ST_CSETUP) | (1u << ST_CCOUNT) | (1u << ST_CWRITE);
    stg |= 1u << ST_BASE;
    if (BaseItem<DT>::SPLIT) stg |= 1u << ST_SPLIT;
  }
  if (!c.capture && !c.host_levels) stg |= 1u << ST_NEXT;
  A.stages = stg;
  return A;
}

template <int DT> __host__ __device__ PlanTotals root_totals(const SortCfg &c) {
  PlanTotals P{};
  add_shape(P, task_shape<DT>(c, c.n, 0, level_stripe_elems<DT>(c, c.n), c.n));
  return P;
}

// Host: arena capacity = the larger of the root level's plan and the plan of
// a second level of k' equal tasks (its more numerous stripes, trees and
// overlap blocks); skewed levels beyond it are split into rounds.
// (min_bytes > 0: the caller's arena size, at least the root level's plan)
template <int DT> u64 host_arena_bytes(const SortCfg &c, u64 min_bytes = 0) {
  PlanTotals P1{};
  const u64 n = c.n;
  const u64 se1 = level_stripe_elems<DT>(c, n);
  const TaskShape r = task_shape<DT>(c, n, 0, se1, n);
  add_shape(P1, r);
  u64 b = plan_bytes<DT>(P1, c);
  if (min_bytes) return rup(b > min_bytes ? b : min_bytes, 4096);
  const u64 k1 = r.kr, child = n / (k1 ? k1 : 1);
  if (child > c.base_split) {
    PlanTotals P2{};
    const u64 N2 = child * k1;
    const u64 se2 = level_stripe_elems<DT>(c, N2);
    const TaskShape s = task_shape<DT>(c, child, 0, se2, N2);
    for (u64 i = 0; i < k1; ++i) add_shape(P2, s);
    const u64 b2 = plan_bytes<DT>(P2, c);
    b = b > b2 ? b : b2;
  }
  return rup(b + b / 32 + (1 << 20), 4096);
}

// ------------------------------------------------------------------ device planner
__device__ __forceinline__ u64 block_sum_u64(u64 v, u64 *ws) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  u64 t = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
  return t;
}
__device__ __forceinline__ u64 block_max_u64(u64 v, u64 *ws) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 y = __shfl_xor_sync(0xffffffffu, v, o);
    v = y > v ? y : v;
  }
  __syncthreads();
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  u64 t = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = ws[w] > t ? ws[w] : t;
  return t;
}

// Totals of the plan of the first q pending tasks (all threads).
template <int DT>
__device__ PlanTotals round_totals(const SortCfg &c, const TaskDesc *P, u32 q, u64 &N, u64 &se, u64 *ws) {
  u64 nloc = 0;
  for (u32 i = threadIdx.x; i < q; i += blockDim.x) nloc += P[i].size;
  N = block_sum_u64(nloc, ws);
  se = level_stripe_elems<DT>(c, N);
  PlanTotals L{};
  for (u32 i = threadIdx.x; i < q; i += blockDim.x) add_shape(L, task_shape<DT>(c, P[i].size, P[i].flags, se, N));
  PlanTotals T{};
  T.T = block_sum_u64(L.T, ws);
  T.S = block_sum_u64(L.S, ws);
  T.NP = block_sum_u64(L.NP, ws);
  T.nbk = block_sum_u64(L.nbk, ws);
  T.nsbk = block_sum_u64(L.nsbk, ws);
  T.nblk = block_sum_u64(L.nblk, ws);
  T.child = block_sum_u64(L.child, ws);
  T.mparts = block_sum_u64(L.mparts, ws);
  T.mtasks = block_sum_u64(L.mtasks, ws);
  T.luts = block_sum_u64(L.luts, ws);
  T.max_m = block_max_u64(L.max_m, ws);
  return T;
}

template <int DT, int ALGO> __global__ void driver_kernel(SortCtl *ctl, int phase);

// ------------------------------------------------------------------ stage launches
// A device-side launch call costs ~10 us of the launching thread (measured:
// tools/exp/cdp2_cost.cu).  The planner launches the round's first stage
// fire-and-forget, so that it starts at once, and then enqueues the other
// stages as tail launches while it runs: tail launches start after the
// planner grid AND its fire-and-forget children complete, in launch order
// (tools/exp/cdp2_ff.cu), so the launch calls overlap the first stage.
template <int DT, int ALGO>
__device__ void launch_stage(const LevelArgs &A, int st, cudaStream_t tl) {
  using Tr = Traits<DT>;
  SortCtl *ctl = reinterpret_cast<SortCtl *>(A.ctl);
  switch (st) {
    case ST_MEAS: measure_part_kernel<DT><<<A.nmparts, MEAS_THREADS, 0, tl>>>(A); break;
    case ST_MEASRED: measure_reduce_kernel<DT><<<(A.nmtasks + 127) / 128, 128, 0, tl>>>(A, A.nmtasks); break;
    case ST_SAMPLE:
      sample_kernel<DT, ALGO><<<A.ntasks, SAMPLE_THREADS,
                                ALGO == ALGO_TREE ? sample_smem<DT>((size_t)A.sample_p) : 0, tl>>>(A);
      break;
    case ST_CLASSIFY:
      if constexpr (Tr::D > 16) classify_kernel<DT, ALGO><<<A.nstripes, Tr::CLS_THREADS, ClsSmem<DT>::bytes, tl>>>(A);
      else classify_v2_kernel<DT, ALGO><<<A.nstripes, ClsV2<DT>::NT, ClsV2<DT>::bytes, tl>>>(A);
      break;
    case ST_BOUND: boundaries_kernel<DT, ALGO><<<A.ntasks, BND_THREADS, 0, tl>>>(A); break;
    case ST_FIX: stripe_fix_kernel<DT><<<A.nstripes, FIX_THREADS, 0, tl>>>(A); break;
    case ST_PERM: permute_kernel<DT, ALGO><<<A.nperm, PERM_THREADS, 0, tl>>>(A); break;
    case ST_CSAVE: cleanup_save_kernel<DT><<<A.ntasks * cleanup_groups<DT>(), CLN_WARPS * 32, 0, tl>>>(A); break;
    case ST_CFILL: cleanup_fill_kernel<DT><<<A.nstripes, FILL_THREADS, 0, tl>>>(A); break;
    case ST_BASE:
    case ST_SPLIT: {
      const BaseSplitArgs sp{A.bc_scratch, (u32)A.base_cap_elems, A.next_tasks, A.next_count, A.next_cap,
                             reinterpret_cast<unsigned long long *>(ctl->counters + 6), &ctl->error};
      if (st == ST_BASE)
        basecase_kernel<DT, false><<<A.bc_grid, BaseItem<DT>::THREADS, BaseSmem<DT>::bytes, tl>>>(
            A.base, A.base_tasks, ctl->counters + 1, A.base_cap_tasks, sp, A.tslot);
      else if constexpr (BaseItem<DT>::SPLIT)
        basecase_kernel<DT, true><<<A.bc_grid, BaseItem<DT>::THREADS, BaseSmem<DT>::bytes, tl>>>(
            A.base, A.split_tasks, ctl->counters + 8, A.base_cap_tasks, sp, A.tslot);
      break;
    }
    case ST_CSETUP: count_setup_kernel<<<1, CNT_SETUP_THREADS, 0, tl>>>(A); break;
    case ST_CCOUNT:
      if constexpr (BaseItem<DT>::KEY_ONLY) count_kernel<DT><<<A.count_grid, CNT_THREADS, 0, tl>>>(A);
      break;
    case ST_CWRITE:
      if constexpr (BaseItem<DT>::KEY_ONLY) count_write_kernel<DT><<<A.count_grid, CNT_THREADS, 0, tl>>>(A);
      break;
    case ST_NEXT: driver_kernel<DT, ALGO><<<1, PLAN_THREADS, 0, tl>>>(ctl, 2); break;
  }
}

#ifdef IPS4O_PLAN_CLOCKS
#define PLAN_CLK(i) \
  if (threadIdx.x == 0) pclk[i] = clock64();
#define PLAN_CLK_DECL long long pclk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define PLAN_CLK_PRINT(r)                                                                                     \
  if (threadIdx.x == 0) printf("plan round %u: totals %lld layout %lld tasks %lld maps %lld tail %lld launch %lld cycles\n", r,      \
         pclk[1] - pclk[0], pclk[2] - pclk[1], pclk[3] - pclk[2], pclk[4] - pclk[3], pclk[5] - pclk[4], pclk[6] - pclk[5]);
#else
#define PLAN_CLK(i)
#define PLAN_CLK_DECL
#define PLAN_CLK_PRINT(r)
#endif

#define IPS4O_DLAUNCH_CHECK(ctl)                                   \
  do {                                                             \
    if (cudaGetLastError() != cudaSuccess) atomicOr(&(ctl)->error, (u32)ERR_LAUNCH); \
  } while (0)

// Plan and launch one round (all PLAN_THREADS threads of the calling CTA).
// Round 0 is launched by the host (launch = false: plan only, then go = 1).
template <int DT, int ALGO>
__device__ void plan_round(SortCtl *ctl, bool launch) {
  using Tr = Traits<DT>;
  constexpr int KI = Tr::KIDX;
  __shared__ u64 ws[PLAN_THREADS / 32];
  __shared__ u32 s_ws[PLAN_THREADS / 32 + 1];
  __shared__ int s_stop;
  __shared__ LevelArgs s_A;
  const SortCfg &c = ctl->cfg;
  const int tid = threadIdx.x;
  const u32 cur = ctl->cur, r = ctl->round;
  if (tid == 0) {
    s_stop = 0;
    if (r > 0) {  // fold the previous round's base-case counts
      const u32 cap = ctl->A.base_cap_tasks;
      const u32 b1 = ctl->counters[1], b8 = ctl->counters[8];
      ctl->base_tasks += (b1 < cap ? b1 : cap) + (b8 < cap ? b8 : cap);
    }
    if (ctl->count[cur] == 0 || (c.max_levels > 0 && r >= (u32)c.max_levels) || ctl->error)
      s_stop = 1;
  }
  __syncthreads();
  if (s_stop) {
    if (tid == 0 && ctl->error) atomicOr(c.status, ctl->error);
    return;
  }
  PLAN_CLK_DECL
  PLAN_CLK(0)
  const u32 p = ctl->count[cur];
  TaskDesc *P = ctl->list[cur];
  TaskDesc *Q = ctl->list[cur ^ 1];
  // ---- the longest prefix of the pending list whose plan fits the arena
  u64 N = 0, se = 0;
  PlanTotals tot = round_totals<DT>(c, P, p, N, se, ws);
  u32 q = p;
  if (plan_bytes<DT>(tot, c) > c.arena_cap) {
    u32 lo = 0, hi = p;  // largest q in [lo, hi) that fits; q = lo fits (0 trivially)
    while (hi - lo > 1) {
      const u32 mid = lo + (hi - lo) / 2;
      PlanTotals t2 = round_totals<DT>(c, P, mid, N, se, ws);
      if (plan_bytes<DT>(t2, c) <= c.arena_cap) lo = mid;
      else hi = mid;
    }
    q = lo;
    if (q == 0) {
      if (tid == 0) {
        atomicOr(&ctl->error, (u32)ERR_ARENA);
        atomicOr(c.status, (u32)ERR_ARENA);
      }
      return;
    }
    tot = round_totals<DT>(c, P, q, N, se, ws);
  }
  PLAN_CLK(1)
  // ---- layout
  if (tid == 0) {
    u64 used = 0;
    s_A = level_args<DT, ALGO>(ctl, c, tot, r, cur, &used);
    if (used > ctl->arena_peak) ctl->arena_peak = used;
  }
  __syncthreads();
  const LevelArgs &A = s_A;
  PLAN_CLK(2)
  // ---- per-task records: a contiguous chunk of tasks per thread, offsets by scans
  const u32 per = (q + PLAN_THREADS - 1) / PLAN_THREADS;
  const u32 i0 = tid * per < q ? tid * per : q, i1 = i0 + per < q ? i0 + per : q;
  u32 ls = 0, lp = 0, lbk = 0, lsbk = 0, lmp = 0, lmt = 0, llut = 0;
  u64 lblk = 0;
  for (u32 i = i0; i < i1; ++i) {
    const TaskShape s = task_shape<DT>(c, P[i].size, P[i].flags, se, N);
    ls += s.ns;
    lp += s.np;
    lbk += s.kidx + 1;
    lsbk += s.ns * s.kidx;
    lblk += s.nblk;
    lmp += s.mparts;
    lmt += s.mparts ? 1 : 0;
    llut += s.lut_slots;
  }
  u32 tt;
  u32 os = block_exclusive_scan<PLAN_THREADS>(ls, s_ws, &tt);
  u32 op = block_exclusive_scan<PLAN_THREADS>(lp, s_ws, &tt);
  u32 obk = block_exclusive_scan<PLAN_THREADS>(lbk, s_ws, &tt);
  u32 osbk = block_exclusive_scan<PLAN_THREADS>(lsbk, s_ws, &tt);
  u32 omp = block_exclusive_scan<PLAN_THREADS>(lmp, s_ws, &tt);
  u32 omt = block_exclusive_scan<PLAN_THREADS>(lmt, s_ws, &tt);
  // nblk can exceed 2^32 / PLAN_THREADS per thread only for n >= 2^32 (rejected)
  u64 oblk = block_exclusive_scan<PLAN_THREADS>((u32)lblk, s_ws, &tt);
  u64 olut = block_exclusive_scan<PLAN_THREADS>(llut, s_ws, &tt);
  u32 *stripe_task = const_cast<u32 *>(A.stripe_task);
  u32 *perm_task = const_cast<u32 *>(A.perm_task);
  u32 *mpart = const_cast<u32 *>(A.measure_part);
  u32 *mtask = const_cast<u32 *>(A.measure_task);
  for (u32 i = i0; i < i1; ++i) {
    const TaskShape s = task_shape<DT>(c, P[i].size, P[i].flags, se, N);
    LevelTask L;
    memset(&L, 0, sizeof L);
    L.t = P[i];
    L.k_req = s.kr;
    L.kidx = s.kidx;
    L.m = s.m;
    L.stripe_first = os;
    L.nstripes = s.ns;
    L.perm_first = op;
    L.nperm = s.np;
    L.stripe_elems = s.se_t;
    L.bucket_off = obk;
    L.blk_off = oblk;
    L.sbk_off = osbk;
    L.lut_bits = s.lut_bits;
    L.lut_off = olut;
    A.tasks[i] = L;
    if (s.mparts) {
      mtask[3 * omt] = i;
      mtask[3 * omt + 1] = omp;
      mtask[3 * omt + 2] = s.mparts;
      for (u32 x = 0; x < s.mparts; ++x) {
        mpart[2 * (omp + x)] = i;
        mpart[2 * (omp + x) + 1] = x | (s.mparts << 16);
      }
      ++omt;
      omp += s.mparts;
    }
    os += s.ns;
    op += s.np;
    obk += s.kidx + 1;
    osbk += s.ns * s.kidx;
    oblk += s.nblk;
    olut += s.lut_slots;
    A.task_done[i] = 0;
  }
  __syncthreads();
  PLAN_CLK(3)
  // ---- stripe -> task and permutation CTA -> task maps, all threads: the
  //      task of entry x is the last one whose first entry is <= x
  auto owner = [&](u32 x, bool perm) -> u32 {
    u32 lo = 0, hi = q;
    while (hi - lo > 1) {
      const u32 mid = (lo + hi) >> 1;
      const u32 f = perm ? A.tasks[mid].perm_first : A.tasks[mid].stripe_first;
      if (f <= x) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  for (u32 x = tid; x < (u32)tot.S; x += PLAN_THREADS) stripe_task[x] = owner(x, false);
  for (u32 x = tid; x < (u32)tot.NP; x += PLAN_THREADS) perm_task[x] = owner(x, true);
  PLAN_CLK(4)
  // ---- deferred tasks go first into the next round's list
  for (u32 i = q + tid; i < p; i += PLAN_THREADS) Q[i - q] = P[i];
  if (tid == 0) {
    ctl->count[cur ^ 1] = p - q;
    ctl->count[cur] = 0;
    ctl->deferred += p - q;
    ctl->counters[1] = 0;
    ctl->counters[8] = 0;
    ctl->counters[9] = 0;
    ctl->counters[10] = 0;
    if (r < MAX_ROUNDS) {
      ctl->tasks_per_round[r] = q;
      ctl->elems_per_round[r] = N;
    }
    ctl->levels = r + 1;
    ctl->cur = cur ^ 1;
    ctl->round = r + 1;
    ctl->A = A;
  }
  __syncthreads();
  __threadfence();
  PLAN_CLK(5)
  // ---- launch the first stage; each stage launches the next (launch_after)
  if (!launch) {
    if (tid == 0) ctl->go = 1;
  } else if (tid == 0) {
    u64 nl = 0;
    for (int st = 0; st < ST_N; ++st)
      if ((A.stages >> st) & 1u) {
        launch_stage<DT, ALGO>(A, st, nl == 0 ? cudaStreamFireAndForget : cudaStreamTailLaunch);
        ++nl;
      }
    IPS4O_DLAUNCH_CHECK(ctl);
    atomicAdd(reinterpret_cast<unsigned long long *>(&ctl->launches), (unsigned long long)nl);
  }
  PLAN_CLK(6)
  PLAN_CLK_PRINT(r)
  (void)KI;
}

// Root of the recursion once the key range is known (all threads): round 0
// (the whole array as its only task) is planned here and launched by the
// host; n <= M is a single base case, also launched by the host.
template <int DT, int ALGO>
__device__ void start_rounds(SortCtl *ctl, TaskDesc root) {
  const SortCfg &c = ctl->cfg;
  if (!c.capture && c.n <= c.base_cap) {
    if (threadIdx.x == 0 && !c.skip_basecase) {
      TaskDesc *t = reinterpret_cast<TaskDesc *>(c.scratch + c.arena_off);
      *t = root;
      ctl->counters[1] = 1;  // the host-launched base case reads this count
      ctl->base_tasks = 1;
      *reinterpret_cast<unsigned long long *>(ctl->counters + 6) = c.n;
    }
    return;
  }
  if (threadIdx.x == 0) {
    ctl->list[0][0] = root;
    ctl->count[0] = 1;
    ctl->cur = 0;
    ctl->round = 0;
  }
  __syncthreads();
  plan_round<DT, ALGO>(ctl, false);
}

// phase 1: after the full pre-pass; phase 2: the next round.
template <int DT, int ALGO>
__global__ void __launch_bounds__(PLAN_THREADS) driver_kernel(SortCtl *ctl, int phase) {
  using Key = typename Traits<DT>::Key;
  const SortCfg &c = ctl->cfg;
  const u32 r = ctl->round;
  unsigned long long *const kts = c.timing ? &ctl->tslot[phase == 1 ? 0 : (r < MAX_ROUNDS ? r : MAX_ROUNDS - 1)][0][0] : nullptr;
  KTIMER(kts, KS_PLAN);
  if (phase >= 2) {  // 3: plan only (profiling mode: the host launches the round)
    plan_round<DT, ALGO>(ctl, phase == 2);
    return;
  }
  if (!ctl->need_prepass) return;  // (host-launched after the pre-pass kernels)
  const PrepassOut &po = ctl->pre;
  const Key mn = key_from_words<Key>(po.minkey), mx = key_from_words<Key>(po.maxkey);
  if (!c.capture && !c.skip_prepass) {
    if (po.nondecreasing) {  // P:1654 sorted input: nothing to do
      if (threadIdx.x == 0) ctl->easy = (mn == mx) ? 3 : 1;
      return;
    }
    if (po.nonincreasing) {  // P:1655 decreasing: reverse and return
      if (threadIdx.x == 0) {
        ctl->easy = 2;
        reverse_kernel<DT><<<c.sms * 8, 256, 0, cudaStreamTailLaunch>>>(c.base, c.n,
                                                                          c.timing ? &ctl->tslot[0][0][0] : nullptr);
        IPS4O_DLAUNCH_CHECK(ctl);
        atomicAdd(reinterpret_cast<unsigned long long *>(&ctl->launches), 1ull);
      }
      return;
    }
  }
  if (!(mn < mx) && !c.capture) {
    if (threadIdx.x == 0) ctl->easy = 3;
    return;  // all keys equal
  }
  TaskDesc root;
  memset(&root, 0, sizeof root);
  root.size = c.n;
  key_to_words<Key>(mn, root.lo);
  key_to_words<Key>(mx, root.hi);
  start_rounds<DT, ALGO>(ctl, root);
}

// The one kernel the host launches per sort.
template <int DT, int ALGO>
__global__ void __launch_bounds__(PLAN_THREADS) entry_kernel(SortCfg cfg) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  SortCtl *ctl = reinterpret_cast<SortCtl *>(cfg.scratch);
  const int tid = threadIdx.x;
  // ---- initialise the control block
  {
    unsigned long long *ts = &ctl->tslot[0][0][0];
    for (int i = tid; i < MAX_ROUNDS * KS_COUNT; i += PLAN_THREADS) {
      ts[2 * i] = ~0ull;
      ts[2 * i + 1] = 0;
    }
    for (int i = tid; i < MAX_ROUNDS; i += PLAN_THREADS) ctl->tasks_per_round[i] = ctl->elems_per_round[i] = 0;
    if (tid < 16) ctl->counters[tid] = 0;
    if (tid == 0) {
      ctl->cfg = cfg;
      TaskDesc *lists = reinterpret_cast<TaskDesc *>(cfg.scratch + rup(sizeof(SortCtl), 256));
      ctl->list[0] = lists;
      ctl->list[1] = lists + cfg.list_cap;
      ctl->count[0] = ctl->count[1] = 0;
      ctl->cur = ctl->round = 0;
      ctl->error = 0;
      ctl->easy = 0;
      ctl->levels = 0;
      ctl->launches = 0;
      ctl->go = 0;
      ctl->need_prepass = 0;
      ctl->arena_peak = 0;
      ctl->base_tasks = 0;
      ctl->deferred = 0;
      memset(&ctl->A, 0, sizeof(LevelArgs));
    }
  }
  __syncthreads();
  __threadfence_block();
  unsigned long long *const kts = cfg.timing ? &ctl->tslot[0][0][0] : nullptr;
  KTIMER(kts, KS_PRESAMPLE);
  const SortCfg &c = cfg;
  bool need_prepass = !c.skip_prepass || c.algo == ALGO_DIGIT || c.capture;
  u32 flags = 0;
#ifdef IPS4O_PLAN_CLOCKS
  long long e0 = clock64();
#endif
  if (need_prepass && !c.capture && !c.skip_prepass && c.algo == ALGO_TREE && sizeof(Key) == 8 &&
      c.n > c.base_cap && c.n >= (1ull << 22)) {
    // cheap sample pre-check: an ascending and a descending sampled pair
    // prove the input is not an easy input; the root's bounds are then the
    // whole key space (TF_LOOSE: the base case measures edge buckets)
    const int f = presample_block<DT>(c.base, c.n);
    if (f == 3) {
      need_prepass = false;
      flags = TF_LOOSE;
    }
  }
#ifdef IPS4O_PLAN_CLOCKS
  if (tid == 0) printf("entry: presample %lld cycles\n", clock64() - e0);
#endif
  if (need_prepass) {
    // the host enqueued the pre-pass kernels and the driver (phase 1) behind us
    if (tid == 0) ctl->need_prepass = 1;
    return;
  }
  TaskDesc root;
  memset(&root, 0, sizeof root);
  root.size = c.n;
  root.flags = flags | TF_LOOSE;  // bounds [0, max] (no pre-pass)
  key_to_words<Key>((Key)0, root.lo);
  key_to_words<Key>(key_max<Key>(), root.hi);
  start_rounds<DT, ALGO>(ctl, root);
}

}  // namespace ips4o
