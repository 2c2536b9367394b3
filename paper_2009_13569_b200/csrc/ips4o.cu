// ips4o.cu -- host driver and C ABI (include/ips4o.h) of the B200-native
// in-place samplesort partitioning step.  Product code: no PyTorch types, no
// CPU fallback, nothing from oracle/.
//
// Host loop (DESIGN "Host loop"): per partitioning level the host plans the
// level from the task list (stripes, permutation agents, scratch layout),
// enqueues K1..K7 on the caller's stream, and reads back the next task list
// (one stream synchronisation per level).  All element work runs in the
// kernels of k_*.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ips4o.h"
#include "common.cuh"
#include "internal.h"
#include "k_basecase.cuh"
#include "k_classify.cuh"
#include "k_cleanup.cuh"
#include "k_misc.cuh"
#include "k_permute.cuh"
#include "k_sample.cuh"

namespace ips4o {

static thread_local std::string g_err = "no error";

static int set_cuda_err(cudaError_t e, const char *what, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %d (%s) at ips4o.cu:%d in %s", (int)e, cudaGetErrorString(e), line, what);
  g_err = buf;
  return IPS4O_ERR_CUDA;
}
#define CK(call)                                                   \
  do {                                                             \
    cudaError_t e_ = (call);                                       \
    if (e_ != cudaSuccess) return set_cuda_err(e_, #call, __LINE__); \
  } while (0)
#define CKLAUNCH()                                                          \
  do {                                                                      \
    cudaError_t e_ = cudaGetLastError();                                    \
    if (e_ != cudaSuccess) return set_cuda_err(e_, "kernel launch", __LINE__); \
    ++c.launches;                                                           \
  } while (0)

static inline u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }
static inline u64 round_up(u64 a, u64 b) { return ceil_div(a, b) * b; }
static inline u64 next_pow2_u64(u64 x) {
  u64 p = 1;
  while (p < x) p <<= 1;
  return p;
}

enum KFam { KF_PRE = 0, KF_SAMPLE, KF_CLASSIFY, KF_BOUND, KF_FIX, KF_PERM, KF_CLEAN, KF_SCHED, KF_BASE, KF_REV, KF_HOST, KF_TOTAL };

struct Ctx {
  cudaStream_t st = nullptr;
  int dev = 0;
  int sms = 148;
  int algo = ALGO_TREE;
  int k_max = 256;
  u64 seed = 0x1F4A2C7ull;
  int alpha_min = 64;
  u64 base_cap = 0;
  int max_levels = 0;
  bool skip_prepass = false, skip_basecase = false;
  bool timing = false;
  bool dbg_one_agent = false;  // IPS4O_DEBUG_ONE_AGENT=1: one permute CTA per task
  ips4o_stats *stats = nullptr;
  u64 launches = 0;
  u64 peak_scratch = 0;
  // timing
  std::vector<std::pair<int, cudaEvent_t>> evs;
  cudaEvent_t ev0 = nullptr;
  float ms[IPS4O_NUM_KERNELS] = {0};
  // pinned staging for host<->device control data (thread-local cache)
  char *pinned = nullptr;
};

static thread_local char *t_pinned = nullptr;
static thread_local size_t t_pinned_cap = 0;

static int mark(Ctx &c, int fam) {
  if (!c.timing) return 0;
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  CK(cudaEventRecord(e, c.st));
  c.evs.push_back({fam, e});
  return 0;
}
// accumulate recorded events (stream must be synchronised)
static void flush_marks(Ctx &c) {
  if (!c.timing) return;
  cudaEvent_t prev = c.ev0;
  for (auto &pe : c.evs) {
    float t = 0;
    if (prev && cudaEventElapsedTime(&t, prev, pe.second) == cudaSuccess) c.ms[pe.first] += t;
    if (prev != c.ev0) cudaEventDestroy(prev);
    prev = pe.second;
  }
  if (!c.evs.empty()) {
    // keep the last event as the new origin
    if (c.ev0) cudaEventDestroy(c.ev0);
    c.ev0 = c.evs.back().second;
  }
  c.evs.clear();
}

// The caller's stream is synchronised before the buffer is reused or grown.
static int ensure_pinned(Ctx &c, size_t bytes) {
  if (t_pinned_cap < bytes) {
    if (t_pinned) cudaFreeHost(t_pinned);
    t_pinned = nullptr;
    t_pinned_cap = 0;
    size_t cap = std::max<size_t>(next_pow2_u64(bytes), 1 << 20);
    if (cudaMallocHost(&t_pinned, cap) != cudaSuccess) {
      cudaGetLastError();
      g_err = "cudaMallocHost failed";
      return IPS4O_ERR_NOMEM;
    }
    t_pinned_cap = cap;
  }
  c.pinned = t_pinned;
  return 0;
}

// ------------------------------------------------------------------ arena
struct Arena {
  char *base = nullptr;
  size_t used = 0;
  template <class T> T *take(size_t count) {
    size_t off = round_up(used, 256);
    used = off + count * sizeof(T);
    return reinterpret_cast<T *>(base + off);
  }
};

struct LevelPlan {
  std::vector<LevelTask> lt;
  std::vector<u32> stripe_task, perm_task;
  std::vector<u32> measure_part, measure_task;  // K0m lists (TF_MEASURE tasks)
  u32 max_stripes_per_task = 1;
  u32 max_m = 0;
  u64 nbk = 0;      // bucket slots
  u64 nsbk = 0;     // stripe-bucket slots
  u64 nblk = 0;     // block slots (read-done flags)
  u64 child_cap = 0;
  u64 N = 0;
  u32 bc_grid = 0;   // base-case CTAs
  u64 bc_cap = 0;    // base-case capacity in use
};

template <int DT>
static void layout(LevelArgs &A, Arena &ar, const LevelPlan &P) {
  using Tr = Traits<DT>;
  constexpr int KI = Tr::KIDX, B = Tr::B, D = Tr::D;
  using Key = typename Tr::Key;
  const size_t T = P.lt.size(), S = P.stripe_task.size(), NP = P.perm_task.size();
  A.tasks = ar.take<LevelTask>(T);
  A.stripe_task = ar.take<u32>(S);
  A.perm_task = ar.take<u32>(NP);
  A.counters = ar.take<u32>(16);
  A.trees = ar.take<Key>(T * 2 * KI);
  A.counts = ar.take<u32>(P.nsbk);
  A.pfill = ar.take<u32>(P.nsbk);
  A.pcum = ar.take<u32>(P.nsbk);
  A.ptot = ar.take<u32>(P.nbk);
  A.fullblocks = ar.take<u32>(S);
  A.fcum = ar.take<u32>(S);
  A.partials = ar.take<char>(P.nsbk * (size_t)B * D);
  A.E = ar.take<u64>(P.nbk);
  A.fblk = ar.take<u32>(P.nbk);
  A.wr = ar.take<u64>(P.nbk * WR_STRIDE);
  A.overlap = ar.take<char>(P.nbk * (size_t)B * D);
  A.overflow = ar.take<char>(T * (size_t)B * D);
  A.ovf_used = ar.take<u32>(T);
  A.rdone = ar.take<unsigned char>(P.nblk);
  A.bid = ar.take<unsigned short>(P.nblk);
  A.task_done = ar.take<u32>(T);
  A.minmax = ar.take<u64>(2);
  A.measure_part = ar.take<u32>(P.measure_part.size());
  A.measure_task = ar.take<u32>(P.measure_task.size());
  A.measure_out = ar.take<PrepassPart>(P.measure_part.size() / 2);
  A.bc_scratch = BaseItem<DT>::SPLIT ? ar.take<char>((size_t)P.bc_grid * P.bc_cap * sizeof(typename BaseItem<DT>::Item))
                                     : nullptr;
  A.next_tasks = ar.take<TaskDesc>(P.child_cap);
  A.base_tasks = ar.take<TaskDesc>(P.child_cap);
  A.split_tasks = BaseItem<DT>::SPLIT ? ar.take<TaskDesc>(P.child_cap) : nullptr;
  A.ntasks = (u32)T;
  A.nstripes = (u32)S;
  A.nperm = (u32)NP;
  A.next_cap = (u32)P.child_cap;
  A.base_cap_tasks = (u32)P.child_cap;
}

// ------------------------------------------------------------------ per-dtype info
template <int DT> static int perm_occupancy() {
  static int occ = 0;
  if (!occ) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, permute_kernel<DT, ALGO_TREE>, PERM_THREADS, 0) !=
            cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  return occ;
}

template <int DT, int ALGO> static int set_attrs() {
  static bool done = false;
  if (done) return 0;
  if constexpr (Traits<DT>::D > 16) {
    CK(cudaFuncSetAttribute(classify_kernel<DT, ALGO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ClsSmem<DT>::bytes));
  } else {
    CK(cudaFuncSetAttribute(classify_v2_kernel<DT, ALGO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ClsV2<DT>::bytes));
  }
  CK(cudaFuncSetAttribute(basecase_kernel<DT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)BaseSmem<DT>::bytes));
  CK(cudaFuncSetAttribute(basecase_kernel<DT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)BaseSmem<DT>::bytes));
  CK(cudaFuncSetAttribute(sample_kernel<DT, ALGO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)sample_smem<DT>()));
  CK(cudaFuncSetAttribute(stripe_fix_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  done = true;
  return 0;
}

// ------------------------------------------------------------------ level planning
template <int DT>
static LevelPlan plan_level(const Ctx &c, const std::vector<TaskDesc> &tasks) {
  using Tr = Traits<DT>;
  constexpr int KI = Tr::KIDX, B = Tr::B;
  LevelPlan P;
  const u64 M = c.base_cap;
  for (auto &t : tasks) P.N += t.size;
  u64 spm = 6;  // stripes per SM: smaller CTAs shorten the tail of levels of unequal tasks
  if (const char *e = getenv("IPS4O_STRIPES_PER_SM")) spm = (u64)std::min(8, std::max(1, atoi(e)));  // tuning
  const u64 target_stripes = (u64)c.sms * spm;
  u64 se = round_up(ceil_div(P.N, target_stripes), B);
  se = std::max<u64>(se, round_up((u64)Tr::CLS_TILE * 2, B));
  const int occ = perm_occupancy<DT>();
  u64 G_perm = (u64)c.sms * occ;
  if (const char *e = getenv("IPS4O_PERM_CTAS_PER_SM")) G_perm = (u64)c.sms * (u64)std::max(1, atoi(e));  // tuning
  P.lt.resize(tasks.size());
  u64 bo = 0;
  for (size_t i = 0; i < tasks.size(); ++i) {
    const TaskDesc &t = tasks[i];
    LevelTask &L = P.lt[i];
    memset(&L, 0, sizeof L);
    L.t = t;
    // bucket count: expected child <= M/2 (DESIGN "Adaptive k"), P:983-990 analogue
    u64 kr = next_pow2_u64(ceil_div(2 * t.size, std::max<u64>(M, 1)));
    kr = std::min<u64>(std::max<u64>(kr, 2), (u64)c.k_max);
    L.k_req = (u32)kr;
    L.kidx = (u32)std::min<u64>(KI, c.algo == ALGO_TREE ? 2 * kr : kr);
    // oversampling alpha = max(ceil(0.2 log2 n'), alpha_min) (DESIGN R7)
    u64 alpha = (u64)std::ceil(0.2 * std::log2((double)std::max<u64>(t.size, 2)));
    alpha = std::max<u64>(alpha, (u64)c.alpha_min);
    u64 smax = (u64)sample_max<DT>();
    if (alpha * kr > smax) alpha = std::max<u64>(1, smax / kr);
    L.m = (u32)(alpha * kr);
    P.max_m = std::max(P.max_m, L.m);
    // stripes: task-relative, multiples of b
    u64 ns = std::max<u64>(1, ceil_div(t.size, se));
    u64 se_t = round_up(ceil_div(t.size, ns), B);
    ns = ceil_div(t.size, se_t);
    L.stripe_first = (u32)P.stripe_task.size();
    L.nstripes = (u32)ns;
    L.stripe_elems = se_t;
    for (u64 s = 0; s < ns; ++s) P.stripe_task.push_back((u32)i);
    P.max_stripes_per_task = std::max<u32>(P.max_stripes_per_task, (u32)ns);
    // permutation agents proportional to the task size (P:974-977 analogue)
    u64 np = (u64)std::llround((double)t.size * (double)G_perm / (double)std::max<u64>(P.N, 1));
    u64 nblocks = t.size / B;
    np = std::min<u64>(np, ceil_div(nblocks, (u64)PERM_WARPS * 2));
    np = std::max<u64>(np, 1);
    if (c.dbg_one_agent) np = 1;
    L.perm_first = (u32)P.perm_task.size();
    L.nperm = (u32)np;
    for (u64 s = 0; s < np; ++s) P.perm_task.push_back((u32)i);
    L.bucket_off = bo;
    bo += L.kidx + 1;
    L.blk_off = P.nblk;
    P.nblk += ceil_div(t.size, B) + 1;
    L.sbk_off = P.nsbk;
    P.nsbk += ns * L.kidx;
    P.child_cap += L.kidx;
    if (t.flags & TF_MEASURE) {
      const u32 np = (u32)std::min<u64>(MEAS_MAXPARTS, std::max<u64>(1, ceil_div(t.size, MEAS_PART_ELEMS)));
      P.measure_task.push_back((u32)i);
      P.measure_task.push_back((u32)(P.measure_part.size() / 2));
      P.measure_task.push_back(np);
      for (u32 q = 0; q < np; ++q) {
        P.measure_part.push_back((u32)i);
        P.measure_part.push_back(q | np << 16);
      }
    }
  }
  P.nbk = bo;
  P.bc_grid = (u32)std::min<u64>(std::max<u64>(P.child_cap, 1), (u64)c.sms);
  P.bc_cap = M;
  return P;
}

// host-side raw <-> internal key conversion (for the test hooks)
template <int DT> static void key_to_raw(const u64 *w, unsigned char *out) {
  if (DT == DT_REC100) {
    u128 k = ((u128)w[1] << 64) | w[0];
    for (int i = 0; i < 10; ++i) out[i] = (unsigned char)(k >> (8 * (9 - i)));
    memset(out + 10, 0, 6);
  } else if (DT == DT_F64) {
    u64 b = key_to_f64(w[0]);
    memcpy(out, &b, 8);
  } else if (DT == DT_U32) {
    u32 b = (u32)w[0];
    memcpy(out, &b, 4);
  } else if (DT == DT_QUARTET) {  // raw key = element bytes 0..23: a, b, c
    memcpy(out, &w[2], 8);
    memcpy(out + 8, &w[1], 8);
    memcpy(out + 16, &w[0], 8);
  } else {
    memcpy(out, &w[0], 8);
  }
}
template <int DT> static void raw_to_key(const unsigned char *in, u64 *w) {
  if (DT == DT_REC100) {
    u128 k = 0;
    for (int i = 0; i < 10; ++i) k = (k << 8) | in[i];
    w[0] = (u64)k;
    w[1] = (u64)(k >> 64);
    w[2] = 0;
  } else if (DT == DT_U32) {
    u32 b;
    memcpy(&b, in, 4);
    w[0] = b;
    w[1] = 0;
    w[2] = 0;
  } else if (DT == DT_QUARTET) {
    memcpy(&w[2], in, 8);
    memcpy(&w[1], in + 8, 8);
    memcpy(&w[0], in + 16, 8);
  } else {
    u64 b;
    memcpy(&b, in, 8);
    w[0] = DT == DT_F64 ? f64_to_key(b) : b;
    w[1] = 0;
    w[2] = 0;
  }
}

struct StepCapture {
  ips4o_step_info *info;
  int key_bytes;
};

// ------------------------------------------------------------------ one level
template <int DT, int ALGO>
static int run_level(Ctx &c, char *base, std::vector<TaskDesc> &tasks, std::vector<TaskDesc> &next,
                     StepCapture *cap, int level_no) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  constexpr int KI = Tr::KIDX;
  int rc = set_attrs<DT, ALGO>();
  if (rc) return rc;
  auto h0 = std::chrono::steady_clock::now();
  LevelPlan P = plan_level<DT>(c, tasks);
  LevelArgs A;
  memset(&A, 0, sizeof A);
  Arena dry;
  layout<DT>(A, dry, P);
  const size_t bytes = dry.used + 256;
  c.peak_scratch = std::max<u64>(c.peak_scratch, bytes);
  char *arena = nullptr;
  if (cudaMallocAsync((void **)&arena, bytes, c.st) != cudaSuccess) {
    cudaGetLastError();
    g_err = "cudaMallocAsync of level scratch failed";
    return IPS4O_ERR_NOMEM;
  }
  Arena ar;
  ar.base = arena;
  layout<DT>(A, ar, P);
  A.base = base;
  A.algo = ALGO;
  A.seed = c.seed;
  A.base_cap_elems = c.base_cap;
  // (16-bit run counters: a split bucket stays below 2^16 elements)
  A.base_split_elems = BaseItem<DT>::SPLIT ? std::min<u64>(2 * c.base_cap, 65535) : c.base_cap;
  A.dbg_one_agent = c.dbg_one_agent ? 1 : 0;
  // upload the plan (tasks, stripe->task, perm->task) through pinned staging
  const size_t T = P.lt.size(), S = P.stripe_task.size(), NP = P.perm_task.size();
  const size_t MPW = P.measure_part.size(), MTW = P.measure_task.size();
  const size_t up = T * sizeof(LevelTask) + (S + NP + MPW + MTW) * 4 + 64;
  rc = ensure_pinned(c, std::max<size_t>(up, (P.child_cap + 16) * sizeof(TaskDesc) + 4096));
  if (rc) return rc;
  char *hp = c.pinned;
  memcpy(hp, P.lt.data(), T * sizeof(LevelTask));
  memcpy(hp + T * sizeof(LevelTask), P.stripe_task.data(), S * 4);
  memcpy(hp + T * sizeof(LevelTask) + S * 4, P.perm_task.data(), NP * 4);
  CK(cudaMemcpyAsync(A.tasks, hp, T * sizeof(LevelTask), cudaMemcpyHostToDevice, c.st));
  CK(cudaMemcpyAsync((void *)A.stripe_task, hp + T * sizeof(LevelTask), S * 4, cudaMemcpyHostToDevice, c.st));
  CK(cudaMemcpyAsync((void *)A.perm_task, hp + T * sizeof(LevelTask) + S * 4, NP * 4, cudaMemcpyHostToDevice, c.st));
  if (MTW) {
    char *mp = hp + T * sizeof(LevelTask) + (S + NP) * 4;
    memcpy(mp, P.measure_part.data(), MPW * 4);
    memcpy(mp + MPW * 4, P.measure_task.data(), MTW * 4);
    CK(cudaMemcpyAsync((void *)A.measure_part, mp, MPW * 4, cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync((void *)A.measure_task, mp + MPW * 4, MTW * 4, cudaMemcpyHostToDevice, c.st));
  }
  CK(cudaMemsetAsync(A.counters, 0, 16 * 4, c.st));
  CK(cudaMemsetAsync(A.rdone, 0, P.nblk, c.st));
  CK(cudaMemsetAsync(A.task_done, 0, T * 4, c.st));
  CK(cudaMemsetAsync(A.minmax, 0xFF, 8, c.st));  // min = all ones
  CK(cudaMemsetAsync(A.minmax + 1, 0, 8, c.st));  // max = 0
  c.ms[KF_HOST] += std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - h0).count();

  // K0m exact key ranges of the TF_MEASURE tasks (DIGIT, DESIGN R27)
  if (ALGO == ALGO_DIGIT && MTW) {
    measure_part_kernel<DT><<<(unsigned)(MPW / 2), MEAS_THREADS, 0, c.st>>>(A);
    CKLAUNCH();
    const unsigned nm = (unsigned)(MTW / 3);
    measure_reduce_kernel<DT><<<(nm + 127) / 128, 128, 0, c.st>>>(A, nm);
    CKLAUNCH();
    if ((rc = mark(c, KF_SAMPLE))) return rc;
  }
  // K1 sampling + tree (or digit setup)
  {
    const u64 sp = next_pow2_u64(std::max<u64>(P.max_m, SORT_THREADS));
    size_t sm = ALGO == ALGO_TREE ? sample_smem<DT>((size_t)sp) : 0;
    if (ALGO == ALGO_TREE) {
      // the per-level layout lives in the kernel argument (A is passed by value)
      A.sample_p = (u32)sp;
    }
    sample_kernel<DT, ALGO><<<(unsigned)T, SAMPLE_THREADS, sm, c.st>>>(A);
    CKLAUNCH();
    if ((rc = mark(c, KF_SAMPLE))) return rc;
  }
  // K2 classification + block flush
  if constexpr (Traits<DT>::D > 16) {
    classify_kernel<DT, ALGO><<<(unsigned)S, Tr::CLS_THREADS, ClsSmem<DT>::bytes, c.st>>>(A);
  } else {
    classify_v2_kernel<DT, ALGO><<<(unsigned)S, ClsV2<DT>::NT, ClsV2<DT>::bytes, c.st>>>(A);
  }
  CKLAUNCH();
  if ((rc = mark(c, KF_CLASSIFY))) return rc;
  // K3 boundaries + stripe fix
  boundaries_kernel<DT><<<(unsigned)T, BND_THREADS, 0, c.st>>>(A);
  CKLAUNCH();
  if ((rc = mark(c, KF_BOUND))) return rc;
  stripe_fix_kernel<DT><<<(unsigned)S, FIX_THREADS, 0, c.st>>>(A);
  CKLAUNCH();
  if ((rc = mark(c, KF_FIX))) return rc;
  // K4 block permutation
#ifdef IPS4O_PERM_CLOCKS
  {
    unsigned long long z[6] = {0};
    CK(cudaMemcpyToSymbolAsync(g_perm_clk, z, sizeof z, 0, cudaMemcpyHostToDevice, c.st));
  }
#endif
#ifdef IPS4O_PERM_STATS
  {
    unsigned long long z[8] = {0};
    CK(cudaMemcpyToSymbolAsync(g_perm_stats, z, sizeof z, 0, cudaMemcpyHostToDevice, c.st));
  }
#endif
  permute_kernel<DT, ALGO><<<(unsigned)NP, PERM_THREADS, 0, c.st>>>(A);
  CKLAUNCH();
#ifdef IPS4O_PERM_CLOCKS
  {
    unsigned long long z[6];
    CK(cudaMemcpyFromSymbolAsync(z, g_perm_clk, sizeof z, 0, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    fprintf(stderr, "permute L%d cycles/step: fetch %.0f atomic %.0f load %.0f emptywait %.0f  (steps %llu)\n", level_no,
            (double)z[0] / z[4], (double)z[1] / z[4], (double)z[2] / z[4], (double)z[3] / z[4], z[4]);
  }
#endif
#ifdef IPS4O_PERM_STATS
  {
    unsigned long long z[8];
    CK(cudaMemcpyFromSymbolAsync(z, g_perm_stats, sizeof z, 0, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    fprintf(stderr, "permute L%d: attempts %llu fetches %llu misses %llu swaps %llu skips %llu empty %llu waits %llu polls %llu\n",
            level_no, z[0], z[1], z[2], z[3], z[4], z[5], z[6], z[7]);
  }
#endif
  if ((rc = mark(c, KF_PERM))) return rc;
  // K5 cleanup
  cleanup_save_kernel<DT><<<dim3((KI + CLN_WARPS - 1) / CLN_WARPS, (unsigned)T), CLN_WARPS * 32, 0, c.st>>>(A);
  CKLAUNCH();
  cleanup_fill_kernel<DT><<<dim3(P.max_stripes_per_task, (unsigned)T), FILL_THREADS, 0, c.st>>>(A);
  CKLAUNCH();
  if ((rc = mark(c, KF_CLEAN))) return rc;
  const bool last_level = c.max_levels > 0 && level_no + 1 >= c.max_levels;
  if (!cap) {
    // K6 scheduler, K7 base cases of this level
    schedule_kernel<DT, ALGO><<<(unsigned)T, SCHED_THREADS, 0, c.st>>>(A);
    CKLAUNCH();
    if ((rc = mark(c, KF_SCHED))) return rc;
    if (!c.skip_basecase) {
      const unsigned g = P.bc_grid;
      BaseSplitArgs sp{A.bc_scratch, (u32)c.base_cap, A.next_tasks, A.counters, A.next_cap,
                       reinterpret_cast<unsigned long long *>(A.counters + 6)};
      basecase_kernel<DT, false><<<g, BaseItem<DT>::THREADS, BaseSmem<DT>::bytes, c.st>>>(
          base, A.base_tasks, A.counters + 1, A.base_cap_tasks, sp);
      if constexpr (BaseItem<DT>::SPLIT) {
        CKLAUNCH();
        basecase_kernel<DT, true><<<g, BaseItem<DT>::THREADS, BaseSmem<DT>::bytes, c.st>>>(
            base, A.split_tasks, A.counters + 8, A.base_cap_tasks, sp);
      }
      CKLAUNCH();
      if ((rc = mark(c, KF_BASE))) return rc;
    }
  }
  // read back the counters (and the capture)
  u32 *hc = reinterpret_cast<u32 *>(c.pinned);
  CK(cudaMemcpyAsync(hc, A.counters, 16 * 4, cudaMemcpyDeviceToHost, c.st));
  LevelTask *hlt = reinterpret_cast<LevelTask *>(c.pinned + 256);
  if (cap) CK(cudaMemcpyAsync(hlt, A.tasks, sizeof(LevelTask), cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  flush_marks(c);
  if (hc[4] != 0) {
    g_err = "internal invariant violated: cleanup holes != overlap + partial buffers";
    cudaFreeAsync(arena, c.st);
    return IPS4O_ERR_CUDA;
  }
  if (cap) {
    ips4o_step_info *info = cap->info;
    const LevelTask L = *hlt;
    info->algo = ALGO;
    info->num_buckets = (int)L.K;
    info->l = (int)L.l;
    info->equality = (int)L.equality;
    info->shift = L.shift;
    info->k_used = (int)L.k_used;
    info->k_req = (int)L.k_req;
    info->samples = ALGO == ALGO_TREE ? (int)L.m : 0;
    info->kidx_budget = (int)L.kidx;
    info->level = 0;
    info->seed = c.seed;
    std::vector<u64> E(L.K + 1);
    CK(cudaMemcpy(E.data(), A.E + L.bucket_off, (L.K + 1) * 8, cudaMemcpyDeviceToHost));
    if (info->E) memcpy(info->E, E.data(), (L.K + 1) * 8);
    if (ALGO == ALGO_TREE) {
      std::vector<Key> tr(2 * KI);
      CK(cudaMemcpy(tr.data(), A.trees, 2 * KI * sizeof(Key), cudaMemcpyDeviceToHost));
      const int leaves = 1 << L.l;
      for (int i = 0; i < leaves; ++i) {
        u64 w[KEY_WORDS];
        key_to_words<Key>(tr[i], w);
        if (info->tree) key_to_raw<DT>(w, (unsigned char *)info->tree + (size_t)i * cap->key_bytes);
        key_to_words<Key>(tr[KI + i], w);
        if (info->splitter) key_to_raw<DT>(w, (unsigned char *)info->splitter + (size_t)i * cap->key_bytes);
      }
      if (info->tree) memset(info->tree, 0, cap->key_bytes);  // tree[0] is a dummy
    }
    next.clear();
    cudaFreeAsync(arena, c.st);
    return 0;
  }
  const u32 nnext = std::min<u32>(hc[0], A.next_cap);
  const u32 nbase = std::min<u32>(hc[1], A.base_cap_tasks);
  if (c.stats) {
    c.stats->basecase_tasks += nbase + std::min<u32>(hc[8], A.base_cap_tasks);
    c.stats->equal_elems += (u64)hc[2] | ((u64)hc[3] << 32);
  }
  next.resize(nnext);
  if (nnext && !last_level) {
    CK(cudaMemcpyAsync(c.pinned, A.next_tasks, nnext * sizeof(TaskDesc), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    memcpy(next.data(), c.pinned, nnext * sizeof(TaskDesc));
  } else {
    next.clear();
  }
  if (c.stats && !c.skip_basecase) c.stats->basecase_elems += (u64)hc[6] | ((u64)hc[7] << 32);
  CK(cudaFreeAsync(arena, c.st));
  return 0;
}

// ------------------------------------------------------------------ prepass
template <int DT>
static int run_prepass(Ctx &c, const char *base, u64 n, PrepassOut *out) {
  const int nparts = c.sms * 4;
  PrepassPart *parts = nullptr;
  PrepassOut *dout = nullptr;
  if (cudaMallocAsync((void **)&parts, nparts * sizeof(PrepassPart) + sizeof(PrepassOut) + 256, c.st) !=
      cudaSuccess) {
    cudaGetLastError();
    g_err = "cudaMallocAsync failed";
    return IPS4O_ERR_NOMEM;
  }
  dout = reinterpret_cast<PrepassOut *>(reinterpret_cast<char *>(parts) + round_up(nparts * sizeof(PrepassPart), 256));
  prepass_kernel<DT><<<nparts, PRE_THREADS, 0, c.st>>>(base, n, parts);
  CKLAUNCH();
  prepass_reduce_kernel<DT><<<1, 32, 0, c.st>>>(parts, nparts, dout);
  CKLAUNCH();
  int rc = mark(c, KF_PRE);
  if (rc) return rc;
  rc = ensure_pinned(c, 1 << 20);
  if (rc) return rc;
  CK(cudaMemcpyAsync(c.pinned, dout, sizeof(PrepassOut), cudaMemcpyDeviceToHost, c.st));
  CK(cudaFreeAsync(parts, c.st));
  CK(cudaStreamSynchronize(c.st));
  memcpy(out, c.pinned, sizeof(PrepassOut));
  return 0;
}

template <int DT>
static int run_base_single(Ctx &c, char *base, const TaskDesc &t) {
  int rc = set_attrs<DT, ALGO_TREE>();
  if (rc) return rc;
  char *buf = nullptr;
  if (cudaMallocAsync((void **)&buf, 512, c.st) != cudaSuccess) {
    cudaGetLastError();
    return IPS4O_ERR_NOMEM;
  }
  rc = ensure_pinned(c, 1 << 20);
  if (rc) return rc;
  memcpy(c.pinned, &t, sizeof t);
  u32 one = 1;
  memcpy(c.pinned + 256, &one, 4);
  CK(cudaMemcpyAsync(buf, c.pinned, 512, cudaMemcpyHostToDevice, c.st));
  BaseSplitArgs sp{nullptr, (u32)c.base_cap, nullptr, nullptr, 0, nullptr};  // m <= cap: no split
  basecase_kernel<DT, false><<<1, BaseItem<DT>::THREADS, BaseSmem<DT>::bytes, c.st>>>(
      base, reinterpret_cast<TaskDesc *>(buf), reinterpret_cast<u32 *>(buf + 256), 1, sp);
  CKLAUNCH();
  if ((rc = mark(c, KF_BASE))) return rc;
  CK(cudaFreeAsync(buf, c.st));
  CK(cudaStreamSynchronize(c.st));  // the pinned staging is reused by the caller
  if (c.stats) {
    c.stats->basecase_tasks += 1;
    c.stats->basecase_elems += t.size;
  }
  return 0;
}

template <int DT>
static int sort_impl(Ctx &c, char *base, u64 n, StepCapture *cap) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  int rc;
  if (c.base_cap == 0 || c.base_cap > (u64)Tr::BASE_CAP) c.base_cap = Tr::BASE_CAP;
  if (c.k_max <= 0 || c.k_max > Tr::KIDX) c.k_max = Tr::KIDX;
  TaskDesc root;
  memset(&root, 0, sizeof root);
  root.begin = 0;
  root.size = n;
  key_to_words<Key>((Key)0, root.lo);
  key_to_words<Key>(key_max<Key>(), root.hi);
  bool need_prepass = !c.skip_prepass || c.algo == ALGO_DIGIT || cap;
  if (need_prepass && !cap && !c.skip_prepass && c.algo == ALGO_TREE && sizeof(Key) == 8 &&
      n > c.base_cap && n >= (1ull << 22)) {
    // cheap sample pre-check: an ascending and a descending sampled pair
    // prove the input is not an easy input; the key range then comes from K2
    u32 *d = nullptr;
    if (cudaMallocAsync((void **)&d, 256, c.st) != cudaSuccess) {
      cudaGetLastError();
      return IPS4O_ERR_NOMEM;
    }
    presample_kernel<DT><<<1, 1024, 0, c.st>>>(base, n, d);
    CKLAUNCH();
    if ((rc = ensure_pinned(c, 1 << 20))) return rc;
    CK(cudaMemcpyAsync(c.pinned, d, 8, cudaMemcpyDeviceToHost, c.st));
    CK(cudaFreeAsync(d, c.st));
    CK(cudaStreamSynchronize(c.st));
    const u32 *f = reinterpret_cast<const u32 *>(c.pinned);
    if (f[0] && f[1]) {
      need_prepass = false;
      root.flags |= TF_MINMAX;
    }
    if ((rc = mark(c, KF_PRE))) return rc;
  }
  if (need_prepass) {
    PrepassOut po;
    if ((rc = run_prepass<DT>(c, base, n, &po))) return rc;
    Key mn = key_from_words<Key>(po.minkey), mx = key_from_words<Key>(po.maxkey);
    if (!cap && !c.skip_prepass) {
      if (po.nondecreasing) {  // P:1654 sorted input: nothing to do
        if (c.stats) c.stats->easy_input = (mn == mx) ? 3 : 1;
        return 0;
      }
      if (po.nonincreasing) {  // P:1655 decreasing: reverse and return
        reverse_kernel<DT><<<c.sms * 8, 256, 0, c.st>>>(base, n);
        CKLAUNCH();
        if ((rc = mark(c, KF_REV))) return rc;
        if (c.stats) c.stats->easy_input = 2;
        return 0;
      }
    }
    key_to_words<Key>(mn, root.lo);
    key_to_words<Key>(mx, root.hi);
    if (!(mn < mx) && !cap) return 0;  // all keys equal
  }
  if (!cap && n <= c.base_cap) {
    if (c.skip_basecase) return 0;
    return run_base_single<DT>(c, base, root);
  }
  std::vector<TaskDesc> tasks{root}, next;
  int level = 0;
  while (!tasks.empty()) {
    if (c.max_levels > 0 && level >= c.max_levels) break;
    if (c.stats && level < IPS4O_MAX_LEVELS_REPORTED) {
      c.stats->tasks_per_level[level] = tasks.size();
      u64 s = 0;
      for (auto &t : tasks) s += t.size;
      c.stats->elems_per_level[level] = s;
    }
    rc = c.algo == ALGO_TREE ? run_level<DT, ALGO_TREE>(c, base, tasks, next, cap, level)
                             : run_level<DT, ALGO_DIGIT>(c, base, tasks, next, cap, level);
    if (rc) return rc;
    ++level;
    if (c.stats) c.stats->levels = level;
    if (cap) break;
    tasks.swap(next);
  }
  return 0;
}

static int dtype_bytes(int dtype) {
  switch (dtype) {
    case DT_U64: return 8;
    case DT_F64: return 8;
    case DT_PAIR: return 16;
    case DT_REC100: return 100;
    case DT_U32: return 4;
    case DT_QUARTET: return 32;
    default: return 0;
  }
}

static int init_ctx(Ctx &c, void *stream, const ips4o_options *opt, ips4o_stats *out) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    g_err = "no CUDA device";
    return IPS4O_ERR_NOGPU;
  }
  CK(cudaGetDevice(&c.dev));
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c.dev));
  if (major != 10) {
    g_err = "this library is built for sm_100a (B200) only";
    return IPS4O_ERR_NOGPU;
  }
  CK(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, c.dev));
  c.st = reinterpret_cast<cudaStream_t>(stream);
  if (opt) {
    if (opt->algo != ALGO_TREE && opt->algo != ALGO_DIGIT) return IPS4O_ERR_INVALID;
    c.algo = opt->algo;
    if (opt->k_max) {
      if (opt->k_max < 2 || opt->k_max > 256 || (opt->k_max & (opt->k_max - 1))) return IPS4O_ERR_INVALID;
      c.k_max = opt->k_max;
    }
    if (opt->seed) c.seed = opt->seed;
    if (opt->alpha_min < 0) return IPS4O_ERR_INVALID;
    if (opt->alpha_min) c.alpha_min = opt->alpha_min;
    if (opt->base_cap < 0 || opt->max_levels < 0) return IPS4O_ERR_INVALID;
    c.base_cap = (u64)opt->base_cap;
    c.max_levels = opt->max_levels;
    c.skip_prepass = opt->skip_prepass != 0;
    c.skip_basecase = opt->skip_basecase != 0;
    c.timing = opt->timing != 0;
  }
  c.stats = out;
  if (out) memset(out, 0, sizeof *out);
  if (const char *e = getenv("IPS4O_DEBUG_ONE_AGENT")) c.dbg_one_agent = atoi(e) != 0;
  static bool pool_set = false;
  if (!pool_set) {
    // keep freed scratch in the pool between calls (setup amortisation,
    // the paper's "sorter object" P:3941-3944)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, c.dev) == cudaSuccess) {
      u64 thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_set = true;
  }
  if (c.timing) {
    CK(cudaEventCreate(&c.ev0));
    CK(cudaEventRecord(c.ev0, c.st));
  }
  return 0;
}

static void finish_ctx(Ctx &c, int rc) {
  if (c.timing && rc == 0) {
    cudaStreamSynchronize(c.st);
    flush_marks(c);
  }
  if (c.stats) {
    c.stats->scratch_bytes = c.peak_scratch;
    c.stats->kernel_launches = c.launches;
    float tot = 0;
    for (int i = 0; i < KF_TOTAL; ++i) {
      if (i != KF_HOST) tot += c.ms[i];
      c.stats->kernel_ms[i] = c.ms[i];
    }
    c.stats->kernel_ms[KF_TOTAL] = tot;
    if (rc == 0) cudaStreamSynchronize(c.st);
  }
  if (c.ev0) cudaEventDestroy(c.ev0);
}

}  // namespace ips4o

using namespace ips4o;

extern "C" {

int ips4o_sort_ex(void *ptr, uint64_t n, int dtype, void *stream, const ips4o_options *opt, ips4o_stats *out) {
  const int D = dtype_bytes(dtype);
  if (!D) return IPS4O_ERR_INVALID;
  if (out) memset(out, 0, sizeof *out);
  if (n <= 1) return IPS4O_OK;
  if (!ptr || ((uintptr_t)ptr & 15) || n >= (1ull << 32)) return IPS4O_ERR_INVALID;
  Ctx c;
  int rc = init_ctx(c, stream, opt, out);
  if (rc) return rc;
  char *base = reinterpret_cast<char *>(ptr);
  switch (dtype) {
    case DT_U64: rc = sort_impl<DT_U64>(c, base, n, nullptr); break;
    case DT_F64: rc = sort_impl<DT_F64>(c, base, n, nullptr); break;
    case DT_PAIR: rc = sort_impl<DT_PAIR>(c, base, n, nullptr); break;
    case DT_REC100: rc = sort_impl<DT_REC100>(c, base, n, nullptr); break;
    case DT_U32: rc = sort_impl<DT_U32>(c, base, n, nullptr); break;
    case DT_QUARTET: rc = sort_impl<DT_QUARTET>(c, base, n, nullptr); break;
  }
  finish_ctx(c, rc);
  return rc;
}

int ips4o_sort(void *ptr, uint64_t n, int dtype, void *stream) {
  return ips4o_sort_ex(ptr, n, dtype, stream, nullptr, nullptr);
}

int ips4o_sort_host(void *host_ptr, uint64_t n, int dtype, const ips4o_options *opt, ips4o_stats *out) {
  const int D = dtype_bytes(dtype);
  if (!D) return IPS4O_ERR_INVALID;
  if (n <= 1) return IPS4O_OK;
  if (!host_ptr || ((uintptr_t)host_ptr & 15) || n >= (1ull << 32)) return IPS4O_ERR_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return IPS4O_ERR_NOGPU;
  }
  const size_t bytes = (size_t)n * D;
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaPointerAttributes pa;
  bool pinned = cudaPointerGetAttributes(&pa, host_ptr) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  char *dev = nullptr;
  if (cudaMallocAsync((void **)&dev, bytes, st) != cudaSuccess) {
    cudaGetLastError();
    cudaStreamDestroy(st);
    return IPS4O_ERR_NOMEM;
  }
  const size_t CH = 64ull << 20;
  char *stage[2] = {nullptr, nullptr};
  cudaEvent_t done[2];
  if (!pinned) {
    CK(cudaMallocHost(&stage[0], CH));
    CK(cudaMallocHost(&stage[1], CH));
    CK(cudaEventCreate(&done[0]));
    CK(cudaEventCreate(&done[1]));
  }
  char *h = reinterpret_cast<char *>(host_ptr);
  if (pinned) {
    CK(cudaMemcpyAsync(dev, h, bytes, cudaMemcpyHostToDevice, st));
  } else {
    int k = 0;
    for (size_t off = 0; off < bytes; off += CH, k ^= 1) {
      size_t len = std::min(CH, bytes - off);
      if (off >= 2 * CH) CK(cudaEventSynchronize(done[k]));
      memcpy(stage[k], h + off, len);
      CK(cudaMemcpyAsync(dev + off, stage[k], len, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(done[k], st));
    }
  }
  int rc = ips4o_sort_ex(dev, n, dtype, st, opt, out);
  if (rc == 0) {
    if (pinned) {
      CK(cudaMemcpyAsync(h, dev, bytes, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    } else {
      for (size_t off = 0; off < bytes; off += CH) {
        size_t len = std::min(CH, bytes - off);
        CK(cudaMemcpyAsync(stage[0], dev + off, len, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        memcpy(h + off, stage[0], len);
      }
    }
  }
  cudaFreeAsync(dev, st);
  cudaStreamSynchronize(st);
  if (!pinned) {
    cudaFreeHost(stage[0]);
    cudaFreeHost(stage[1]);
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
  }
  cudaStreamDestroy(st);
  return rc;
}

uint64_t ips4o_scratch_bytes(uint64_t n, int dtype, const ips4o_options *opt) {
  // Upper bound: the largest level arena over all possible levels + prepass.
  // #tasks at a level >= 2 is at most n / (M + 1) (only buckets larger than M
  // recurse); stripes <= 4 * SMs + #tasks; bucket slots <= sum (kidx + 1).
  int D = dtype_bytes(dtype);
  if (!D) return 0;
  int B = 0, KI = 0, keyb = 8;
  u64 M = 0;
  switch (dtype) {
    case DT_U64: B = Traits<DT_U64>::B; KI = Traits<DT_U64>::KIDX; M = Traits<DT_U64>::BASE_CAP; break;
    case DT_F64: B = Traits<DT_F64>::B; KI = Traits<DT_F64>::KIDX; M = Traits<DT_F64>::BASE_CAP; break;
    case DT_PAIR: B = Traits<DT_PAIR>::B; KI = Traits<DT_PAIR>::KIDX; M = Traits<DT_PAIR>::BASE_CAP; break;
    case DT_U32: B = Traits<DT_U32>::B; KI = Traits<DT_U32>::KIDX; M = Traits<DT_U32>::BASE_CAP; break;
    case DT_QUARTET: B = Traits<DT_QUARTET>::B; KI = Traits<DT_QUARTET>::KIDX; M = Traits<DT_QUARTET>::BASE_CAP; keyb = 24; break;
    default: B = Traits<DT_REC100>::B; KI = Traits<DT_REC100>::KIDX; M = Traits<DT_REC100>::BASE_CAP; keyb = 16; break;
  }
  if (opt && opt->base_cap > 0 && (u64)opt->base_cap < M) M = (u64)opt->base_cap;
  int sms = 148;
  int dev;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  // Level 1 has one task; at a level >= 2 every task is a bucket larger than
  // M, so T <= n / (M + 1).  kidx_t <= 2 * next_pow2(ceil(2 s_t / M)) gives
  // sum kidx_t <= 8n/M + 4T; stripes per task <= s_t / se + 1 with
  // se >= n / (8 SMs) gives S <= 8 SMs + T and sum ns_t kidx_t <= 8 SMs KI + sum kidx_t.
  const u64 T = std::max<u64>(1, n / (M + 1));
  const u64 S = (u64)sms * 8 + T;  // plan_level: <= 8 stripes per SM (+1 per task)
  const u64 NP = (u64)sms * 16 + T;
  const u64 sum_kidx = std::min<u64>(T * KI, 8 * (n / std::max<u64>(M, 1) + 1) + 4 * T) + KI;
  const u64 NBK = sum_kidx + T;
  const u64 NSBK = (u64)sms * 8 * KI + sum_kidx;
  const u64 BD = (u64)B * D;
  u64 bytes = 0;
  auto add = [&](u64 b) { bytes += round_up(b, 256); };
  add(T * sizeof(LevelTask));
  add(S * 4);
  add(NP * 4);
  add(64);
  add(T * 2 * KI * keyb);
  add(NSBK * 4);
  add(NSBK * 4);
  add(S * 4);
  add(NSBK * BD);
  add(NBK * 8);
  add(NBK * 4);
  add(NBK * WR_STRIDE * 8);
  add(NBK * BD);
  add(T * BD);
  add(T * 4);
  add(n / B + 2 * T);                   // read-done flags
  add(2 * (n / B + 2 * T));             // block buckets
  add(T * 4);                           // task_done
  add(16);                              // minmax
  const u64 MP = T + n / MEAS_PART_ELEMS + 1;  // K0m parts
  add(MP * 8);
  add(T * 12);
  add(MP * sizeof(PrepassPart));
  add(3 * sum_kidx * sizeof(TaskDesc));  // next, base, split lists
  add((u64)sms * M * (u64)D);  // base-case split scratch (one capacity per CTA)
  return bytes + 256;
}

const char *ips4o_status_string(int status) {
  switch (status) {
    case IPS4O_OK: return "ok";
    case IPS4O_ERR_INVALID: return "invalid argument";
    case IPS4O_ERR_NOMEM: return "out of device or pinned memory";
    case IPS4O_ERR_CUDA: return g_err.c_str();
    case IPS4O_ERR_NOGPU: return "no usable CUDA device (sm_100 required)";
    default: return "unknown status";
  }
}

int ips4o_get_dtype_info(int dtype, ips4o_dtype_info *out) {
  if (!out) return IPS4O_ERR_INVALID;
  switch (dtype) {
#define FILL(DTc)                                 \
  out->elem_bytes = Traits<DTc>::D;               \
  out->block_elems = Traits<DTc>::B;              \
  out->kidx_max = Traits<DTc>::KIDX;              \
  out->base_cap = Traits<DTc>::BASE_CAP;          \
  out->key_bytes = DTc == DT_REC100 ? 16 : DTc == DT_U32 ? 4 : DTc == DT_QUARTET ? 24 : 8; \
  return IPS4O_OK;
    case DT_U64: FILL(DT_U64)
    case DT_F64: FILL(DT_F64)
    case DT_PAIR: FILL(DT_PAIR)
    case DT_REC100: FILL(DT_REC100)
    case DT_U32: FILL(DT_U32)
    case DT_QUARTET: FILL(DT_QUARTET)
#undef FILL
    default: return IPS4O_ERR_INVALID;
  }
}

int ips4o_partition_step(void *ptr, uint64_t n, int dtype, void *stream, const ips4o_options *opt,
                         ips4o_step_info *info) {
  const int D = dtype_bytes(dtype);
  if (!D || !info) return IPS4O_ERR_INVALID;
  if (n < 2 || !ptr || ((uintptr_t)ptr & 15) || n >= (1ull << 32)) return IPS4O_ERR_INVALID;
  Ctx c;
  int rc = init_ctx(c, stream, opt, nullptr);
  if (rc) return rc;
  StepCapture cap{info, dtype == DT_REC100 ? 16 : dtype == DT_U32 ? 4 : dtype == DT_QUARTET ? 24 : 8};
  char *base = reinterpret_cast<char *>(ptr);
  switch (dtype) {
    case DT_U64: rc = sort_impl<DT_U64>(c, base, n, &cap); break;
    case DT_F64: rc = sort_impl<DT_F64>(c, base, n, &cap); break;
    case DT_PAIR: rc = sort_impl<DT_PAIR>(c, base, n, &cap); break;
    case DT_REC100: rc = sort_impl<DT_REC100>(c, base, n, &cap); break;
    case DT_U32: rc = sort_impl<DT_U32>(c, base, n, &cap); break;
    case DT_QUARTET: rc = sort_impl<DT_QUARTET>(c, base, n, &cap); break;
  }
  if (rc == 0) {
    cudaError_t e = cudaStreamSynchronize(c.st);
    if (e != cudaSuccess) rc = set_cuda_err(e, "partition_step sync", __LINE__);
  }
  finish_ctx(c, rc);
  return rc;
}

}  // extern "C"

namespace ips4o {
template <int DT>
static int classify_impl(const void *elems, u64 n, const unsigned char *raw, int u, int eq, u32 *out,
                         cudaStream_t st) {
  using Key = typename Traits<DT>::Key;
  const int kb = DT == DT_REC100 ? 16 : DT == DT_U32 ? 4 : DT == DT_QUARTET ? 24 : 8;
  int leaves = 1;
  while (leaves < u + 1) leaves <<= 1;
  if (leaves > 256) return IPS4O_ERR_INVALID;
  int l = 0;
  while ((1 << l) < leaves) ++l;
  std::vector<Key> keys(u), tree(leaves), spl(leaves);
  for (int i = 0; i < u; ++i) {
    u64 w[KEY_WORDS];
    raw_to_key<DT>(raw + (size_t)i * kb, w);
    keys[i] = key_from_words<Key>(w);
  }
  // P:446-451 padding and P:402-406 breadth-first layout (product-side copy)
  for (int i = 0; i < leaves; ++i) spl[i] = keys[i < u ? i : u - 1];
  tree[0] = 0;
  for (int i = 1; i < leaves; ++i) {
    int d = 0;
    while ((2 << d) <= i) ++d;
    int p = i - (1 << d);
    int rank = (2 * p + 1) * (1 << (l - 1 - d)) - 1;
    tree[i] = spl[rank];
  }
  Key *dt = nullptr;
  CK(cudaMalloc((void **)&dt, 2 * leaves * sizeof(Key)));
  CK(cudaMemcpy(dt, tree.data(), leaves * sizeof(Key), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dt + leaves, spl.data(), leaves * sizeof(Key), cudaMemcpyHostToDevice));
  if (n) {
    unsigned g = (unsigned)std::min<u64>(ceil_div(n, 256), 148 * 8);
    classify_test_kernel<DT><<<g, 256, 0, st>>>(reinterpret_cast<const char *>(elems), n, dt, dt + leaves, l, eq, out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_err(e, "classify_test_kernel", __LINE__);
  }
  CK(cudaStreamSynchronize(st));
  CK(cudaFree(dt));
  return 0;
}
}  // namespace ips4o

extern "C" int ips4o_classify(const void *elems, uint64_t n, int dtype, const void *splitters, int u, int equality,
                              uint32_t *out, void *stream) {
  if (!dtype_bytes(dtype) || u < 1 || !splitters || (n && (!elems || !out))) return IPS4O_ERR_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned char *raw = reinterpret_cast<const unsigned char *>(splitters);
  switch (dtype) {
    case DT_U64: return classify_impl<DT_U64>(elems, n, raw, u, equality, out, st);
    case DT_F64: return classify_impl<DT_F64>(elems, n, raw, u, equality, out, st);
    case DT_PAIR: return classify_impl<DT_PAIR>(elems, n, raw, u, equality, out, st);
    case DT_U32: return classify_impl<DT_U32>(elems, n, raw, u, equality, out, st);
    case DT_QUARTET: return classify_impl<DT_QUARTET>(elems, n, raw, u, equality, out, st);
    default: return classify_impl<DT_REC100>(elems, n, raw, u, equality, out, st);
  }
}
