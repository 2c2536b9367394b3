// ips4o.cu -- host side and C ABI (include/ips4o.h) of the B200-native
// in-place samplesort partitioning step.  Product code: no PyTorch types, no
// CPU fallback, nothing from oracle/.
//
// A sort is ONE host launch (entry_kernel, k_plan.cuh) into the caller's
// stream, bracketed by a stream-ordered allocation and free of its scratch
// from a library-owned memory pool.  The levels of the recursion are planned
// and launched on the device (DESIGN "Device planner"), so ips4o_sort returns
// without synchronising and can be captured into a CUDA graph.  The host only
// validates arguments, sizes the scratch (with the planner's own plan
// arithmetic) and, when statistics are requested, reads the control block
// back after a synchronisation.  All element work runs in the kernels of
// k_*.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
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
#include "k_plan.cuh"
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

enum KFam { KF_PRE = 0, KF_SAMPLE, KF_CLASSIFY, KF_BOUND, KF_FIX, KF_PERM, KF_CLEAN, KF_SCHED, KF_BASE, KF_REV, KF_PLAN, KF_TOTAL };
static const int kSlotFamily[KS_COUNT] = {
    KF_PRE,  KF_PRE,  KF_PRE,   KF_SAMPLE, KF_SAMPLE, KF_SAMPLE, KF_CLASSIFY, KF_BOUND,
    KF_FIX,  KF_PERM, KF_CLEAN, KF_CLEAN,  KF_BASE,   KF_BASE,   KF_REV,      KF_PLAN, KF_BASE};

static const int NDT = 6;

// ------------------------------------------------------------------ per-device state
// Everything the library keeps between calls, per device: its memory pool
// (scratch is allocated stream-ordered from it; the pool keeps freed memory
// for the next call -- the paper's reusable "sorter object", P:3941-3944 --
// without touching the device's default pool), a status word that device
// code ORs error flags into, and the kernel attributes / occupancy queries.
struct DevState {
  std::once_flag init_flag;
  int init_rc = 0;
  std::string init_err;
  int sms = 148;
  cudaMemPool_t pool = nullptr;
  u32 *status = nullptr;
  std::once_flag attr_flag[NDT][2];
  int attr_rc[NDT][2] = {};
  int perm_occ[NDT] = {};
};
constexpr int MAX_DEVICES = 64;
static DevState g_dev[MAX_DEVICES];

template <int DT, int ALGO> static int set_attrs_once() {
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
  return 0;
}

static int device_state(DevState *&ds) {
  int dev = 0, ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    g_err = "no CUDA device";
    return IPS4O_ERR_NOGPU;
  }
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= MAX_DEVICES) {
    g_err = "device index out of range";
    return IPS4O_ERR_NOGPU;
  }
  ds = &g_dev[dev];
  std::call_once(ds->init_flag, [ds, dev]() {
    int major = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess || major != 10) {
      cudaGetLastError();
      ds->init_rc = IPS4O_ERR_NOGPU;
      ds->init_err = "this library is built for sm_100a (B200) only";
      return;
    }
    cudaDeviceGetAttribute(&ds->sms, cudaDevAttrMultiProcessorCount, dev);
    cudaMemPoolProps props;
    memset(&props, 0, sizeof props);
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&ds->pool, &props) != cudaSuccess) {
      ds->init_rc = set_cuda_err(cudaGetLastError(), "cudaMemPoolCreate", __LINE__);
      ds->init_err = g_err;
      return;
    }
    u64 thr = ~0ull;
    cudaMemPoolSetAttribute(ds->pool, cudaMemPoolAttrReleaseThreshold, &thr);
    if (cudaMalloc((void **)&ds->status, 4) != cudaSuccess || cudaMemset(ds->status, 0, 4) != cudaSuccess) {
      ds->init_rc = set_cuda_err(cudaGetLastError(), "status word", __LINE__);
      ds->init_err = g_err;
      return;
    }
    for (int d = 0; d < NDT; ++d) ds->perm_occ[d] = 0;
  });
  if (ds->init_rc) g_err = ds->init_err;
  return ds->init_rc;
}

template <int DT, int ALGO> static int ensure_attrs(DevState *ds) {
  std::call_once(ds->attr_flag[DT][ALGO], [ds]() {
    ds->attr_rc[DT][ALGO] = set_attrs_once<DT, ALGO>();
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, permute_kernel<DT, ALGO_TREE>, PERM_THREADS, 0) !=
            cudaSuccess ||
        occ < 1)
      occ = 1;
    cudaGetLastError();
    ds->perm_occ[DT] = occ;
  });
  return ds->attr_rc[DT][ALGO];
}

static int env_int(const char *name, int dflt, int lo, int hi) {
  const char *e = getenv(name);
  if (!e) return dflt;
  return std::min(hi, std::max(lo, atoi(e)));
}

// Scratch of one sort: the control block, two pending task lists, the arena.
struct ScratchPlan {
  u64 ctl_bytes, list_cap, list_bytes, arena_off, arena_cap, total;
};

template <int DT> static ScratchPlan scratch_plan(const SortCfg &c, u64 arena_bytes) {
  ScratchPlan s;
  s.ctl_bytes = rup(sizeof(SortCtl), 256);
  // a pending task is larger than M and tasks are disjoint (DESIGN "Device planner")
  s.list_cap = c.n / (c.base_cap + 1) + 2;
  s.list_bytes = rup(2 * s.list_cap * sizeof(TaskDesc), 256);
  s.arena_off = s.ctl_bytes + s.list_bytes;
  s.arena_cap = host_arena_bytes<DT>(c, arena_bytes);
  s.total = s.arena_off + s.arena_cap;
  return s;
}

struct Call {
  int algo = ALGO_TREE;
  int k_max = 0;
  u64 seed = 0x1F4A2C7ull;
  int alpha_min = 64;
  u64 base_cap = 0;
  int max_levels = 0;
  u64 arena_bytes = 0;
  bool skip_prepass = false, skip_basecase = false, timing = false, capture = false;
  const char *ext_spl = nullptr;  // ips4o_partition_splitters: the given splitters (device)
  int ext_n = 0;
};

static int parse_options(Call &k, const ips4o_options *opt) {
  if (!opt) return 0;
  if (opt->algo != ALGO_TREE && opt->algo != ALGO_DIGIT) return IPS4O_ERR_INVALID;
  k.algo = opt->algo;
  if (opt->k_max) {
    if (opt->k_max < 2 || opt->k_max > 256 || (opt->k_max & (opt->k_max - 1))) return IPS4O_ERR_INVALID;
    // the tree needs >= 3 splitters to guarantee progress (a single splitter
    // equal to the task's maximum leaves everything in one bucket)
    if (opt->algo == ALGO_TREE && opt->k_max < 4) return IPS4O_ERR_INVALID;
    k.k_max = opt->k_max;
  }
  if (opt->seed) k.seed = opt->seed;
  if (opt->alpha_min < 0 || opt->base_cap < 0 || opt->max_levels < 0) return IPS4O_ERR_INVALID;
  if (opt->alpha_min) k.alpha_min = opt->alpha_min;
  k.base_cap = (u64)opt->base_cap;
  k.max_levels = opt->max_levels;
  k.skip_prepass = opt->skip_prepass != 0;
  k.skip_basecase = opt->skip_basecase != 0;
  k.timing = opt->timing != 0;
  if (opt->arena_mb < 0) return IPS4O_ERR_INVALID;
  k.arena_bytes = (u64)opt->arena_mb << 20;
  return 0;
}

template <int DT> static SortCfg make_cfg(const Call &k, const DevState &ds, char *base, u64 n) {
  using Tr = Traits<DT>;
  SortCfg c;
  memset(&c, 0, sizeof c);
  c.base = base;
  c.n = n;
  c.seed = k.seed;
  c.base_cap = (k.base_cap == 0 || k.base_cap > (u64)Tr::BASE_CAP) ? (u64)Tr::BASE_CAP : k.base_cap;
  // (16-bit run counters: a split bucket stays below 2^16 elements)
  c.base_split = BaseItem<DT>::SPLIT ? std::min<u64>(2 * c.base_cap, 65535) : c.base_cap;
  c.algo = k.algo;
  c.k_max = (k.k_max <= 0 || k.k_max > Tr::KIDX) ? Tr::KIDX : k.k_max;
  c.alpha_min = k.alpha_min;
  c.max_levels = k.capture ? 1 : k.max_levels;
  c.skip_prepass = k.skip_prepass;
  c.skip_basecase = k.skip_basecase;
  c.timing = k.timing;
  c.capture = k.capture;
  c.ext_spl = k.ext_spl;
  c.ext_n = k.ext_n;
  c.dbg_one_agent = env_int("IPS4O_DEBUG_ONE_AGENT", 0, 0, 1);
  // profiling mode: every round launched from the host (one synchronisation
  // per round) so that ncu sees each kernel; same plans, grids and kernels
  c.host_levels = k.capture ? 0 : env_int("IPS4O_HOST_LEVELS", 0, 0, 1);
  c.sms = ds.sms;
  // stripes per SM: smaller CTAs shorten the tail of levels of unequal tasks
  c.spm = env_int("IPS4O_STRIPES_PER_SM", 6, 1, 8);
  const int occ = env_int("IPS4O_PERM_CTAS_PER_SM", std::max(1, ds.perm_occ[DT]), 1, 32);
  c.g_perm = (u32)(ds.sms * occ);
  return c;
}

static u64 scratch_for(int dtype, const SortCfg &c, u64 arena_bytes) {
  switch (dtype) {
    case DT_U64: return scratch_plan<DT_U64>(c, arena_bytes).total;
    case DT_F64: return scratch_plan<DT_F64>(c, arena_bytes).total;
    case DT_PAIR: return scratch_plan<DT_PAIR>(c, arena_bytes).total;
    case DT_REC100: return scratch_plan<DT_REC100>(c, arena_bytes).total;
    case DT_U32: return scratch_plan<DT_U32>(c, arena_bytes).total;
    default: return scratch_plan<DT_QUARTET>(c, arena_bytes).total;
  }
}

// Host view of the control block (everything before the pre-pass parts).
constexpr size_t CTL_READ = offsetof(SortCtl, parts);

static const char *err_text(u32 f) {
  if (f & ERR_CLEANUP) return "internal invariant violated: cleanup holes != overlap + partial buffers";
  if (f & ERR_LIST_OVERFLOW) return "internal error: task list overflow";
  if (f & ERR_NO_PROGRESS) return "internal error: a task made no progress";
  if (f & ERR_LAUNCH) return "a device-side kernel launch failed";
  if (f & ERR_ARENA) return "a task does not fit the scratch arena";
  if (f & ERR_CHECK) return "checked build: an index failed its bounds check";
  return "device error";
}

static void fill_stats(const SortCtl &h, ips4o_stats *out, u64 scratch) {
  memset(out, 0, sizeof *out);
  out->scratch_bytes = scratch;
  out->levels = (int)h.levels;
  out->easy_input = (int)h.easy;
  for (int r = 0; r < IPS4O_MAX_LEVELS_REPORTED && r < MAX_ROUNDS; ++r) {
    out->tasks_per_level[r] = h.tasks_per_round[r];
    out->elems_per_level[r] = h.elems_per_round[r];
  }
  out->basecase_tasks = h.base_tasks;
  out->basecase_elems = (u64)h.counters[6] | ((u64)h.counters[7] << 32);
  out->equal_elems = (u64)h.counters[2] | ((u64)h.counters[3] << 32);
  out->kernel_launches = h.launches;
  out->deferred_tasks = h.deferred;
  double fam[IPS4O_NUM_KERNELS] = {0};
  unsigned long long t0 = ~0ull, t1 = 0;
  for (int r = 0; r < MAX_ROUNDS; ++r)
    for (int k = 0; k < KS_COUNT; ++k) {
      const unsigned long long a = h.tslot[r][k][0], b = h.tslot[r][k][1];
      if (a == ~0ull || b < a) continue;
      fam[kSlotFamily[k]] += (double)(b - a) * 1e-6;
      t0 = std::min(t0, a);
      t1 = std::max(t1, b);
    }
  for (int i = 0; i < KF_TOTAL; ++i) out->kernel_ms[i] = (float)fam[i];
  for (int r = 0; r < IPS4O_MAX_LEVELS_REPORTED && r < MAX_ROUNDS; ++r)
    for (int k = 0; k < KS_COUNT; ++k) {
      const unsigned long long a = h.tslot[r][k][0], b = h.tslot[r][k][1];
      if (a == ~0ull || b < a) continue;
      const int c = k == KS_CLASSIFY ? 0 : k == KS_PERM ? 1 : (k == KS_BASE || k == KS_SPLIT || k == KS_NARROW) ? 2 : 3;
      out->round_kernel_ms[r][c] += (float)((double)(b - a) * 1e-6);
    }
  out->kernel_ms[KF_TOTAL] = t1 > t0 ? (float)((double)(t1 - t0) * 1e-6) : 0.f;
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

template <int DT> struct Sorter {
  // Enqueue the sort; with `hctl` (stats / test hook) synchronise and read the
  // control block back before the scratch is released.
  static int run(const Call &k, char *base, u64 n, cudaStream_t st, SortCtl *hctl, u64 *scratch_out,
                 ips4o_step_info *cap) {
    DevState *ds = nullptr;
    int rc = device_state(ds);
    if (rc) return rc;
    rc = k.algo == ALGO_TREE ? ensure_attrs<DT, ALGO_TREE>(ds) : ensure_attrs<DT, ALGO_DIGIT>(ds);
    if (rc) return rc;
    SortCfg c = make_cfg<DT>(k, *ds, base, n);
    const ScratchPlan sp = scratch_plan<DT>(c, k.arena_bytes);
    char *scratch = nullptr;
    if (cudaMallocFromPoolAsync((void **)&scratch, sp.total, ds->pool, st) != cudaSuccess) {
      cudaGetLastError();
      g_err = "scratch allocation from the library pool failed";
      return IPS4O_ERR_NOMEM;
    }
    c.scratch = scratch;
    c.list_cap = sp.list_cap;
    c.arena_off = sp.arena_off;
    c.arena_cap = sp.arena_cap;
    c.status = ds->status;
    if (scratch_out) *scratch_out = sp.total;
    u64 host_launches = k.algo == ALGO_TREE ? enqueue<ALGO_TREE>(c, st) : enqueue<ALGO_DIGIT>(c, st);
    if (c.host_levels && !(c.n <= c.base_cap)) {
      rc = k.algo == ALGO_TREE ? host_rounds<ALGO_TREE>(c, st, host_launches) : host_rounds<ALGO_DIGIT>(c, st, host_launches);
      if (rc) {
        cudaFreeAsync(scratch, st);
        return rc;
      }
    }
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) {
      cudaFreeAsync(scratch, st);
      return set_cuda_err(le, "entry_kernel launch", __LINE__);
    }
    if (hctl) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = cudaMemcpy(hctl, scratch, CTL_READ, cudaMemcpyDeviceToHost);
      hctl->launches += host_launches;
      if (e == cudaSuccess && cap) rc = capture_step(*hctl, cap);
      cudaFreeAsync(scratch, st);
      if (e != cudaSuccess) return set_cuda_err(e, "sort (synchronised)", __LINE__);
      if (rc) return rc;
      if (hctl->error) {
        g_err = err_text(hctl->error);
        return IPS4O_ERR_CUDA;
      }
      return 0;
    }
    CK(cudaFreeAsync(scratch, st));
    return 0;
  }

  // The host's part of a sort, all enqueued on `st` without waiting: the
  // entry kernel (easy-input pre-check, plan of round 0), the full pre-pass
  // when the entry kernel may need it (its kernels exit at once otherwise),
  // then round 0 itself -- its plan is a function of n alone, so the host
  // computes the same grids and arguments the device planner lays out
  // (level_args); the kernels run only if the device set `go` -- and the
  // device planner of round 1, which launches every later round itself.
  template <int ALGO> static u64 enqueue(const SortCfg &c, cudaStream_t st) {
    SortCtl *ctl = reinterpret_cast<SortCtl *>(c.scratch);
    u64 nl = 0;
    entry_kernel<DT, ALGO><<<1, PLAN_THREADS, 0, st>>>(c);
    ++nl;
    using Key = typename Traits<DT>::Key;
    const bool presample = !c.capture && !c.skip_prepass && c.algo == ALGO_TREE && sizeof(Key) == 8 &&
                           c.n > c.base_cap && c.n >= (1ull << 22);
    const bool may_prepass = !c.skip_prepass || c.algo == ALGO_DIGIT || c.capture;
    unsigned long long *ts0 = c.timing ? &ctl->tslot[0][0][0] : nullptr;
    if (may_prepass) {
      const int nparts = std::min(c.sms * PRE_PARTS_PER_SM, MAX_PRE_PARTS);
      const u32 *need = presample ? &ctl->need_prepass : nullptr;
      prepass_kernel<DT><<<nparts, PRE_THREADS, 0, st>>>(c.base, c.n, ctl->parts, ts0, need);
      prepass_reduce_kernel<DT><<<1, PRERED_THREADS, 0, st>>>(ctl->parts, nparts, &ctl->pre, ts0, need);
      driver_kernel<DT, ALGO><<<1, PLAN_THREADS, 0, st>>>(ctl, 1);
      nl += 3;
    }
    if (!c.capture && c.n <= c.base_cap) {
      if (!c.skip_basecase) {
        const BaseSplitArgs sp{nullptr, (u32)c.base_cap, nullptr, nullptr, 0, nullptr, &ctl->error};  // m <= cap
        basecase_kernel<DT, false><<<1, BaseItem<DT>::THREADS, BaseSmem<DT>::bytes, st>>>(
            c.base, reinterpret_cast<const TaskDesc *>(c.scratch + c.arena_off), ctl->counters + 1, 1, sp, ts0);
        ++nl;
      }
      return nl;
    }
    const LevelArgs A = level_args<DT, ALGO>(ctl, c, root_totals<DT>(c), 0, 0, nullptr);
    for (int s = 0; s < ST_N; ++s)
      if ((A.stages >> s) & 1u) {
        host_stage<ALGO>(A, s, st);
        ++nl;
      }
    return nl;
  }

  // Profiling mode: the device planner plans each later round (phase 3, no
  // launches); the host reads the plan back and launches the round.
  template <int ALGO> static int host_rounds(const SortCfg &c, cudaStream_t st, u64 &nl) {
    SortCtl *ctl = reinterpret_cast<SortCtl *>(c.scratch);
    for (;;) {
      u32 r0 = 0, r1 = 0;
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpy(&r0, &ctl->round, 4, cudaMemcpyDeviceToHost));
      driver_kernel<DT, ALGO><<<1, PLAN_THREADS, 0, st>>>(ctl, 3);
      ++nl;
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpy(&r1, &ctl->round, 4, cudaMemcpyDeviceToHost));
      if (r1 == r0) return 0;  // nothing planned: the sort is done
      LevelArgs A;
      CK(cudaMemcpy(&A, &ctl->A, sizeof A, cudaMemcpyDeviceToHost));
      for (int s = 0; s < ST_N; ++s)
        if ((A.stages >> s) & 1u) {
          host_stage<ALGO>(A, s, st);
          ++nl;
        }
    }
  }

  template <int ALGO> static void host_stage(const LevelArgs &A, int s, cudaStream_t st) {
    using Tr = Traits<DT>;
    SortCtl *ctl = reinterpret_cast<SortCtl *>(A.ctl);
    switch (s) {
      case ST_SAMPLE:
        sample_kernel<DT, ALGO><<<A.ntasks, SAMPLE_THREADS,
                                  ALGO == ALGO_TREE ? sample_smem<DT>((size_t)A.sample_p) : 0, st>>>(A);
        break;
      case ST_CLASSIFY:
        if constexpr (Tr::D > 16) classify_kernel<DT, ALGO><<<A.nstripes, Tr::CLS_THREADS, ClsSmem<DT>::bytes, st>>>(A);
        else classify_v2_kernel<DT, ALGO><<<A.nstripes, ClsV2<DT>::NT, ClsV2<DT>::bytes, st>>>(A);
        break;
      case ST_BOUND: boundaries_kernel<DT, ALGO><<<A.ntasks, BND_THREADS, 0, st>>>(A); break;
      case ST_FIX: stripe_fix_kernel<DT><<<A.nstripes, FIX_THREADS, 0, st>>>(A); break;
      case ST_PERM: permute_kernel<DT, ALGO><<<A.nperm, PERM_THREADS, 0, st>>>(A); break;
      case ST_CSAVE: cleanup_save_kernel<DT><<<A.ntasks * cleanup_groups<DT>(), CLN_WARPS * 32, 0, st>>>(A); break;
      case ST_CFILL: cleanup_fill_kernel<DT><<<A.nstripes, FILL_THREADS, 0, st>>>(A); break;
      case ST_BASE:
      case ST_SPLIT: {
        const BaseSplitArgs sp{A.bc_scratch, (u32)A.base_cap_elems, A.next_tasks, A.next_count, A.next_cap,
                               reinterpret_cast<unsigned long long *>(ctl->counters + 6), &ctl->error};
        if (s == ST_BASE)
          basecase_kernel<DT, false><<<A.bc_grid, BaseItem<DT>::THREADS, BaseSmem<DT>::bytes, st>>>(
              A.base, A.base_tasks, ctl->counters + 1, A.base_cap_tasks, sp, A.tslot);
        else if constexpr (BaseItem<DT>::SPLIT)
          basecase_kernel<DT, true><<<A.bc_grid, BaseItem<DT>::THREADS, BaseSmem<DT>::bytes, st>>>(
              A.base, A.split_tasks, ctl->counters + 8, A.base_cap_tasks, sp, A.tslot);
        break;
      }
      case ST_CSETUP: count_setup_kernel<<<1, CNT_SETUP_THREADS, 0, st>>>(A); break;
      case ST_CCOUNT:
        if constexpr (BaseItem<DT>::KEY_ONLY) count_kernel<DT><<<A.count_grid, CNT_THREADS, 0, st>>>(A);
        break;
      case ST_CWRITE:
        if constexpr (BaseItem<DT>::KEY_ONLY) count_write_kernel<DT><<<A.count_grid, CNT_THREADS, 0, st>>>(A);
        break;
      case ST_NEXT: driver_kernel<DT, ALGO><<<1, PLAN_THREADS, 0, st>>>(ctl, 2); break;
      case ST_MEAS: measure_part_kernel<DT><<<A.nmparts, MEAS_THREADS, 0, st>>>(A); break;
      case ST_MEASRED: measure_reduce_kernel<DT><<<(A.nmtasks + 127) / 128, 128, 0, st>>>(A, A.nmtasks); break;
      default: break;
    }
  }

  static int capture_step(const SortCtl &h, ips4o_step_info *info) {
    using Key = typename Traits<DT>::Key;
    constexpr int KI = Traits<DT>::KIDX;
    const int kb = DT == DT_REC100 ? 16 : DT == DT_U32 ? 4 : DT == DT_QUARTET ? 24 : 8;
    LevelTask L;
    CK(cudaMemcpy(&L, h.A.tasks, sizeof L, cudaMemcpyDeviceToHost));
    info->algo = h.cfg.algo;
    info->num_buckets = (int)L.K;
    info->l = (int)L.l;
    info->equality = (int)L.equality;
    info->shift = L.shift;
    info->k_used = (int)L.k_used;
    info->k_req = (int)L.k_req;
    info->samples = h.cfg.algo == ALGO_TREE ? (int)L.m : 0;
    info->kidx_budget = (int)L.kidx;
    info->level = 0;
    info->seed = h.cfg.seed;
    info->lut_log = (int)L.lut_log;
    std::vector<u64> E(L.K + 1);
    CK(cudaMemcpy(E.data(), h.A.E + L.bucket_off, (L.K + 1) * 8, cudaMemcpyDeviceToHost));
    if (info->E) memcpy(info->E, E.data(), (L.K + 1) * 8);
    if (h.cfg.algo == ALGO_TREE) {
      std::vector<Key> tr(2 * KI);
      CK(cudaMemcpy(tr.data(), h.A.trees, 2 * KI * sizeof(Key), cudaMemcpyDeviceToHost));
      const int leaves = 1 << L.l;
      for (int i = 0; i < leaves; ++i) {
        u64 w[KEY_WORDS];
        key_to_words<Key>(tr[i], w);
        if (info->tree) key_to_raw<DT>(w, (unsigned char *)info->tree + (size_t)i * kb);
        key_to_words<Key>(tr[KI + i], w);
        if (info->splitter) key_to_raw<DT>(w, (unsigned char *)info->splitter + (size_t)i * kb);
      }
      if (info->tree) memset(info->tree, 0, kb);  // tree[0] is a dummy
    }
    return 0;
  }
};

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
// pointer alignment the kernels need: the element's widest access unit
static int dtype_align(int dtype) {
  switch (dtype) {
    case DT_U32: return 4;
    case DT_U64:
    case DT_F64: return 8;
    default: return 16;
  }
}

// Development builds may compile one element type only (-DIPS4O_ONLY_DT=<dt>,
// a quicker build for kernel experiments; the other types then return
// IPS4O_ERR_INVALID).  Release builds compile all of them.
template <int DT>
static int run_dt(const Call &k, char *base, u64 n, cudaStream_t st, SortCtl *hctl, u64 *scratch,
                  ips4o_step_info *cap) {
#ifdef IPS4O_ONLY_DT
  if constexpr (DT != IPS4O_ONLY_DT) return IPS4O_ERR_INVALID;
  else
#endif
    return Sorter<DT>::run(k, base, n, st, hctl, scratch, cap);
}

static int dispatch(int dtype, const Call &k, char *base, u64 n, cudaStream_t st, SortCtl *hctl, u64 *scratch,
                    ips4o_step_info *cap) {
  switch (dtype) {
    case DT_U64: return run_dt<DT_U64>(k, base, n, st, hctl, scratch, cap);
    case DT_F64: return run_dt<DT_F64>(k, base, n, st, hctl, scratch, cap);
    case DT_PAIR: return run_dt<DT_PAIR>(k, base, n, st, hctl, scratch, cap);
    case DT_REC100: return run_dt<DT_REC100>(k, base, n, st, hctl, scratch, cap);
    case DT_U32: return run_dt<DT_U32>(k, base, n, st, hctl, scratch, cap);
    case DT_QUARTET: return run_dt<DT_QUARTET>(k, base, n, st, hctl, scratch, cap);
    default: return IPS4O_ERR_INVALID;
  }
}

// RAII holders for the host-buffer path
struct StreamHolder {
  cudaStream_t s = nullptr;
  ~StreamHolder() {
    if (s) cudaStreamDestroy(s);
  }
};
struct PinnedHolder {
  char *p = nullptr;
  ~PinnedHolder() {
    if (p) cudaFreeHost(p);
  }
};
struct EventHolder {
  cudaEvent_t e = nullptr;
  ~EventHolder() {
    if (e) cudaEventDestroy(e);
  }
};

}  // namespace ips4o

using namespace ips4o;

extern "C" {

int ips4o_sort_ex(void *ptr, uint64_t n, int dtype, void *stream, const ips4o_options *opt, ips4o_stats *out) {
  const int D = dtype_bytes(dtype);
  if (!D) return IPS4O_ERR_INVALID;
  if (out) memset(out, 0, sizeof *out);
  if (n <= 1) return IPS4O_OK;
  if (!ptr || ((uintptr_t)ptr % dtype_align(dtype)) || n >= (1ull << 32)) return IPS4O_ERR_INVALID;
  Call k;
  int rc = parse_options(k, opt);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!out) return dispatch(dtype, k, reinterpret_cast<char *>(ptr), n, st, nullptr, nullptr, nullptr);
  std::vector<char> hbuf(CTL_READ);
  SortCtl *h = reinterpret_cast<SortCtl *>(hbuf.data());
  u64 scratch = 0;
  rc = dispatch(dtype, k, reinterpret_cast<char *>(ptr), n, st, h, &scratch, nullptr);
  if (rc == 0 || rc == IPS4O_ERR_CUDA) fill_stats(*h, out, scratch);
  return rc;
}

int ips4o_sort(void *ptr, uint64_t n, int dtype, void *stream) {
  return ips4o_sort_ex(ptr, n, dtype, stream, nullptr, nullptr);
}

int ips4o_sort_host(void *host_ptr, uint64_t n, int dtype, const ips4o_options *opt, ips4o_stats *out) {
  const int D = dtype_bytes(dtype);
  if (!D) return IPS4O_ERR_INVALID;
  if (out) memset(out, 0, sizeof *out);
  if (n <= 1) return IPS4O_OK;
  if (!host_ptr || ((uintptr_t)host_ptr % dtype_align(dtype)) || n >= (1ull << 32)) return IPS4O_ERR_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return IPS4O_ERR_NOGPU;
  }
  const size_t bytes = (size_t)n * D;
  StreamHolder sh;
  CK(cudaStreamCreateWithFlags(&sh.s, cudaStreamNonBlocking));
  cudaStream_t st = sh.s;
  cudaPointerAttributes pa;
  const bool pinned = cudaPointerGetAttributes(&pa, host_ptr) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  char *dev = nullptr;
  if (cudaMallocAsync((void **)&dev, bytes, st) != cudaSuccess) {
    cudaGetLastError();
    return IPS4O_ERR_NOMEM;
  }
  struct DevFree {
    char *&p;
    cudaStream_t s;
    ~DevFree() {
      if (p) {
        cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
      }
    }
  } dfree{dev, st};
  const size_t CH = 64ull << 20;
  PinnedHolder stage[2];
  EventHolder done[2];
  if (!pinned) {
    CK(cudaMallocHost(&stage[0].p, CH));
    CK(cudaMallocHost(&stage[1].p, CH));
    CK(cudaEventCreate(&done[0].e));
    CK(cudaEventCreate(&done[1].e));
  }
  char *h = reinterpret_cast<char *>(host_ptr);
  if (pinned) {
    CK(cudaMemcpyAsync(dev, h, bytes, cudaMemcpyHostToDevice, st));
  } else {
    int q = 0;
    for (size_t off = 0; off < bytes; off += CH, q ^= 1) {
      size_t len = std::min(CH, bytes - off);
      if (off >= 2 * CH) CK(cudaEventSynchronize(done[q].e));
      memcpy(stage[q].p, h + off, len);
      CK(cudaMemcpyAsync(dev + off, stage[q].p, len, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(done[q].e, st));
    }
  }
  int rc = ips4o_sort_ex(dev, n, dtype, st, opt, out);
  if (rc) return rc;
  if (pinned) {
    CK(cudaMemcpyAsync(h, dev, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  } else {
    for (size_t off = 0; off < bytes; off += CH) {
      size_t len = std::min(CH, bytes - off);
      CK(cudaMemcpyAsync(stage[0].p, dev + off, len, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      memcpy(h + off, stage[0].p, len);
    }
  }
  return 0;
}

uint64_t ips4o_scratch_bytes(uint64_t n, int dtype, const ips4o_options *opt) {
  // Exactly what ips4o_sort_ex allocates for (n, dtype, opt): control block,
  // two pending task lists of n / (M + 1) + 2 tasks, and the level arena.
  if (!dtype_bytes(dtype) || n <= 1) return 0;
  Call k;
  if (parse_options(k, opt)) return 0;
  DevState tmp;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&tmp.sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  if (tmp.sms <= 0) tmp.sms = 148;
  for (int d = 0; d < NDT; ++d) tmp.perm_occ[d] = (dev >= 0 && dev < MAX_DEVICES && g_dev[dev].perm_occ[d]) ? g_dev[dev].perm_occ[d] : 8;
  SortCfg c;
  switch (dtype) {
    case DT_U64: c = make_cfg<DT_U64>(k, tmp, nullptr, n); break;
    case DT_F64: c = make_cfg<DT_F64>(k, tmp, nullptr, n); break;
    case DT_PAIR: c = make_cfg<DT_PAIR>(k, tmp, nullptr, n); break;
    case DT_REC100: c = make_cfg<DT_REC100>(k, tmp, nullptr, n); break;
    case DT_U32: c = make_cfg<DT_U32>(k, tmp, nullptr, n); break;
    default: c = make_cfg<DT_QUARTET>(k, tmp, nullptr, n); break;
  }
  return scratch_for(dtype, c, k.arena_bytes);
}

int ips4o_device_status(int device, uint32_t *flags, int clear) {
  if (!flags || device < 0 || device >= MAX_DEVICES) return IPS4O_ERR_INVALID;
  *flags = 0;
  DevState &ds = g_dev[device];
  if (!ds.status) return IPS4O_OK;  // no sort ran on this device
  int prev = 0;
  CK(cudaGetDevice(&prev));
  CK(cudaSetDevice(device));
  cudaError_t e = cudaMemcpy(flags, ds.status, 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && clear) e = cudaMemset(ds.status, 0, 4);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return set_cuda_err(e, "ips4o_device_status", __LINE__);
  return IPS4O_OK;
}

int ips4o_release_memory(int device) {
  if (device < 0 || device >= MAX_DEVICES) return IPS4O_ERR_INVALID;
  DevState &ds = g_dev[device];
  if (!ds.pool) return IPS4O_OK;
  CK(cudaMemPoolTrimTo(ds.pool, 0));
  return IPS4O_OK;
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
  if (n < 2 || !ptr || ((uintptr_t)ptr % dtype_align(dtype)) || n >= (1ull << 32)) return IPS4O_ERR_INVALID;
  Call k;
  int rc = parse_options(k, opt);
  if (rc) return rc;
  k.capture = true;
  std::vector<char> hbuf(CTL_READ);
  return dispatch(dtype, k, reinterpret_cast<char *>(ptr), n, reinterpret_cast<cudaStream_t>(stream),
                  reinterpret_cast<SortCtl *>(hbuf.data()), nullptr, info);
}

// ---------------------------------------------------------------- distributed samplesort
int ips4o_sample(const void *ptr, uint64_t n, int dtype, void *stream, uint64_t m, uint64_t seed, void *out) {
  const int D = dtype_bytes(dtype);
  if (!D) return IPS4O_ERR_INVALID;
  if (m == 0) return IPS4O_OK;
  if (n == 0 || !ptr || !out || ((uintptr_t)ptr % 4) || ((uintptr_t)out % 4) || m >= (1ull << 40))
    return IPS4O_ERR_INVALID;
  DevState *ds = nullptr;
  int rc = device_state(ds);
  if (rc) return rc;
  const u64 words = m * (u64)(D / 4);
  const u64 grid = std::min<u64>((words + 255) / 256, (u64)ds->sms * 8);
  gather_sample_kernel<<<(unsigned)grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const char *>(ptr), n, seed, m, D, reinterpret_cast<char *>(out));
  CK(cudaGetLastError());
  return IPS4O_OK;
}

int ips4o_select_splitters(void *samples, uint64_t total, int dtype, void *stream, int parts, void *out) {
  const int D = dtype_bytes(dtype);
  if (!D || parts < 1) return IPS4O_ERR_INVALID;
  if (parts == 1) return IPS4O_OK;
  if (!samples || !out || total < (uint64_t)parts || ((uintptr_t)out % 4)) return IPS4O_ERR_INVALID;
  int rc = ips4o_sort(samples, total, dtype, stream);
  if (rc) return rc;
  const int words = (parts - 1) * (D / 4);
  pick_kernel<<<(words + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const char *>(samples), total, parts, D, reinterpret_cast<char *>(out));
  CK(cudaGetLastError());
  return IPS4O_OK;
}

}  // extern "C"

namespace ips4o {
// order of the keys of two elements (host; the dtype's comparator, Alg. 3/4)
template <int DT> static int cmp_elem_keys(const unsigned char *a, const unsigned char *b) {
  u64 x[KEY_WORDS] = {0}, y[KEY_WORDS] = {0};
  raw_to_key<DT>(a, x);
  raw_to_key<DT>(b, y);
  for (int i = KEY_WORDS - 1; i >= 0; --i)
    if (x[i] != y[i]) return x[i] < y[i] ? -1 : 1;
  return 0;
}

template <int DT>
static int partition_splitters_impl(char *ptr, u64 n, cudaStream_t st, const char *splitters, int nspl,
                                    uint64_t *bounds) {
  constexpr int D = Traits<DT>::D, KI = Traits<DT>::KIDX;
  if (nspl > KI / 2 - 1) return IPS4O_ERR_INVALID;
  std::vector<unsigned char> hs((size_t)nspl * D), he(D);
  CK(cudaMemcpyAsync(hs.data(), splitters, hs.size(), cudaMemcpyDeviceToHost, st));
  if (n == 1) CK(cudaMemcpyAsync(he.data(), ptr, D, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  auto S = [&](int r) { return hs.data() + (size_t)r * D; };
  for (int r = 1; r < nspl; ++r)
    if (cmp_elem_keys<DT>(S(r - 1), S(r)) > 0) return IPS4O_ERR_INVALID;  // not sorted
  bounds[0] = 0;
  bounds[nspl + 1] = n;
  if (n < 2) {  // nothing to partition: count the element (if any) per range
    for (int r = 0; r < nspl; ++r) bounds[r + 1] = (n == 1 && cmp_elem_keys<DT>(he.data(), S(r)) <= 0) ? 1 : 0;
    return IPS4O_OK;
  }
  Call k;
  k.capture = true;
  k.ext_spl = splitters;
  k.ext_n = nspl;
  std::vector<char> hbuf(CTL_READ);
  std::vector<uint64_t> E(KI + 1);
  std::vector<unsigned char> tr((size_t)KI * 24), sp((size_t)KI * 24);
  ips4o_step_info info;
  memset(&info, 0, sizeof info);
  info.E = E.data();
  info.tree = tr.data();
  info.splitter = sp.data();
  int rc = Sorter<DT>::run(k, ptr, n, st, reinterpret_cast<SortCtl *>(hbuf.data()), nullptr, &info);
  if (rc) return rc;
  // range r = (S_{r-1}, S_r]: the elements <= S_r are the buckets up to the
  // one of S_r's unique index u (u + 1 buckets, or 2u + 2 with equality
  // buckets: (s_{u-1}, s_u) and {s_u} per unique splitter)
  int u = -1;
  for (int r = 0; r < nspl; ++r) {
    if (r == 0 || cmp_elem_keys<DT>(S(r - 1), S(r)) != 0) ++u;
    const int nb = info.equality ? 2 * u + 2 : u + 1;
    if (nb > info.num_buckets) {
      g_err = "partition_splitters: bucket layout does not match the splitters";
      return IPS4O_ERR_CUDA;
    }
    bounds[r + 1] = E[nb];
  }
  return IPS4O_OK;
}
}  // namespace ips4o

extern "C" {
int ips4o_partition_splitters(void *ptr, uint64_t n, int dtype, void *stream, const void *splitters, int nspl,
                              uint64_t *bounds) {
  const int D = dtype_bytes(dtype);
  if (!D || !bounds || nspl < 1 || !splitters || ((uintptr_t)splitters % 4)) return IPS4O_ERR_INVALID;
  if (n > 0 && (!ptr || ((uintptr_t)ptr % dtype_align(dtype)) || n >= (1ull << 32))) return IPS4O_ERR_INVALID;
  char *p = reinterpret_cast<char *>(ptr);
  const char *s = reinterpret_cast<const char *>(splitters);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (dtype) {
#ifdef IPS4O_ONLY_DT
#define PS(DTc) return DTc == IPS4O_ONLY_DT ? partition_splitters_impl<DTc == IPS4O_ONLY_DT ? DTc : IPS4O_ONLY_DT>(p, n, st, s, nspl, bounds) : IPS4O_ERR_INVALID;
#else
#define PS(DTc) return partition_splitters_impl<DTc>(p, n, st, s, nspl, bounds);
#endif
    case DT_U64: PS(DT_U64)
    case DT_F64: PS(DT_F64)
    case DT_PAIR: PS(DT_PAIR)
    case DT_REC100: PS(DT_REC100)
    case DT_U32: PS(DT_U32)
    case DT_QUARTET: PS(DT_QUARTET)
#undef PS
    default: return IPS4O_ERR_INVALID;
  }
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
  struct Free {
    Key *p;
    ~Free() { cudaFree(p); }
  } guard{dt};
  CK(cudaMemcpy(dt, tree.data(), leaves * sizeof(Key), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dt + leaves, spl.data(), leaves * sizeof(Key), cudaMemcpyHostToDevice));
  if (n) {
    unsigned g = (unsigned)std::min<u64>(cdiv(n, 256), 148 * 8);
    classify_test_kernel<DT><<<g, 256, 0, st>>>(reinterpret_cast<const char *>(elems), n, dt, dt + leaves, l, eq, out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_err(e, "classify_test_kernel", __LINE__);
  }
  CK(cudaStreamSynchronize(st));
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
