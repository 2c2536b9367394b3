// k_basecase.cuh -- K7: the base case, "small buckets are finished inside one
// CTA in shared memory" (north star; P:980-982, P:1652 use insertion sort on
// CPUs).  One CTA per bucket of at most M elements:
//   1. histogram of a digit of (key - lo) scaled to the bucket's key bounds
//      [lo,hi] (bounds come from the splitters, so the digit cuts the bucket
//      into ~m nearly equal runs of ~1 element; 16-bit counters),
//   2. exclusive scan and scatter into shared memory (the second read of the
//      bucket hits L2),
//   3. runs longer than RW + 1 are sorted in place by a warp (warp_sort_run),
//   4. every element computes its rank inside its short run (<= RW + 1, a fixed
//      window of neighbours) by counting the
//      smaller elements -- the parallel form of the paper's insertion-sort
//      base case -- and is written straight to its final global position.
#pragma once
#include "common.cuh"

namespace ips4o {

template <int DT> struct BaseItem;

#ifndef IPS4O_BC_THREADS
#define IPS4O_BC_THREADS 1024
#endif
template <> struct BaseItem<DT_U64> {
  using Item = u64;
  using Key = u64;
  static constexpr int THREADS = IPS4O_BC_THREADS, DBMAX = 14, CAP = Traits<DT_U64>::BASE_CAP;
  static constexpr bool SPLIT = true;   // buckets of up to 2 CAP: two shared-memory passes
  static constexpr bool STAGE_RECORDS = false, KEY_ONLY = true;
  __device__ static Item load(const char *e, u32) { return *reinterpret_cast<const u64 *>(e); }
  __device__ static Key key(const Item &it) { return it; }
  __device__ static bool less(const Item &a, const Item &b) { return a < b; }
};
template <> struct BaseItem<DT_F64> {
  using Item = u64;  // order-preserving key
  using Key = u64;
  static constexpr int THREADS = 1024, DBMAX = 14, CAP = Traits<DT_F64>::BASE_CAP;
  static constexpr bool SPLIT = true;   // buckets of up to 2 CAP: two shared-memory passes
  static constexpr bool STAGE_RECORDS = false, KEY_ONLY = true;
  __device__ static Item load(const char *e, u32) { return f64_to_key(*reinterpret_cast<const u64 *>(e)); }
  __device__ static Key key(const Item &it) { return it; }
  __device__ static bool less(const Item &a, const Item &b) { return a < b; }
};
template <> struct BaseItem<DT_U32> {
  using Item = u32;
  using Key = u64;
  static constexpr int THREADS = 1024, DBMAX = 15, CAP = Traits<DT_U32>::BASE_CAP;
  static constexpr bool SPLIT = true;   // buckets of up to 2 CAP: two shared-memory passes
  static constexpr bool STAGE_RECORDS = false, KEY_ONLY = true;
  __device__ static Item load(const char *e, u32) { return *reinterpret_cast<const u32 *>(e); }
  __device__ static Key key(const Item &it) { return it; }
  __device__ static bool less(const Item &a, const Item &b) { return a < b; }
};
struct alignas(16) QuartetItem {
  u64 a, b, c, v;
};
template <> struct BaseItem<DT_QUARTET> {
  using Item = QuartetItem;
  using Key = K192;
  static constexpr int THREADS = 512, DBMAX = 13, CAP = Traits<DT_QUARTET>::BASE_CAP;
  static constexpr bool SPLIT = true;   // buckets of up to 2 CAP: two shared-memory passes
  static constexpr bool STAGE_RECORDS = false, KEY_ONLY = false;
  __device__ static Item load(const char *e, u32) { return *reinterpret_cast<const QuartetItem *>(e); }
  __device__ static Key key(const Item &it) { return K192(it.c, it.b, it.a); }
  __device__ static bool less(const Item &x, const Item &y) { return key(x) < key(y); }
};
struct alignas(16) PairItem {
  u64 key, val;
};
template <> struct BaseItem<DT_PAIR> {
  using Item = PairItem;
  using Key = u64;
  static constexpr int THREADS = 512, DBMAX = 14, CAP = Traits<DT_PAIR>::BASE_CAP;
  static constexpr bool SPLIT = true;   // buckets of up to 2 CAP: two shared-memory passes
  static constexpr bool STAGE_RECORDS = false, KEY_ONLY = false;
  __device__ static Item load(const char *e, u32) { return *reinterpret_cast<const PairItem *>(e); }
  __device__ static Key key(const Item &it) { return it.key; }
  __device__ static bool less(const Item &a, const Item &b) { return a.key < b.key; }
};
template <> struct BaseItem<DT_REC100> {
  using Item = u128;  // key80 << 16 | index of the record in the staging area
  using Key = u128;
  static constexpr int THREADS = 512, DBMAX = 11, CAP = Traits<DT_REC100>::BASE_CAP;
  static constexpr bool SPLIT = false;
  static constexpr bool STAGE_RECORDS = true, KEY_ONLY = false;
  __device__ static Item load(const char *e, u32 idx) { return (Traits<DT_REC100>::key(e) << 16) | (u128)idx; }
  __device__ static Key key(const Item &it) { return it >> 16; }
  __device__ static bool less(const Item &a, const Item &b) { return a < b; }
};

// Widest key range (hi - lo) a key-only bucket can be counted exactly with
// (one 16-bit counter per key value over the whole shared-memory area; see
// digit_par in basecase_kernel); K6 sends such buckets of up to 65535
// elements to the base case whatever their size.
template <int DT> struct BaseSmem;
template <int DT> constexpr unsigned long long basecase_count_range() {
  return BaseItem<DT>::KEY_ONLY ? (unsigned long long)(BaseSmem<DT>::off_hist + ((size_t)1 << BaseItem<DT>::DBMAX) * 2) / 2 - 16
                                : 0ull;
}

constexpr int RW = 3;        // rank window: runs of up to RW + 1 elements are ranked in registers
constexpr int RANKMAX = 32;  // runs this long count towards the whole-bucket fallback
constexpr int BIGCAP = 512;  // runs longer than RW + 1 listed per bucket (more: digit scan fallback)

template <int DT> struct BaseSmem {
  using BI = BaseItem<DT>;
  static constexpr size_t off_items = 0;
  // (+2 items: the u64 bulk copy-out shifts the bucket by one item so that
  // shared and global addresses agree modulo 16 bytes)
  static constexpr size_t off_rec = off_items + (((size_t)BI::CAP + 2) * sizeof(typename BI::Item) + 15) / 16 * 16;
  static constexpr size_t off_sidx =
      off_rec + (BI::STAGE_RECORDS ? ((size_t)BI::CAP * Traits<DT>::D + 15) / 16 * 16 : 0);
  static constexpr size_t off_hist = off_sidx + (BI::STAGE_RECORDS ? ((size_t)BI::CAP * 2 + 15) / 16 * 16 : 0);
  static constexpr size_t off_big = off_hist + ((size_t)1 << BI::DBMAX) * 2;  // 16-bit counters, two per word
  static constexpr size_t bytes = off_big + (size_t)BIGCAP * 4 + (BI::THREADS / 32 + 4) * 4;
  static_assert(bytes <= 232448, "227 KB of dynamic shared memory per CTA");
};

// Warp bitonic sort of a[0..n) in shared memory.  All comparators point the
// same way (the "flip" form), so the virtual +inf padding to the next power of
// two never moves and comparators that touch it are skipped.
template <class BI>
__device__ void warp_bitonic_run(typename BI::Item *a, int n, int lane) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int q = lane; q < P / 2; q += 32) {
        int i, p;
        int blk = q / j, off = q % j;
        if (j == (k >> 1)) {  // flip step
          i = blk * k + off;
          p = blk * k + (k - 1 - off);
        } else {
          i = blk * 2 * j + off;
          p = i + j;
        }
        if (p < n) {
          typename BI::Item x = a[i], y = a[p];
          if (BI::less(y, x)) {
            a[i] = y;
            a[p] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

// A run longer than the rank window (SIMD warp per run): nothing to do if all
// its keys are equal (any order of equal keys is a sorted result); up to 32
// elements are ranked by counting, one per lane; longer runs of key-only
// items with at most 8 distinct keys are rewritten by counting the keys
// (duplicate-heavy inputs: TwoDup, EightDup); otherwise a bitonic sort.
template <class BI>
__device__ void warp_sort_run(typename BI::Item *a, int n, int lane) {
  using Item = typename BI::Item;
  using Key = typename BI::Key;
  if (n <= 32) {
    // one element per lane, ranked by counting (ties by position); nothing
    // to do if all keys are equal
    const Item x = a[lane < n ? lane : 0];
    if (__all_sync(0xffffffffu, BI::key(x) == BI::key(a[0]))) return;
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const Item y = a[j];
      r += (BI::less(y, x) || (!BI::less(x, y) && j < lane)) ? 1 : 0;
    }
    __syncwarp();
    if (lane < n) a[r] = x;
    __syncwarp();
    return;
  }
  const Key k0 = BI::key(a[0]);
  bool diff = false;
  for (int i = lane; i < n; i += 32) diff |= BI::key(a[i]) != k0;
  if (!__any_sync(0xffffffffu, diff)) return;
  if constexpr (BI::KEY_ONLY) {
    constexpr int MAXV = 8;
    Key val = 0;  // lane r < MAXV holds distinct key r and its count
    int cnt = 0, nv = 0;
    Key prev = 0;
    bool done = false;
    for (int r = 0; r <= MAXV && !done; ++r) {
      Key mn = key_max<Key>();
      bool any = false;
      for (int i = lane; i < n; i += 32) {
        const Key k = BI::key(a[i]);
        if ((r == 0 || k > prev) && k <= mn) {
          mn = k;
          any = true;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const Key y = __shfl_xor_sync(0xffffffffu, mn, o);
        mn = y < mn ? y : mn;
      }
      if (!__any_sync(0xffffffffu, any)) {
        done = true;
        break;
      }
      if (r == MAXV) break;  // more than MAXV distinct keys
      int c = 0;
      for (int i = lane; i < n; i += 32) c += BI::key(a[i]) == mn ? 1 : 0;
      c = __reduce_add_sync(0xffffffffu, c);
      if (lane == r) {
        val = mn;
        cnt = c;
      }
      prev = mn;
      nv = r + 1;
    }
    if (done) {
      int off = 0;
      for (int r = 0; r < nv; ++r) {
        const Key v = __shfl_sync(0xffffffffu, val, r);
        const int c = __shfl_sync(0xffffffffu, cnt, r);
        for (int i = lane; i < c; i += 32) a[off + i] = (Item)v;
        off += c;
      }
      __syncwarp();
      return;
    }
  }
  warp_bitonic_run<BI>(a, n, lane);
}

// Whole-bucket fallback: when the digit leaves more than a quarter of the
// bucket in long runs (keys clustered far below the digit's resolution), the
// CTA sorts all m items with one bitonic network (flip form, comparators that
// touch the virtual padding up to the next power of two are skipped).
template <class BI, int NT>
__device__ void block_bitonic(typename BI::Item *a, int n) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int q = threadIdx.x; q < P / 2; q += NT) {
        int i, p;
        const int blk = q / j, off = q % j;
        if (j == (k >> 1)) {
          i = blk * k + off;
          p = blk * k + (k - 1 - off);
        } else {
          i = blk * 2 * j + off;
          p = i + j;
        }
        if (p < n) {
          const typename BI::Item x = a[i], y = a[p];
          if (BI::less(y, x)) {
            a[i] = y;
            a[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Buckets of cap < m <= 2 cap (cap = the base-case capacity in use): split at
// the largest digit boundary whose start is <= cap; the CTA stages part B in
// its own global scratch (cap items) while part A is scattered, then sorts
// part A and part B one after the other.  A bucket that cannot be split
// that way (one digit run too long) is handed back to the next level.
struct BaseSplitArgs {
  char *scratch;        // [gridDim.x][cap] items
  u32 cap;              // base-case capacity in use (<= BaseItem::CAP)
  TaskDesc *next_tasks; // next-level task list (K6's output)
  u32 *next_count;      // its counter (K6 appended first)
  u32 next_cap;
  unsigned long long *base_elems;  // base-case element statistic (K6 counted the bucket)
  u32 *err;             // error flags (ERR_LIST_OVERFLOW)
};

#ifdef IPS4O_PHASE_TIMING
#define BC_PHASE(k)                                 \
  if (tid == 0) {                                   \
    long long now_ = clock64();                     \
    ph_[k] += now_ - tprev_;                        \
    tprev_ = now_;                                  \
  }
#else
#define BC_PHASE(k)
#endif

template <int DT, bool SPLITK>
__global__ void __launch_bounds__(BaseItem<DT>::THREADS, 1)
    basecase_kernel(char *base, const TaskDesc *tasks, const u32 *count_ptr, u32 count_cap, BaseSplitArgs sp,
                    unsigned long long *tslot) {
  using Tr = Traits<DT>;
  using BI = BaseItem<DT>;
  using Item = typename BI::Item;
  using Key = typename BI::Key;
  using S = BaseSmem<DT>;
  constexpr int NT = BI::THREADS, D = Tr::D;
  // runs of 2..RL elements are sorted by one thread (phase 5: a network over
  // the run list), longer ones by a warp.  (RL = 8 with a 19-comparator
  // network for 8-byte items measured slower: 26.4 -> 27.0 ms at 2^30, the
  // 8-item registers spill and every warp pays the longer network)
#ifndef IPS4O_BC_RL
#define IPS4O_BC_RL 4
#endif
  constexpr int RL = (SPLITK || sizeof(typename BI::Item) > 8) ? RW + 1 : IPS4O_BC_RL;
  // the run-list phase 5 (measured faster than the rank window for 8-byte
  // keys: 2^30 u64 base case 9.0 -> 8.6 ms; slower for pairs, u32 and
  // quartets, which keep the window)
  constexpr bool RUNLIST = !SPLITK && (DT == DT_U64 || DT == DT_F64);
  // copy-out of the sorted bucket by one bulk (TMA) store instead of a
  // thread loop; the next bucket's histogram overlaps it
#ifndef IPS4O_BC_BULK
#define IPS4O_BC_BULK 1
#endif
#ifndef IPS4O_BC_HEVEC
#define IPS4O_BC_HEVEC 1
#endif
  constexpr bool BULK = IPS4O_BC_BULK && RUNLIST && DT == DT_U64;
  bool pend = false;  // a bulk store may still read s_items (CTA-uniform)
  extern __shared__ __align__(16) char smem[];
  Item *s_items = reinterpret_cast<Item *>(smem + S::off_items);
  char *s_rec = smem + S::off_rec;
  unsigned short *s_sidx = reinterpret_cast<unsigned short *>(smem + S::off_sidx);
  u32 *s_big = reinterpret_cast<u32 *>(smem + S::off_big);
  u32 *s_ws = s_big + BIGCAP;  // scan workspace (NT/32+1)
  __shared__ u32 s_nbig, s_bigsum, s_dsplit, s_scnt;
  KTIMER(tslot, SPLITK ? KS_SPLIT : KS_BASE);
  Item *scratch = reinterpret_cast<Item *>(sp.scratch) + (size_t)blockIdx.x * sp.cap;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  u32 count = *count_ptr;
  if (count > count_cap) count = count_cap;
#ifdef IPS4O_PHASE_TIMING
  long long ph_[8] = {0}, tprev_ = clock64();
#endif

  // Task descriptors are double-buffered in shared memory: lanes of warp 0
  // load the next one (one word each) while the current bucket is sorted and
  // publish it after the histogram phase, so no iteration waits on them.
  constexpr int TDW = sizeof(TaskDesc) / 4;
  static_assert(TDW <= 32 && sizeof(TaskDesc) % 4 == 0, "one word per lane");
  __shared__ TaskDesc s_task[2];
  // The digit parameters of a bucket (see below) are computed once, by thread
  // 0, for the NEXT bucket while the current one is sorted.
  struct DigitPar {
    int ds, nd, direct, exact;
    u32 dmul, hoff;  // hoff: byte offset of the counters in shared memory
    int nwz, pad;    // nwz: counter words to clear (multiple of 4)
  };
  constexpr int HSTAT = (1 << BI::DBMAX) / 2;  // counter words of the static area
  __shared__ DigitPar s_par[2];
  auto digit_par = [&](const TaskDesc &tt, DigitPar &P) {
    const int mm = (int)tt.size;
    int lg = 1;
    while ((1 << lg) < mm && lg < BI::DBMAX) ++lg;
    const Key range = key_from_words<Key>(tt.hi) - key_from_words<Key>(tt.lo);
    const int bits = bitlen(range);
    const int ds = bits > 32 ? bits - 32 : 0;
    const u32 r32 = (u32)(range >> ds);
    bool direct = r32 < (1u << lg);
    P.hoff = (u32)S::off_hist;
    P.nwz = HSTAT;
    if constexpr (!BI::STAGE_RECORDS) {
      // A narrow key range (duplicate-heavy inputs) is counted exactly, one
      // counter per key value, when the counters fit the static area plus the
      // unused tail of the item array (the counters then start below it).
      if (!direct && ds == 0 && r32 < (1u << BI::DBMAX)) {
        direct = true;  // the static area holds the r32 + 1 counters
      } else if (!direct && ds == 0) {
        // (key-only buckets larger than the item array are then written from
        // the counts alone: no item array at all)
        const u64 used = BI::KEY_ONLY && mm > BI::CAP ? 0 : (u64)(mm < BI::CAP ? mm : BI::CAP) * sizeof(Item) + (BULK ? 16 : 0);
        const u64 hb = (((u64)r32 / 2 + 1) * 4 + 15) & ~15ull;  // bytes for r32 + 1 counters
        const u64 hend = S::off_hist + (u64)HSTAT * 4;
        if (hend >= hb && hend - hb >= S::off_items + used) {
          direct = true;
          P.hoff = (u32)(hend - hb);
          P.nwz = (int)(hb / 4);
        }
      }
    }
    P.ds = ds;
    P.nd = direct ? (int)r32 + 1 : (1 << lg);
    P.direct = direct;
    P.exact = direct && ds == 0;  // a digit holds a single key value
    // dmul = floor(2^(32+lg) / (r32 + 1)) (digits < 2^lg): one double
    // division and a correction instead of a 64-bit integer division (thread
    // 0 computes it while the CTA waits at the next barrier)
    u64 dm = 1;
    if (!direct) {
      dm = (u64)(ldexp(1.0, 32 + lg) / (double)((u64)r32 + 1));
      if (dm * ((u64)r32 + 1) > (1ull << (32 + lg))) --dm;
    }
    P.dmul = (u32)dm;
  };
  u32 tdw = 0;
  if (blockIdx.x < count) {
    if (tid < TDW) reinterpret_cast<u32 *>(&s_task[0])[tid] = reinterpret_cast<const u32 *>(&tasks[blockIdx.x])[tid];
    __syncthreads();
    if (tid == 0) digit_par(s_task[0], s_par[0]);
    prefetch_l2(base + s_task[0].begin * (u64)D, s_task[0].size * (u64)D, tid, NT);
    __syncthreads();
  }
  int cur = 0;
  for (u32 ti = blockIdx.x; ti < count; ti += gridDim.x, cur ^= 1) {
    const TaskDesc &t = s_task[cur];  // valid for the whole iteration
    const bool has_next = ti + gridDim.x < count;
    if (has_next && tid < TDW) tdw = reinterpret_cast<const u32 *>(&tasks[ti + gridDim.x])[tid];
    auto publish_next = [&]() {
      if (has_next && tid < TDW) reinterpret_cast<u32 *>(&s_task[cur ^ 1])[tid] = tdw;
    };
    const int m = (int)t.size;
    char *g = base + t.begin * (u64)D;
    if constexpr (!BI::STAGE_RECORDS) {
      if (t.flags & TF_LOOSE) {
        // bounds inherited from a loose root bound (TF_LOOSE, an edge bucket
        // of a sort whose pre-pass was skipped): measure the exact key range
        // first, one extra read of the bucket, so that the digit below
        // spreads the keys
        __shared__ Key s_mm[2][NT / 32];
        Key mn = key_max<Key>(), mx = (Key)0;
        for (int i = tid; i < m; i += NT) {
          const Key k = BI::key(BI::load(g + (size_t)i * D, (u32)i));
          mn = k < mn ? k : mn;
          mx = k > mx ? k : mx;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const Key a = shfl_xor_key(mn, o), b = shfl_xor_key(mx, o);
          mn = a < mn ? a : mn;
          mx = b > mx ? b : mx;
        }
        if (lane == 0) {
          s_mm[0][wid] = mn;
          s_mm[1][wid] = mx;
        }
        __syncthreads();
        if (tid == 0) {
          for (int w = 1; w < NT / 32; ++w) {
            mn = s_mm[0][w] < mn ? s_mm[0][w] : mn;
            mx = s_mm[1][w] > mx ? s_mm[1][w] : mx;
          }
          key_to_words<Key>(mn, s_task[cur].lo);
          key_to_words<Key>(mx, s_task[cur].hi);
          s_task[cur].flags &= ~(u32)TF_LOOSE;
          digit_par(s_task[cur], s_par[cur]);
        }
        __syncthreads();
      }
    }
    const Key lo = key_from_words<Key>(t.lo), hi = key_from_words<Key>(t.hi);
    if (m <= 1 || !(lo < hi)) {
      publish_next();
      __syncthreads();
      if (has_next && tid == 0) digit_par(s_task[cur ^ 1], s_par[cur ^ 1]);
      __syncthreads();
      continue;
    }
    // digit(x) = floor(v(x) * dmul / 2^32) with v(x) = the top 32 bits of
    // x - lo over the bucket's range: monotone in x (all the counting sort
    // needs; the runs are finished by key comparisons) and spread evenly over
    // nd digits, ~1 element per digit (nd = pow2 >= m).  Ranges narrower than
    // nd use v itself (one key per digit when ds == 0).
    const DigitPar &par = s_par[cur];
    const int ds = par.ds, nd = par.nd;
    const bool direct = par.direct != 0, exact = par.exact != 0;
    const u32 dmul = par.dmul;
    auto digit = [&](const Item &it) -> u32 {
      const u32 v = (u32)((BI::key(it) - lo) >> ds);
      return direct ? v : __umulhi(v, dmul);
    };
    const int nw = (nd + 1) >> 1;  // hist words: digit 2w in the low half, 2w+1 in the high half
    u32 *s_hist = reinterpret_cast<u32 *>(smem + par.hoff);
    const bool hbig = nw > HSTAT;  // exact counters beyond the static area
    if (BULK && pend && par.hoff < (u32)S::off_hist) {
      // the counters overlap the item array that the last bulk store reads
      if (tid == 0) bulk_wait_read();
      pend = false;
      __syncthreads();
    }
    // items of this bucket: s_it[i] <-> g[i], equal addresses modulo 16 B (BULK)
    Item *const s_it = s_items + (BULK ? (int)((reinterpret_cast<uintptr_t>(g) >> 3) & 1) : 0);
    BC_PHASE(7)
    for (int w = tid; w < par.nwz / 4; w += NT) reinterpret_cast<uint4 *>(s_hist)[w] = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
      s_nbig = 0;
      s_bigsum = 0;
      s_dsplit = 0;
      s_scnt = 0;
    }
    if constexpr (BI::STAGE_RECORDS) {
      // stage the records (coalesced u32 copy)
      const u32 *src = reinterpret_cast<const u32 *>(g);
      u32 *dst = reinterpret_cast<u32 *>(s_rec);
      for (int w = tid; w < m * (D / 4); w += NT) dst[w] = src[w];
    }
    __syncthreads();
    BC_PHASE(0)
    // 1. histogram of 16-bit counters (BU independent loads in flight)
#ifndef IPS4O_BC_BU
#define IPS4O_BC_BU 4
#endif
    constexpr int BU = IPS4O_BC_BU;
    auto load_batch = [&](Item (&it)[BU], int i0) {
#pragma unroll
      for (int u = 0; u < BU; ++u) {
        const int i = i0 + u * NT;
        if (i < m) it[u] = BI::load(BI::STAGE_RECORDS ? s_rec + (size_t)i * D : g + (size_t)i * D, (u32)i);
      }
    };
#ifndef IPS4O_BC_PIPE
#define IPS4O_BC_PIPE 0  // (measured: 26.2 -> 27.0 ms with 4, 26.7 with 2 per batch: spills)
#endif
#if IPS4O_BC_PIPE
    // software-pipelined: the next batch's loads (from L2) are in flight
    // while this batch's digits are counted
    {
      Item cur[BU];
      load_batch(cur, tid);
      for (int i0 = tid; i0 < m; i0 += NT * BU) {
        Item nxt[BU];
        if (i0 + NT * BU < m) load_batch(nxt, i0 + NT * BU);
#pragma unroll
        for (int u = 0; u < BU; ++u) {
          if (i0 + u * NT < m) {
            const u32 d = digit(cur[u]);
            atomicAdd(&s_hist[d >> 1], 1u << ((d & 1) << 4));
          }
        }
#pragma unroll
        for (int u = 0; u < BU; ++u) cur[u] = nxt[u];
      }
    }
#else
    for (int i0 = tid; i0 < m; i0 += NT * BU) {
      Item it[BU];
      load_batch(it, i0);
#pragma unroll
      for (int u = 0; u < BU; ++u) {
        if (i0 + u * NT < m) {
          const u32 d = digit(it[u]);
          atomicAdd(&s_hist[d >> 1], 1u << ((d & 1) << 4));
        }
      }
    }
#endif
    publish_next();
    if (BULK && pend) {  // the scatter below overwrites the items
      if (tid == 0) bulk_wait_read();
      pend = false;
    }
    __syncthreads();
    BC_PHASE(1)
    if (has_next && tid == 0) digit_par(s_task[cur ^ 1], s_par[cur ^ 1]);  // visible after the scan
    // the next bucket of this CTA streams into L2 while this one is sorted
    if (has_next) prefetch_l2(base + s_task[cur ^ 1].begin * (u64)D, s_task[cur ^ 1].size * (u64)D, tid, NT);
    // 2. exclusive scan in place: thread t owns the WPT consecutive words
    //    [t*WPT, (t+1)*WPT) (vector loads), one block-wide scan of the thread
    //    totals.  Each word becomes (start(2w), start(2w+1)).
    u32 run_off = 0, nruns = 0;  // short runs (2..RW+1 elements): this thread's list offset, total
    if (hbig) {
      // exact counters (no long runs): warp wi scans the word segment
      // [wi*seg, (wi+1)*seg) row by row (lane l reads word row + l: no bank
      // conflicts), after a block scan of the warp totals
      const int seg = ((nw + NT / 32 - 1) / (NT / 32) + 31) & ~31;
      const int s0 = min(wid * seg, nw), s1 = min(s0 + seg, nw);
      u32 wtot = 0;
      for (int w = s0 + lane; w < s1; w += 32) wtot += (s_hist[w] & 0xFFFFu) + (s_hist[w] >> 16);
      wtot = __reduce_add_sync(0xffffffffu, wtot);
      u32 all;
      u32 carry = __shfl_sync(0xffffffffu, block_exclusive_scan_1b<NT>(lane == 0 ? wtot : 0u, s_ws, &all), 0);
      for (int row = s0; row < s1; row += 32) {
        const int w = row + lane;
        const u32 h = w < s1 ? s_hist[w] : 0u, c0 = h & 0xFFFFu, t = c0 + (h >> 16);
        u32 x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u32 y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        const u32 st = carry + x - t;
        if (w < s1) s_hist[w] = st | ((st + c0) << 16);
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
    } else {
      constexpr int WPT = ((1 << BI::DBMAX) / 2 + NT - 1) / NT;
      u32 h[WPT];
      if constexpr (WPT % 4 == 0) {
#pragma unroll
        for (int q = 0; q < WPT / 4; ++q) {
          const uint4 v4 = reinterpret_cast<const uint4 *>(s_hist)[tid * (WPT / 4) + q];
          h[4 * q] = v4.x;
          h[4 * q + 1] = v4.y;
          h[4 * q + 2] = v4.z;
          h[4 * q + 3] = v4.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < WPT; ++q) h[q] = s_hist[tid * WPT + q];
      }
      u32 tot = 0, nr = 0;
      auto short_run = [](u32 c) -> u32 { return (c >= 2u && c <= (u32)RL) ? 1u : 0u; };
#pragma unroll
      for (int q = 0; q < WPT; ++q) {
        tot += (h[q] & 0xFFFFu) + (h[q] >> 16);
        if constexpr (RUNLIST) nr += short_run(h[q] & 0xFFFFu) + short_run(h[q] >> 16);
      }
      // one scan for both: elements (low half; <= CAP < 2^16) and short runs
      // (high half; <= 2^13) -- the run list offsets of phase 5
      u32 all;
      const u32 pre = block_exclusive_scan_1b<NT>(tot | (nr << 16), s_ws, &all);  // (s_ws is next written after this bucket's barriers)
      u32 st = pre & 0xFFFFu;
      run_off = pre >> 16;
      nruns = all >> 16;
#pragma unroll
      for (int q = 0; q < WPT; ++q) {
        const u32 c0 = h[q] & 0xFFFFu, c1 = h[q] >> 16;
        const u32 w = (u32)(tid * WPT + q);
        // runs longer than RL are listed for the warp sort
        if (!exact && (c0 > (u32)RL || c1 > (u32)RL) && w < (u32)nw) {
          if (c0 > (u32)RL) {
            const u32 slot = atomicAdd(&s_nbig, 1u);
            if (slot < BIGCAP) s_big[slot] = 2u * w;
            if (c0 > RANKMAX) atomicAdd(&s_bigsum, c0);
          }
          if (c1 > (u32)RL) {
            const u32 slot = atomicAdd(&s_nbig, 1u);
            if (slot < BIGCAP) s_big[slot] = 2u * w + 1u;
            if (c1 > RANKMAX) atomicAdd(&s_bigsum, c1);
          }
        }
        h[q] = st | ((st + c0) << 16);
        st += c0 + c1;
      }
      if constexpr (WPT % 4 == 0) {
#pragma unroll
        for (int q = 0; q < WPT / 4; ++q)
          reinterpret_cast<uint4 *>(s_hist)[tid * (WPT / 4) + q] =
              make_uint4(h[4 * q], h[4 * q + 1], h[4 * q + 2], h[4 * q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < WPT; ++q) s_hist[tid * WPT + q] = h[q];
      }
    }
    __syncthreads();
    BC_PHASE(2)
    const unsigned short *s_end = reinterpret_cast<const unsigned short *>(s_hist);  // starts, ends after the scatter
    if constexpr (BI::KEY_ONLY) {
      if (exact && m > BI::CAP) {
        // One key value per digit and nothing but the key in an item: the
        // counts alone are the sorted bucket (the bucket size is then not
        // limited by the item array; buckets that fit take the scatter below).
        // Position j holds lo + d for the largest d with start_d <= j: a warp
        // takes 32 consecutive positions (coalesced stores), two lanes bound
        // the digits of its first and last position by binary search over
        // all starts, and each lane searches between those bounds.
        auto put = [&](int j, u32 d) {
          const Key v = lo + (Key)d;
          if constexpr (DT == DT_F64) {
            reinterpret_cast<u64 *>(g)[j] = key_to_f64(v);
          } else {
            reinterpret_cast<Item *>(g)[j] = (Item)v;
          }
        };
        auto last_start_le = [&](int j, u32 a, u32 b) -> u32 {  // in [a, b]
          while (a < b) {
            const u32 mid = (a + b + 1) >> 1;
            if ((int)s_end[mid] <= j) a = mid;
            else b = mid - 1;
          }
          return a;
        };
        for (int sg = wid; sg * 32 < m; sg += NT / 32) {
          const int j = sg * 32 + lane;
          u32 bd = 0;
          if (lane < 2) bd = last_start_le(lane == 0 ? sg * 32 : min(sg * 32 + 31, m - 1), 0u, (u32)nd - 1);
          const u32 da = __shfl_sync(0xffffffffu, bd, 0), db = __shfl_sync(0xffffffffu, bd, 1);
          if (j < m) put(j, last_start_le(j, da, db));
        }
        __syncthreads();
        continue;
      }
    }
    // split point of an oversized bucket (see BaseSplitArgs)
    int dsplit = nd, mA = m;
    if (SPLITK && BI::SPLIT && m > (int)sp.cap) {
      for (int d = tid; d < nd; d += NT)
        if ((u32)s_end[d] <= sp.cap) atomicMax(&s_dsplit, (u32)d);
      __syncthreads();
      dsplit = (int)s_dsplit;
      mA = (int)s_end[dsplit];
      if (m - mA > (int)sp.cap || mA == 0) {
        // no digit boundary leaves both parts within the capacity: the
        // bucket goes to the next partitioning level instead
        if (tid == 0) {
          const u32 slot = atomicAdd(sp.next_count, 1u);
          if (slot < sp.next_cap) sp.next_tasks[slot] = t;
          else atomicOr(sp.err, (u32)ERR_LIST_OVERFLOW);
          atomicAdd(sp.base_elems, (unsigned long long)(-(long long)m));
        }
        __syncthreads();
        continue;
      }
    }
    const int npass = SPLITK && dsplit < nd ? 2 : 1;
    for (int pass = 0; pass < npass; ++pass) {
      const int off = pass ? mA : 0;           // global position of s_items[0]
      const int mp = pass ? m - mA : mA;       // items of this pass
      const int dlo = pass ? dsplit : 0, dhi = pass ? nd : dsplit;
      // 3. scatter into shared memory in digit order (pass 0 reads the bucket
      //    again, from L2; items of part B go to the scratch); afterwards the
      //    counters of the pass's digits hold the run ENDS
      if (pass == 0) {
#if IPS4O_BC_PIPE
        Item it[BU];
        load_batch(it, tid);
#endif
        for (int i0 = tid; i0 < m; i0 += NT * BU) {
#if IPS4O_BC_PIPE
          Item nxt[BU];
          if (i0 + NT * BU < m) load_batch(nxt, i0 + NT * BU);
#else
          Item it[BU];
          load_batch(it, i0);
#endif
#pragma unroll
          for (int u = 0; u < BU; ++u) {
            if (i0 + u * NT < m) {
              const u32 d = digit(it[u]);
              if (!SPLITK || (int)d < dsplit) {
                const int sh = (d & 1) << 4;
                const u32 old = atomicAdd(&s_hist[d >> 1], 1u << sh);
                if (IPS4O_GUARD(((old >> sh) & 0xFFFFu) < (u32)(m < BI::CAP ? m : BI::CAP), sp.err))
                  s_it[(old >> sh) & 0xFFFFu] = it[u];
              } else {
                scratch[atomicAdd(&s_scnt, 1u)] = it[u];
              }
            }
          }
#if IPS4O_BC_PIPE
#pragma unroll
          for (int u = 0; u < BU; ++u) it[u] = nxt[u];
#endif
        }
      } else if constexpr (SPLITK) {
        for (int i = tid; i < mp; i += NT) {
          const Item it = scratch[i];
          const u32 d = digit(it);
          const int sh = (d & 1) << 4;
          const u32 old = atomicAdd(&s_hist[d >> 1], 1u << sh);
          s_it[(int)((old >> sh) & 0xFFFFu) - off] = it;
        }
      }
      __syncthreads();
      BC_PHASE(3)
      // 4. long runs: warp sort in place (warp_sort_run).  The list holds
      //    BIGCAP entries; if there are more (a skewed bucket), warps scan the
      //    digits.  Mostly long runs of records or pairs (keys clustered far
      //    below the digit's resolution): the whole pass is sorted at once.
      //    (key-only items keep the per-run path: its all-equal / few-keys
      //    cases are what long runs of duplicate-heavy inputs are made of)
      const bool whole = !BI::KEY_ONLY && !exact && s_bigsum > (u32)(m / 4);
#ifdef IPS4O_BC_DEBUG
      if (tid == 0 && blockIdx.x < 2 && ti < 4 * gridDim.x) {
        u64 lw[3], hw[3];
        key_to_words<Key>(lo, lw);
        key_to_words<Key>(hi, hw);
        printf("bc task %u m %d pass %d lo %llx:%llx:%llx hi %llx:%llx:%llx ds %d nd %d nbig %u bigsum %u whole %d\n",
               ti, m, pass, lw[2], lw[1], lw[0], hw[2], hw[1], hw[0], ds, nd, s_nbig, s_bigsum, (int)whole);
      }
#endif
      if (whole) {
        block_bitonic<BI, NT>(s_it, mp);
      } else if (!exact) {
        const int nbig = (int)s_nbig;
        if (nbig <= BIGCAP) {
          for (int q = wid; q < nbig; q += NT / 32) {
            const int d = (int)s_big[q];
            if (d < dlo || d >= dhi) continue;
            const int a = d ? (int)s_end[d - 1] : 0;
            warp_sort_run<BI>(s_it + (a - off), (int)s_end[d] - a, lane);
          }
        } else {
          for (int d = dlo + wid; d < dhi; d += NT / 32) {
            const int a = d ? (int)s_end[d - 1] : 0;
            const int n = (int)s_end[d] - a;
            if (n > RL) warp_sort_run<BI>(s_it + (a - off), n, lane);
          }
        }
        if (nbig) __syncthreads();
      }
      BC_PHASE(4)
      if constexpr (RUNLIST) {
        // 5. runs of 2..RW+1 elements, sorted from a dense list: each thread
        //    re-reads the run ends of its scan words, then (once every
        //    thread has read them) writes its short runs (start | count << 16)
        //    into the counter area at its scan offset; thread r then sorts
        //    runs r, r + NT, ... (neighbouring threads, neighbouring runs) by
        //    a 4-input network whose comparators past the run are skipped --
        //    the parallel form of the paper's insertion-sort base case
        //    (P:1652).  No thread works on a run of one element.
        constexpr int WPT = ((1 << BI::DBMAX) / 2 + NT - 1) / NT;
        static_assert(RW + 1 == 4 && (RL == 4 || RL == 8), "4- and 8-input networks");
        if (!exact && !whole && nruns > 0) {
          u32 he[WPT];
#if IPS4O_BC_HEVEC
          // (vector loads: scalar loads at a stride of WPT words are WPT-way
          // bank conflicts; the counters start at a multiple of 16 bytes)
          if constexpr (WPT % 4 == 0) {
#pragma unroll
            for (int q = 0; q < WPT / 4; ++q) {
              const uint4 v4 = reinterpret_cast<const uint4 *>(s_hist)[tid * (WPT / 4) + q];
              he[4 * q] = v4.x;
              he[4 * q + 1] = v4.y;
              he[4 * q + 2] = v4.z;
              he[4 * q + 3] = v4.w;
            }
          } else
#endif
          {
#pragma unroll
            for (int q = 0; q < WPT; ++q) he[q] = s_hist[tid * WPT + q];
          }
          // end of the digit before this thread's: the neighbour lane's last
          // word (lane 0 reads it from shared memory)
          u32 prev = __shfl_up_sync(0xffffffffu, he[WPT - 1], 1) >> 16;
          if (lane == 0) prev = tid ? (s_hist[tid * WPT - 1] >> 16) : 0u;
          __syncthreads();  // (every thread has read its run ends)
          u32 *s_runs = s_hist;
          u32 k = run_off;
#pragma unroll
          for (int q = 0; q < WPT; ++q) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const u32 b = hh ? he[q] >> 16 : he[q] & 0xFFFFu;
              const u32 c = b - prev;
              if (c >= 2u && c <= (u32)RL) s_runs[k++] = prev | (c << 16);
              prev = b;
            }
          }
          __syncthreads();
          for (u32 r = tid; r < nruns; r += NT) {
            const u32 e = s_runs[r];
            const int a = (int)(e & 0xFFFFu), c = (int)(e >> 16);
            Item v[RL];
#pragma unroll
            for (int u = 0; u < RL; ++u)
              if (u < c) v[u] = s_it[a + u];
            auto cx = [&](int i, int j) {
              if (j < c && BI::less(v[j], v[i])) {
                const Item t = v[i];
                v[i] = v[j];
                v[j] = t;
              }
            };
            if (RL == 4 || c <= 4) {
              cx(0, 1);
              cx(2, 3);
              cx(0, 2);
              cx(1, 3);
              cx(1, 2);
            } else if constexpr (RL == 8) {
              // 19-comparator 8-input network (checked on all 0-1 inputs of
              // every length <= 8 with the skipped padding comparators)
              cx(0, 2), cx(1, 3), cx(4, 6), cx(5, 7);
              cx(0, 4), cx(1, 5), cx(2, 6), cx(3, 7);
              cx(0, 1), cx(2, 3), cx(4, 5), cx(6, 7);
              cx(2, 4), cx(3, 5);
              cx(1, 4), cx(3, 6);
              cx(1, 2), cx(3, 4), cx(5, 6);
            }
#pragma unroll
            for (int u = 0; u < RL; ++u)
              if (u < c) s_it[a + u] = v[u];  // (skipping runs already in order: +0.2 ms)
          }
          __syncthreads();
        }
        // 6. the bucket is sorted in shared memory: coalesced copy out
        if constexpr (BULK) {
          // one bulk store of the 16-byte aligned middle (thread 0, after
          // every thread's async-proxy fence and a barrier); the unaligned
          // first / odd last item by single stores
          const int a0 = (int)((reinterpret_cast<uintptr_t>(g) >> 3) & 1);
          const int nb = (m - a0) & ~1;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncthreads();
          if (tid == 0 && nb > 0) bulk_store_s2g(reinterpret_cast<Item *>(g) + a0, s_it + a0, (u32)nb * (u32)sizeof(Item));
          if (tid == 32 && a0) reinterpret_cast<Item *>(g)[0] = s_it[0];
          if (tid == 64 && a0 + nb < m) reinterpret_cast<Item *>(g)[m - 1] = s_it[m - 1];
          pend = nb > 0;
        }
#pragma unroll 4
        for (int i = tid; i < (BULK ? 0 : m); i += NT) {
          const Item it = s_it[i];
          if constexpr (DT == DT_U64 || DT == DT_PAIR || DT == DT_U32 || DT == DT_QUARTET) {
            reinterpret_cast<Item *>(g)[i] = it;
          } else if constexpr (DT == DT_F64) {
            reinterpret_cast<u64 *>(g)[i] = key_to_f64(it);
          } else {
            s_sidx[i] = (unsigned short)(it & (Item)0xFFFF);
          }
        }
      } else {
        // 5. (split passes) rank inside the run by counting (independent
        //    compares, so warps keep several loads in flight), write to the
        //    final position
        for (int i = tid; i < mp; i += NT) {
          const Item it = s_it[i];
          const u32 d = digit(it);
          const int a = (d ? (int)s_end[d - 1] : 0) - off;
          const int b = (int)s_end[d] - off;
          int rank = i - a;
          if (!exact && !whole && b - a > 1 && b - a <= RW + 1) {
            // the run lies inside [i - RW, i + RW]: a fixed, branch-free window
            // (ties by position)
            rank = 0;
#pragma unroll
            for (int o = -RW; o <= RW; ++o) {
              const int j = i + o;
              if (o != 0 && j >= a && j < b) {
                const Item y = s_it[j];
                rank += (o < 0 ? !BI::less(it, y) : BI::less(y, it)) ? 1 : 0;
              }
            }
          }
          const int pos = off + a + rank;
          if constexpr (DT == DT_U64 || DT == DT_PAIR || DT == DT_U32 || DT == DT_QUARTET) {
            if (IPS4O_GUARD(pos >= 0 && pos < m, sp.err)) reinterpret_cast<Item *>(g)[pos] = it;
          } else if constexpr (DT == DT_F64) {
            reinterpret_cast<u64 *>(g)[pos] = key_to_f64(it);
          } else {
            s_sidx[pos] = (unsigned short)(it & (Item)0xFFFF);
          }
        }
      }
      if constexpr (BI::STAGE_RECORDS) {
        __syncthreads();
        // records: warp per record, lanes copy the 25 words
        u32 *out = reinterpret_cast<u32 *>(g);
        for (int i = wid; i < m; i += NT / 32) {
          const u32 *src = reinterpret_cast<const u32 *>(s_rec + (size_t)s_sidx[i] * D);
          if (lane < D / 4) out[(size_t)i * (D / 4) + lane] = src[lane];
        }
      }
      BC_PHASE(5)
      __syncthreads();
      BC_PHASE(6)
    }
  }
  if (BULK && tid == 0) bulk_wait_all();
#ifdef IPS4O_PHASE_TIMING
  if (tid == 0 && blockIdx.x == 0)
    printf("basecase CTA0 cycles: setup %lld zero %lld hist %lld scan %lld scatter %lld big %lld rank+write %lld endbar %lld\n",
           ph_[7], ph_[0], ph_[1], ph_[2], ph_[3], ph_[4], ph_[5], ph_[6]);
#endif
}

}  // namespace ips4o
