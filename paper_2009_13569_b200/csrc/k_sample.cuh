// k_sample.cuh -- K1: sampling phase + branchless splitter tree (P:719-737,
// P:399-451, Fig. 2), one CTA per task; and the IPS2Ra digit setup
// (P:1687-1696).
#pragma once
#include "common.cuh"

namespace ips4o {

constexpr int SAMPLE_THREADS = 1024;  // = SORT_THREADS
// at most 16 keys per thread of the register sort (4 for 16-byte keys)
// (records: 8192, i.e. alpha = 64 at their k = 128, so that level-2 buckets
// stay below the 1 792-record base case -- records have no split pass)
template <int DT> __host__ __device__ constexpr int sample_max() {
  return Traits<DT>::D == 100 ? 8192 : Traits<DT>::D >= 32 ? 4096 : 16384;
}
// dynamic shared memory of sample_kernel: p sample slots + 16-bit digit
// counters (sized per launch, so levels of small tasks run 2 CTAs per SM)
template <int DT> __host__ __device__ constexpr size_t sample_smem(size_t p = (size_t)sample_max<DT>()) {
  return p * sizeof(typename Traits<DT>::Key) + (sizeof(typename Traits<DT>::Key) == 8 ? 16384 : Traits<DT>::D == 100 ? 8192 : 4096) * 2;
}

__host__ __device__ __forceinline__ int next_pow2_i(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
__host__ __device__ __forceinline__ int log2_i(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}

// Ascending bitonic sort of the P = SORT_THREADS * E keys a[0..P) in shared
// memory (Batcher's network, the same comparators as a plain smem bitonic
// sort).  Thread t holds keys [t*E, (t+1)*E) in registers; compare-exchange
// stages with stride j < E run inside the thread, E <= j < 32E across lanes
// by shuffle, and only j >= 32E through shared memory (15 barrier-separated
// stages at P = 16384 instead of 105).
constexpr int SORT_THREADS = 1024;

template <class Key>
__device__ __forceinline__ Key shfl_xor_k(Key v, int m) {
  if constexpr (sizeof(Key) == sizeof(K192)) {
    return Key(__shfl_xor_sync(0xffffffffu, v.w[0], m), __shfl_xor_sync(0xffffffffu, v.w[1], m),
               __shfl_xor_sync(0xffffffffu, v.w[2], m));
  } else if constexpr (sizeof(Key) == 8) {
    return __shfl_xor_sync(0xffffffffu, v, m);
  } else {
    u64 lo = __shfl_xor_sync(0xffffffffu, (u64)v, m);
    u64 hi = __shfl_xor_sync(0xffffffffu, (u64)(v >> 64), m);
    return ((u128)hi << 64) | lo;
  }
}

template <class Key, int E>
__device__ void bitonic_sort_reg(Key *a) {
  constexpr int P = SORT_THREADS * E;
  const int t = threadIdx.x;
  Key r[E];
#pragma unroll
  for (int q = 0; q < E; ++q) r[q] = a[t * E + q];
  for (int k = 2; k <= P; k <<= 1) {
    if (k / 2 >= 32 * E) {
      // strides that cross warps: through shared memory
#pragma unroll
      for (int q = 0; q < E; ++q) a[t * E + q] = r[q];
      __syncthreads();
      for (int j = k >> 1; j >= 32 * E; j >>= 1) {
        for (int i = t; i < P; i += SORT_THREADS) {
          const int p = i ^ j;
          if (p > i) {
            Key x = a[i], y = a[p];
            if ((x > y) == ((i & k) == 0)) {
              a[i] = y;
              a[p] = x;
            }
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int q = 0; q < E; ++q) r[q] = a[t * E + q];
    }
    // strides E <= j < 32E: partner on lane ^ (j / E), same register
    for (int j = (k >> 1) < 32 * E ? (k >> 1) : 16 * E; j >= E; j >>= 1) {
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int i = t * E + q;
        const Key o = shfl_xor_k<Key>(r[q], j / E);
        const bool lower = (i & j) == 0, up = (i & k) == 0;
        const bool take_min = lower == up;
        r[q] = take_min ? (o < r[q] ? o : r[q]) : (o > r[q] ? o : r[q]);
      }
    }
    // strides j < E: inside the thread
#pragma unroll
    for (int j = E >> 1; j > 0; j >>= 1) {
      if (j >= k) continue;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        if ((q & j) == 0) {
          const int i = t * E + q;
          const bool up = (i & k) == 0;
          Key x = r[q], y = r[q | j];
          if ((x > y) == up) {
            r[q] = y;
            r[q | j] = x;
          }
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < E; ++q) a[t * E + q] = r[q];
  __syncthreads();
}

// Digit extractor setup for a task with key bounds [lo, hi] (IPS2Ra): all keys
// share the bits above bitlen(lo ^ hi); the next log2(k) bits are the digit.
template <class Key>
__device__ __forceinline__ void digit_setup(LevelTask &L) {
  Key lo = key_from_words<Key>(L.t.lo), hi = key_from_words<Key>(L.t.hi);
  int h = bitlen((Key)(lo ^ hi));
  int kb = log2_i((int)L.k_req);
  int bits = h < kb ? h : kb;
  // a measured all-equal task (K0m, lo == hi) still gets two buckets; its
  // child is then terminal
  if (bits < 1) bits = 1;
  L.l = bits;
  L.shift = h > bits ? h - bits : 0;
  L.K = 1u << bits;
  L.equality = 0;
  L.k_used = 1u << bits;
  L.lut_log = 0;
}

// Sample-adaptive digit extractor of IPS2Ra ("adapting the
// function for extracting bucket indices to various input distributions
// (which can be approximated analyzing a sample of the input)"; DESIGN R33).
// A sample of the task is counted under the plain digit and under the
// logarithmic slot mapping of the offset from the task's lower bound
// (lut_slot_of: exact below 2^(M+1), then 2^M slots per octave, M the largest
// that fits the bucket budget).  When the plain digit puts more than 1/8 of
// the sample into one bucket and the logarithmic mapping's fullest bucket
// holds less than half of that, the task is partitioned by the logarithmic
// mapping (L.lut_log = M); the children return to the plain digit of their
// own (exact) ranges.  Keys of 8 bytes; bounds must be true bounds of the keys
// (not TF_LOOSE: offsets are taken from lo).
#ifndef IPS4O_DIGIT_ADAPT
#define IPS4O_DIGIT_ADAPT 1
#endif
constexpr int DIG_SAMPLE = 2048;
template <int DT>
__device__ void digit_adapt(const LevelArgs &A, LevelTask &L) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  static_assert(sizeof(Key) == 8, "8-byte keys");
  __shared__ u32 s_h[2][256];
  __shared__ u32 s_mx[2];
  const int tid = threadIdx.x, NT = blockDim.x;
  if (tid == 0) digit_setup<Key>(L);
  __syncthreads();
  if (!IPS4O_DIGIT_ADAPT) return;
  const Key lo = key_from_words<Key>(L.t.lo), hi = key_from_words<Key>(L.t.hi);
  const u64 R = (u64)(hi - lo);
  if ((L.t.flags & TF_LOOSE) || L.t.size < 16 * (u64)DIG_SAMPLE || L.K < 16 || L.k_req > 256 || R < 4096 ||
      bitlen(R) > 62)
    return;
  int M = 0;
  for (int q = 1; q <= 7; ++q)
    if (lut_slot_of(R, 0, q) + 1 <= L.k_req) M = q;
  if (M == 0) return;
  for (int i = tid; i < 512; i += NT) (&s_h[0][0])[i] = 0;
  if (tid < 2) s_mx[tid] = 0;
  __syncthreads();
  const u32 dmask = L.K - 1;
  for (int i = tid; i < DIG_SAMPLE; i += NT) {
    Key x = Tr::key(A.base + sample_index(A.seed, L.t.level, L.t.begin, L.t.size, (u64)i) * Tr::D);
    x = x < lo ? lo : (x > hi ? hi : x);
    atomicAdd(&s_h[0][digit_of(x, L.shift, dmask)], 1u);
    atomicAdd(&s_h[1][min(lut_slot_of((u64)(x - lo), 0, M), 255u)], 1u);
  }
  __syncthreads();
  for (int i = tid; i < 256; i += NT) {
    atomicMax(&s_mx[0], s_h[0][i]);
    atomicMax(&s_mx[1], s_h[1][i]);
  }
  __syncthreads();
  if (tid == 0 && s_mx[0] * 8 > (u32)DIG_SAMPLE && s_mx[1] * 2 < s_mx[0]) {
    const u32 nlog = lut_slot_of(R, 0, M) + 1;
    u32 K = 2;
    while (K < nlog) K <<= 1;
    L.lut_log = (u32)M;
    L.K = K;
    L.l = (u32)log2_i((int)K);
    L.shift = 0;
    L.k_used = K;
  }
}

// The lookup table of starting leaves of a task, built once
// here for all classification CTAs of the task.  Padded splitters
// spl[i] = cand[min(i, u-1)], i < s = 2^l - 1; the table spans
// the sample's key range inside the task's bounds, or the bounds themselves
// when the sample covers a good part of them (every key then falls into a
// slot without clamping).
template <class Key>
__device__ void build_lut(const LevelArgs &A, LevelTask &L, int ti, const Key *cand, int u, int l,
                          const Key *samp, int m) {
  const Key tlo = key_from_words<Key>(L.t.lo), thi = key_from_words<Key>(L.t.hi);
  Key llo = key_from_words<Key>(L.lut_lo), lhi = key_from_words<Key>(L.lut_hi);
  if (llo < tlo) llo = tlo;
  if (lhi > thi) lhi = thi;
  if (lhi < llo) lhi = llo;
  const bool span = (lhi - llo) >= ((thi - tlo) >> 2);
  if (span) {
    llo = tlo;
    lhi = thi;
  }
  const int lbits = (int)L.lut_bits;
  int ls = bitlen((Key)(lhi - llo)) - lbits;
  if (ls < 0) ls = 0;
  const int nspl = (1 << l) - 1;
  const int eq = (int)L.equality;
  auto lower = [&](Key v) -> u32 {  // #{spl[i] < v, i < s}
    u32 a = 0, b = (u32)nspl;
    while (a < b) {
      const u32 mid = (a + b) >> 1;
      if (cand[(int)mid < u ? (int)mid : u - 1] < v) a = mid + 1;
      else b = mid;
    }
    return a;
  };
  // Two slot mappings (lut_slot_of): linear over [llo, lhi], or logarithmic
  // with M = lut_bits - 6 mantissa bits (fits: 2^M (65 - M) <= 2^lut_bits).
  // The table the classification uses is the one whose slots make the
  // sample's keys cheaper to classify: a sample key in a slot without a
  // splitter (or a one-key slot) costs nothing, one with c splitters
  // 1 + log2(c) comparisons (Zipf's splitters crowd the low end
  // of the range, where the linear slots hold up to 63 of them).
  const int logm = lbits >= 8 ? lbits - 6 : 0;
  const u32 nlin = (u32)((lhi - llo) >> ls) + 1;
  const u32 nlog = logm ? lut_slot_of((u64)(lhi - llo), 0, logm) + 1 : 0;
  auto slot_range = [&](u32 q, u32 n, int lm, Key &r0, Key &r1) {
    r0 = q == 0 ? tlo : llo + (Key)lut_slot_start(q, ls, lm);
    r1 = q + 1 == n ? thi : llo + (Key)lut_slot_start(q + 1, ls, lm) - 1;
  };
  auto cost = [&](Key x, u32 n, int lm) -> u32 {
    const u32 q = x < llo ? 0u : min(lut_slot_of((u64)(x - llo), ls, lm), n - 1);
    Key r0, r1;
    slot_range(q, n, lm, r0, r1);
    const u32 a = lower(r0), b = r1 == key_max<Key>() ? (u32)nspl : lower(r1 + 1);
    if (b == a || r0 == r1) return 0u;
    return b - a == 1 ? 1u : 1u + (u32)bitlen((u64)(b - a - 1));
  };
  __shared__ unsigned long long s_cost[2];
  if (threadIdx.x == 0) s_cost[0] = s_cost[1] = 0;
  __syncthreads();  // (all threads have read lut_lo / lut_hi)
  // (every 4th sample: the costs are estimates; the linear table is kept
  // without evaluating the other when it already resolves almost every key
  // without a comparison -- uniform keys)
  constexpr int CSTRIDE = 4;
  if (logm) {
    unsigned long long c0 = 0;
    for (int i = threadIdx.x * CSTRIDE; i < m; i += blockDim.x * CSTRIDE) c0 += cost(samp[i], nlin, 0);
    atomicAdd(&s_cost[0], c0);
  }
  __syncthreads();
  const bool try_log = logm && s_cost[0] * 16 * CSTRIDE > (unsigned long long)m;
  if (try_log) {
    unsigned long long c1 = 0;
    for (int i = threadIdx.x * CSTRIDE; i < m; i += blockDim.x * CSTRIDE) c1 += cost(samp[i], nlog, logm);
    atomicAdd(&s_cost[1], c1);
  }
  __syncthreads();
  const bool use_log = try_log && 5 * s_cost[1] < 4 * s_cost[0];  // (a clear gain only)
  const int lm = use_log ? logm : 0;
  const u32 nlut = use_log ? nlog : nlin;
  if (threadIdx.x == 0) {
    key_to_words<Key>(llo, L.lut_lo);
    L.lut_ls = (u32)ls;
    L.lut_n = nlut;
    L.lut_span = span ? 1u : 0u;
    L.lut_log = (u32)lm;
  }
  unsigned short *lut = A.luts + L.lut_off;
  for (u32 q = threadIdx.x; q < (1u << lbits); q += blockDim.x) {
    u32 e = 0;
    if (q < nlut) {
      Key r0, r1;
      slot_range(q, nlut, lm, r0, r1);
      // a = #{splitters < r0}; the count covers splitters in [r0, r1] (a slot
      // with none cannot hold a key equal to a splitter: key < s_a, except
      // above the last splitter -- bucket 2s+1 with equality buckets)
      const u32 a = lower(r0), b = r1 == key_max<Key>() ? (u32)nspl : lower(r1 + 1);
      if (b == a) {
        e = LUT_FIN | (eq ? 2 * a + (a == (u32)nspl ? 1u : 0u) : a);
      } else if (r0 == r1) {
        // a slot of one key value that equals splitter s_a (b > a): its bucket
        // is final too -- the equality bucket 2a+1, or a without equality
        // buckets (s_{a-1} < r0 <= s_a); duplicate-heavy inputs
        e = LUT_FIN | (eq ? 2 * a + 1 : a);
      } else {
        e = a | (min(b - a, 63u) << 9);
      }
    }
    lut[q] = (unsigned short)e;
  }
}

// Trees are stored as [tree[0..KIDX) | splitter[0..KIDX)] per task.
template <int DT, int ALGO>
__global__ void __launch_bounds__(SAMPLE_THREADS) sample_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  if (A.go && *A.go == 0) return;  // round 0 of an easy input (k_plan.cuh)
  KTIMER(A.tslot, KS_SAMPLE);
  const int ti = blockIdx.x;
  LevelTask &L = A.tasks[ti];
  if (ALGO == ALGO_DIGIT) {
    if constexpr (sizeof(Key) == 8) {
      digit_adapt<DT>(A, L);
    } else {
      if (threadIdx.x == 0) digit_setup<Key>(L);
    }
    return;
  }
  extern __shared__ __align__(16) char smem_raw[];
  Key *s_keys = reinterpret_cast<Key *>(smem_raw);
  u32 *s_hist = reinterpret_cast<u32 *>(smem_raw + (size_t)A.sample_p * sizeof(Key));
  const unsigned short *s_end = reinterpret_cast<const unsigned short *>(s_hist);
  __shared__ Key s_cand[256], s_pick[256], s_red[2][32];
  __shared__ int s_wt[256];  // picks per unique splitter (R10)
  __shared__ unsigned char s_drop[256];
  __shared__ u32 s_ws[SAMPLE_THREADS / 32 + 1];
  __shared__ int s_u, s_leaves, s_k, s_slow;
  Key *tree = reinterpret_cast<Key *>(A.trees) + (size_t)ti * 2 * Tr::KIDX;
  Key *spl = tree + Tr::KIDX;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NT = SAMPLE_THREADS;
  constexpr int MAXE = sample_max<DT>() / NT;
  constexpr int DB = sizeof(Key) == 8 ? 14 : Tr::D == 100 ? 13 : 12;  // digit bits: 2^DB >= sample_max
  static_assert((1 << DB) >= sample_max<DT>(), "one digit per sample");
  constexpr int RUNMAX = 32;                       // longer runs: full sort instead

  // ips4o_partition_splitters: the picks are the given (sorted) splitters and
  // nothing is sampled (the distributed samplesort)
  const bool ext = A.ext_n > 0;
  const int m = ext ? 0 : (int)L.m;
  const int P = next_pow2_i(m) > SORT_THREADS ? next_pow2_i(m) : SORT_THREADS;
  // P:726 "we sample k*alpha elements" (gathered, not swapped: DESIGN R9);
  // all of a thread's sample loads are issued before any is used
  Key v[MAXE];
  Key kmin = key_max<Key>(), kmax = (Key)0;
#pragma unroll
  for (int q = 0; q < MAXE; ++q) {
    const int i = tid + q * NT;
    v[q] = key_max<Key>();
    if (i < m) {
      v[q] = Tr::key(A.base + sample_index(A.seed, L.t.level, L.t.begin, L.t.size, (u64)i) * Tr::D);
      kmin = v[q] < kmin ? v[q] : kmin;
      kmax = v[q] > kmax ? v[q] : kmax;
    }
  }
  // The picks only need the sample's order statistics at k'-1 ranks: a
  // counting sort by a digit scaled to the sample's range (~1 sample per
  // digit, the same digit as the base case) puts every sample into its run,
  // and each pick ranks the few samples of its run.  Exact: the same
  // elements a full sort would put at those ranks.
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Key a = shfl_xor_k<Key>(kmin, o), b = shfl_xor_k<Key>(kmax, o);
    kmin = a < kmin ? a : kmin;
    kmax = b > kmax ? b : kmax;
  }
  if (lane == 0) {
    s_red[0][wid] = kmin;
    s_red[1][wid] = kmax;
  }
  for (int w = tid; w < (1 << DB) / 2; w += NT) s_hist[w] = 0;
  if (tid == 0) s_slow = 0;
  __syncthreads();
  kmin = s_red[0][0];
  kmax = s_red[1][0];
  for (int w = 1; w < NT / 32; ++w) {
    kmin = s_red[0][w] < kmin ? s_red[0][w] : kmin;
    kmax = s_red[1][w] > kmax ? s_red[1][w] : kmax;
  }
  if (ext) {
    kmin = Tr::key(A.ext_spl);
    kmax = Tr::key(A.ext_spl + (size_t)(A.ext_n - 1) * Tr::D);
  }
  int lg = 1;
  while ((1 << lg) < m && lg < DB) ++lg;
  const Key range = kmax - kmin;
  const int bits = bitlen(range);
  const int ds = bits > 32 ? bits - 32 : 0;
  const u32 r32 = (u32)(range >> ds);
  const bool direct = r32 < (1u << lg);
  const u32 dmul = direct ? 1u : (u32)((1ull << (32 + lg)) / ((u64)r32 + 1));
  const int nd = direct ? (int)r32 + 1 : (1 << lg);
  auto digit = [&](const Key &x) -> u32 {
    const u32 w = (u32)((x - kmin) >> ds);
    return direct ? w : __umulhi(w, dmul);
  };
#pragma unroll
  for (int q = 0; q < MAXE; ++q)
    if (tid + q * NT < m) {
      const u32 d = digit(v[q]);
      atomicAdd(&s_hist[d >> 1], 1u << ((d & 1) << 4));
    }
  __syncthreads();
  {
    constexpr int WPT = ((1 << DB) / 2 + NT - 1) / NT;
    u32 h[WPT], tot = 0;
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      h[q] = s_hist[tid * WPT + q];
      tot += (h[q] & 0xFFFFu) + (h[q] >> 16);
    }
    u32 all;
    u32 st = block_exclusive_scan<NT>(tot, s_ws, &all);
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      const u32 c0 = h[q] & 0xFFFFu, c1 = h[q] >> 16;
      s_hist[tid * WPT + q] = st | ((st + c0) << 16);
      st += c0 + c1;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < MAXE; ++q)
    if (tid + q * NT < m) {
      const u32 d = digit(v[q]);
      const int sh = (d & 1) << 4;
      const u32 old = atomicAdd(&s_hist[d >> 1], 1u << sh);
      s_keys[(old >> sh) & 0xFFFFu] = v[q];
    }
  __syncthreads();  // s_end[d] = end of run d
  // element of rank p among the samples; flags the slow path for long runs
  auto pick = [&](int p) -> Key {
    int lo = 0, hi = nd - 1;  // smallest d with end(d) > p
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int)s_end[mid] > p) hi = mid;
      else lo = mid + 1;
    }
    const int a = lo ? (int)s_end[lo - 1] : 0, b = (int)s_end[lo];
    if (b - a > RUNMAX) {
      s_slow = 1;
      return (Key)0;
    }
    for (int i = a; i < b; ++i) {
      const Key x = s_keys[i];
      int r = 0;
      for (int j = a; j < b; ++j) {
        const Key y = s_keys[j];
        r += (y < x || (y == x && j < i)) ? 1 : 0;
      }
      if (r == p - a) return x;
    }
    return (Key)0;  // not reached
  };
  const bool all_equal = !(kmin < kmax);

  if (tid == 0) {
    key_to_words<Key>(kmin, L.lut_lo);
    key_to_words<Key>(kmax, L.lut_hi);
    s_k = ext ? (int)A.ext_n + 1 : (int)L.k_req;
  }
  // P:728 equidistant picks; P:729 dedupe; P:733 equality buckets iff a
  // duplicate was removed (R23); R10: keep the most-picked equality
  // splitters that fit the index budget (halve k otherwise).
  bool sorted = false;
  for (;;) {
    __syncthreads();
    const int k = s_k;
    const int alpha = m / k;
    if (tid < k - 1) {
      const int p = (tid + 1) * alpha - 1;
      s_pick[tid] = ext ? Tr::key(A.ext_spl + (size_t)tid * Tr::D) : all_equal ? kmin : sorted ? s_keys[p] : pick(p);
    }
    __syncthreads();
    if (s_slow && !sorted) {
      // a pick fell into a long run of near-equal keys: sort all samples
      for (int i = m + tid; i < P; i += NT) s_keys[i] = key_max<Key>();
      __syncthreads();
      switch (P / SORT_THREADS) {
        case 1: bitonic_sort_reg<Key, 1>(s_keys); break;
        case 2: bitonic_sort_reg<Key, 2>(s_keys); break;
        case 4: bitonic_sort_reg<Key, 4>(s_keys); break;
        default:
          if constexpr (sizeof(Key) == 8) {
            if (P == 8 * SORT_THREADS) bitonic_sort_reg<Key, 8>(s_keys);
            else bitonic_sort_reg<Key, 16>(s_keys);
          } else if constexpr (Tr::D == 100) {
            bitonic_sort_reg<Key, 8>(s_keys);  // P <= 8192
          }
          break;
      }
      sorted = true;
      continue;  // redo the picks from the sorted samples
    }
    if (tid == 0) {
      int u = 0, dup = 0;
      for (int j = 0; j < k - 1; ++j) {
        const Key c = s_pick[j];
        if (u > 0 && s_cand[u - 1] == c) {
          dup = 1;
          ++s_wt[u - 1];
          continue;
        }
        s_wt[u] = 1;
        s_cand[u++] = c;
      }
      int leaves = next_pow2_i(u + 1);
      int need = dup ? 2 * leaves : leaves;
      const int up = (int)L.kidx / 2 - 1;
      if (dup && need > (int)L.kidx && L.kidx >= 4 && u > up) {
        // R10: u - up unique splitters too many for the bucket indices: drop
        // them one at a time, fewest picks first (ties: the smaller), never
        // two neighbours (the open bucket that absorbs a dropped splitter's
        // keys then spans at most two former buckets; RootDup's level 2 keeps
        // every bucket at one key value).  Passes over the pick counts in
        // increasing order; each pass scans the splitters in order, which is
        // the same sequence of choices.  k is unchanged; if fewer can be
        // dropped, k is halved below (the splitters stay evenly spread).
        const int want = u - up;
        int got = 0, wprev = 0;
        for (int i = 0; i < u; ++i) s_drop[i] = 0;
        while (got < want) {
          int wc = 0x7fffffff;
          for (int i = 0; i < u; ++i)
            if (!s_drop[i] && s_wt[i] > wprev && s_wt[i] < wc) wc = s_wt[i];
          if (wc == 0x7fffffff) break;
          for (int i = 0; i < u && got < want; ++i)
            if (s_wt[i] == wc && !s_drop[i] && !(i > 0 && s_drop[i - 1]) && !(i + 1 < u && s_drop[i + 1])) {
              s_drop[i] = 1;
              ++got;
            }
          wprev = wc;
        }
        if (got == want) {
          int w = 0;
          for (int i = 0; i < u; ++i)
            if (!s_drop[i]) s_cand[w++] = s_cand[i];
          u = w;
          leaves = next_pow2_i(u + 1);
          need = 2 * leaves;
        }
      }
      if (need <= (int)L.kidx || k <= 2) {
        L.K = (u32)need;
        L.l = (u32)log2_i(leaves);
        L.equality = (u32)dup;
        L.k_used = (u32)k;
        L.shift = 0;
        s_u = u;
        s_leaves = leaves;
        s_k = 0;
      } else {
        s_k = k >> 1;
      }
    }
    __syncthreads();
    if (s_k == 0) break;
  }
  __syncthreads();
  const int u = s_u, leaves = s_leaves, s = leaves - 1;
  const int l = log2_i(leaves);
  // pad with the largest splitter, splitter[s] = splitter[s-1]
  for (int i = threadIdx.x; i < leaves; i += blockDim.x) spl[i] = s_cand[i < u ? i : u - 1];
  // node i at depth d, position p holds in-order rank (2p+1)2^(l-1-d)-1
  for (int i = threadIdx.x; i < leaves; i += blockDim.x) {
    if (i == 0) {
      tree[0] = (Key)0;
      continue;
    }
    int d = 31 - __clz(i);
    int p = i - (1 << d);
    int rank = (2 * p + 1) * (1 << (l - 1 - d)) - 1;
    tree[i] = s_cand[rank < u ? rank : u - 1];
  }
  if constexpr (Tr::D <= 16) build_lut<Key>(A, L, ti, s_cand, u, l, s_keys, m);
  (void)s;
}

}  // namespace ips4o
