// k_misc.cuh -- K0 easy-input pre-pass (P:1654-1656 sorted-input detection;
// IPS2Ra's significant-bit scan P:2344-2346 as min/max of the keys), K8 the
// in-place reversal of a decreasingly sorted input, and the classifier test
// kernel behind ips4o_classify().
#pragma once
#include "common.cuh"
#include "k_classify.cuh"

namespace ips4o {

constexpr int PRE_THREADS = 512;

struct PrepassPart {
  u32 nd, ni, pad0, pad1;
  u64 mn[KEY_WORDS], mx[KEY_WORDS];
};

// Each warp scans one contiguous segment in coalesced chunks of 32*V
// elements (V consecutive elements per lane, read with 16-byte vector loads
// when the array is 16-byte aligned); the right neighbour of a lane's last
// element comes from the next lane by shuffle (one direct load per chunk for
// the element after the chunk).  Two chunks are loaded before either is
// examined, so 32-64 bytes per lane are in flight.
template <int DT> struct PreVec {
  static constexpr int D = Traits<DT>::D;
  static constexpr int V = D == 4 ? 4 : D == 8 ? 4 : D == 16 ? 2 : 1;  // elements per lane per chunk
  static constexpr int NV = (V * D) % 16 == 0 ? (V * D) / 16 : 0;    // uint4 loads per lane per chunk (0: scalar)
};

template <int DT, bool VEC>
__device__ __forceinline__ void prepass_segment(const char *base, u64 n, u64 b0, u64 b1, u32 &nd, u32 &ni,
                                                typename Traits<DT>::Key &mn, typename Traits<DT>::Key &mx) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  constexpr int D = Tr::D;
  constexpr int V = VEC ? PreVec<DT>::V : 1;
  constexpr int CH = 32 * V;
  constexpr int UN = 2;  // chunks per iteration
  const int lane = threadIdx.x & 31;
  auto visit = [&](const Key (&k)[V], u64 c, bool full) {
    // e = c + lane*V + u; neighbours inside the lane, then across lanes (the
    // shuffle is executed by all lanes, before any lane leaves the loop)
    const Key right = shfl_key(k[0], (lane + 1) & 31);
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const u64 e = c + (u64)lane * V + u;
      if (!full && e >= b1) break;
      Key nx;
      bool have = true;
      if (u + 1 < V) {
        nx = k[u + 1];
        have = full || e + 1 < b1;
        if (!have && e + 1 < n) {
          nx = Tr::key(base + (e + 1) * D);
          have = true;
        }
      } else {
        nx = right;
        have = lane < 31 && (full || e + 1 < b1);
        if (!have) {
          have = e + 1 < n;
          if (have) nx = Tr::key(base + (e + 1) * D);
        }
      }
      if (have) {
        nd &= (k[u] <= nx) ? 1u : 0u;
        ni &= (k[u] >= nx) ? 1u : 0u;
      }
      mn = k[u] < mn ? k[u] : mn;
      mx = k[u] > mx ? k[u] : mx;
    }
  };
  u64 c = b0;
  if constexpr (VEC && PreVec<DT>::NV > 0) {
    for (; c + (u64)UN * CH <= b1; c += (u64)UN * CH) {
      uint4 w[UN][PreVec<DT>::NV > 0 ? PreVec<DT>::NV : 1];
#pragma unroll
      for (int q = 0; q < UN; ++q) {
        const uint4 *src = reinterpret_cast<const uint4 *>(base + (c + (u64)q * CH + (u64)lane * V) * D);
#pragma unroll
        for (int v = 0; v < PreVec<DT>::NV; ++v) w[q][v] = __ldcs(src + v);
      }
#pragma unroll
      for (int q = 0; q < UN; ++q) {
        Key k[V];
#pragma unroll
        for (int u = 0; u < V; ++u) k[u] = Tr::key(reinterpret_cast<const char *>(&w[q][0]) + u * D);
        visit(k, c + (u64)q * CH, true);
      }
    }
  }
  for (; c < b1; c += CH) {
    Key k[V];
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const u64 e = c + (u64)lane * V + u;
      k[u] = e < b1 ? Tr::key(base + e * D) : (Key)0;
    }
    visit(k, c, c + CH <= b1);
  }
}

template <int DT>
__global__ void __launch_bounds__(PRE_THREADS) prepass_kernel(const char *base, u64 n, PrepassPart *parts,
                                                              unsigned long long *tslot, const u32 *need) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  if (need && *need == 0) return;  // the entry kernel proved a non-easy input (k_plan.cuh)
  KTIMER(tslot, KS_PREPASS);
  constexpr int CH = 32 * PreVec<DT>::V * 2;  // segment granularity (whole vector chunks)
  u32 nd = 1, ni = 1;
  Key mn = key_max<Key>(), mx = (Key)0;
  const int lane = threadIdx.x & 31;
  const u64 gw = ((u64)blockIdx.x * PRE_THREADS + threadIdx.x) >> 5;
  const u64 W = (u64)gridDim.x * PRE_THREADS / 32;
  const u64 L = (n + W * CH - 1) / (W * CH) * CH;
  const u64 b0 = gw * L < n ? gw * L : n;
  const u64 b1 = b0 + L < n ? b0 + L : n;
  if (PreVec<DT>::NV > 0 && ((uintptr_t)base & 15) == 0) prepass_segment<DT, true>(base, n, b0, b1, nd, ni, mn, mx);
  else prepass_segment<DT, false>(base, n, b0, b1, nd, ni, mn, mx);
  nd = __all_sync(0xffffffffu, nd);
  ni = __all_sync(0xffffffffu, ni);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Key x = shfl_xor_key(mn, o), y = shfl_xor_key(mx, o);
    mn = x < mn ? x : mn;
    mx = y > mx ? y : mx;
  }
  __shared__ u32 s_nd[PRE_THREADS / 32], s_ni[PRE_THREADS / 32];
  __shared__ Key s_mn[PRE_THREADS / 32], s_mx[PRE_THREADS / 32];
  const int wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_nd[wid] = nd;
    s_ni[wid] = ni;
    s_mn[wid] = mn;
    s_mx[wid] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < PRE_THREADS / 32; ++w) {
      nd &= s_nd[w];
      ni &= s_ni[w];
      mn = s_mn[w] < mn ? s_mn[w] : mn;
      mx = s_mx[w] > mx ? s_mx[w] : mx;
    }
    PrepassPart p;
    p.nd = nd;
    p.ni = ni;
    p.pad0 = p.pad1 = 0;
    key_to_words<Key>(mn, p.mn);
    key_to_words<Key>(mx, p.mx);
    parts[blockIdx.x] = p;
  }
}

// Fold the parts: one CTA, a thread per part, then warp shuffles.
constexpr int PRERED_THREADS = 1024;
template <int DT>
__global__ void __launch_bounds__(PRERED_THREADS) prepass_reduce_kernel(const PrepassPart *parts, int nparts,
                                                                        PrepassOut *out, unsigned long long *tslot,
                                                                        const u32 *need) {
  using Key = typename Traits<DT>::Key;
  if (need && *need == 0) return;
  KTIMER(tslot, KS_PREREDUCE);
  u32 nd = 1, ni = 1;
  Key mn = key_max<Key>(), mx = (Key)0;
  for (int i = threadIdx.x; i < nparts; i += PRERED_THREADS) {
    nd &= parts[i].nd;
    ni &= parts[i].ni;
    Key a = key_from_words<Key>(parts[i].mn), b = key_from_words<Key>(parts[i].mx);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  nd = __syncthreads_and(nd);
  ni = __syncthreads_and(ni);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Key x = shfl_xor_key(mn, o), y = shfl_xor_key(mx, o);
    mn = x < mn ? x : mn;
    mx = y > mx ? y : mx;
  }
  __shared__ Key s_mn[PRERED_THREADS / 32], s_mx[PRERED_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_mn[wid] = mn;
    s_mx[wid] = mx;
  }
  __syncthreads();
  if (wid == 0) {
    mn = s_mn[lane];
    mx = s_mx[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Key x = shfl_xor_key(mn, o), y = shfl_xor_key(mx, o);
      mn = x < mn ? x : mn;
      mx = y > mx ? y : mx;
    }
    if (lane == 0) {
      out->nondecreasing = nd;
      out->nonincreasing = ni;
      key_to_words<Key>(mn, out->minkey);
      key_to_words<Key>(mx, out->maxkey);
    }
  }
}

// Sample pre-check of the easy-input test (SURVEY 8(a) a0 "cheaper variant"):
// 16384 stratified adjacent pairs.  If one pair ascends and another descends,
// the input is neither sorted nor reverse-sorted (nor all equal) and the full
// pre-pass can be skipped; otherwise the full pre-pass decides.  Run by a
// whole CTA (the sort's entry kernel); returns asc | desc << 1 to every thread.
constexpr int PRESAMPLE_PAIRS = 16384;

template <int DT>
__device__ int presample_block(const char *base, u64 n) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  int asc = 0, desc = 0;
  constexpr int U = 8;  // pairs per thread with their loads in flight together
  for (int i0 = threadIdx.x; i0 < PRESAMPLE_PAIRS; i0 += U * blockDim.x) {
    Key a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      const u64 p = (u64)(((u128)(u64)(i < PRESAMPLE_PAIRS ? i : 0) * (u128)(n - 1)) / (u128)PRESAMPLE_PAIRS);
      a[u] = Tr::key(base + p * Tr::D);  // 0 <= p <= n-2
      b[u] = Tr::key(base + (p + 1) * Tr::D);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      asc |= a[u] < b[u];
      desc |= b[u] < a[u];
    }
  }
  asc = __syncthreads_or(asc);
  desc = __syncthreads_or(desc);
  return (asc ? 1 : 0) | (desc ? 2 : 0);
}

// In-place reversal of n elements of D bytes ("reverses the input in
// the case that the input was sorted in decreasing order").
template <int DT>
__global__ void reverse_kernel(char *base, u64 n, unsigned long long *tslot) {
  using Tr = Traits<DT>;
  KTIMER(tslot, KS_REV);
  using Unit = typename Tr::Unit;
  constexpr int UPE = Tr::D / (int)sizeof(Unit);
  const u64 half = n / 2;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < half; i += (u64)gridDim.x * blockDim.x) {
    Unit *a = reinterpret_cast<Unit *>(base + i * Tr::D);
    Unit *b = reinterpret_cast<Unit *>(base + (n - 1 - i) * Tr::D);
#pragma unroll
    for (int w = 0; w < UPE; ++w) {
      Unit x = a[w];
      a[w] = b[w];
      b[w] = x;
    }
  }
}

// ips4o_classify test kernel: the same tree_bucket the classification and
// permutation kernels use.
template <int DT>
__global__ void classify_test_kernel(const char *elems, u64 n, const typename Traits<DT>::Key *tree,
                                     const typename Traits<DT>::Key *spl, int l, int eq, u32 *out) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  __shared__ Key s_tree[256], s_spl[256];
  for (int i = threadIdx.x; i < (1 << l); i += blockDim.x) {
    s_tree[i] = tree[i];
    s_spl[i] = spl[i];
  }
  __syncthreads();
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    out[i] = tree_bucket<Key>(s_tree, s_spl, l, eq, Tr::key(elems + i * Tr::D));
}

// K0m: exact key range of the TF_MEASURE tasks of a DIGIT level (DESIGN R27;
// the per-task analogue of IPS2Ra's significant-bit scan).  One
// CTA per part of a task (parts of ~64K elements, at most MEAS_MAXPARTS), then
// one thread per task folds the parts into the task's [lo, hi].
constexpr int MEAS_THREADS = 512;
constexpr u64 MEAS_PART_ELEMS = 65536;
constexpr u32 MEAS_MAXPARTS = 296;

template <int DT>
__global__ void __launch_bounds__(MEAS_THREADS) measure_part_kernel(LevelArgs A) {
  using Tr = Traits<DT>;
  using Key = typename Tr::Key;
  constexpr int D = Tr::D;
  KTIMER(A.tslot, KS_MEASURE);
  const u32 ti = A.measure_part[2 * blockIdx.x];
  const u32 pw = A.measure_part[2 * blockIdx.x + 1];
  const u64 p = pw & 0xFFFFu, np = pw >> 16;
  const TaskDesc &t = A.tasks[ti].t;
  const u64 b0 = t.size * p / np, b1 = t.size * (p + 1) / np;
  const char *src = A.base + t.begin * D;
  Key mn = key_max<Key>(), mx = (Key)0;
  for (u64 e = b0 + threadIdx.x; e < b1; e += MEAS_THREADS) {
    const Key k = Tr::key(src + e * D);
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Key x = shfl_xor_key(mn, o), y = shfl_xor_key(mx, o);
    mn = x < mn ? x : mn;
    mx = y > mx ? y : mx;
  }
  __shared__ Key s_mn[MEAS_THREADS / 32], s_mx[MEAS_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_mn[wid] = mn;
    s_mx[wid] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < MEAS_THREADS / 32; ++w) {
      mn = s_mn[w] < mn ? s_mn[w] : mn;
      mx = s_mx[w] > mx ? s_mx[w] : mx;
    }
    PrepassPart q;
    q.nd = q.ni = q.pad0 = q.pad1 = 0;
    key_to_words<Key>(mn, q.mn);
    key_to_words<Key>(mx, q.mx);
    reinterpret_cast<PrepassPart *>(A.measure_out)[blockIdx.x] = q;
  }
}

template <int DT>
__global__ void measure_reduce_kernel(LevelArgs A, u32 nmeasure) {
  using Key = typename Traits<DT>::Key;
  KTIMER(A.tslot, KS_MEASURE_RED);
  const u32 f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nmeasure) return;
  const u32 ti = A.measure_task[3 * f], first = A.measure_task[3 * f + 1], np = A.measure_task[3 * f + 2];
  const PrepassPart *parts = reinterpret_cast<const PrepassPart *>(A.measure_out) + first;
  Key mn = key_max<Key>(), mx = (Key)0;
  for (u32 i = 0; i < np; ++i) {
    Key a = key_from_words<Key>(parts[i].mn), b = key_from_words<Key>(parts[i].mx);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  TaskDesc &t = A.tasks[ti].t;
  const Key lo = key_from_words<Key>(t.lo), hi = key_from_words<Key>(t.hi);
  // the measured range lies inside the bounds; clamp anyway (the bounds are the invariant)
  if (mn < lo) mn = lo;
  if (mx > hi) mx = hi;
  key_to_words<Key>(mn, t.lo);
  key_to_words<Key>(mx, t.hi);
}

// ---------------------------------------------------------------- distributed samplesort
// The sample of one shard: element j is A[sample_index(seed, 0, 0, n, j)]
// (the counter-based draw of DESIGN R8, "task" = the whole shard), copied as
// D bytes (D is a multiple of 4).
__global__ void gather_sample_kernel(const char *base, u64 n, u64 seed, u64 m, int D, char *out) {
  const int w = D / 4;
  for (u64 x = (u64)blockIdx.x * blockDim.x + threadIdx.x; x < m * (u64)w; x += (u64)gridDim.x * blockDim.x) {
    const u64 j = x / (u64)w, q = x % (u64)w;
    const u64 i = sample_index(seed, 0, 0, n, j);
    reinterpret_cast<u32 *>(out)[j * w + q] = reinterpret_cast<const u32 *>(base + i * (u64)D)[q];
  }
}

// Splitter j < parts - 1 of the sorted global sample: the element at rank
// ((j + 1) * total) / parts - 1 (equidistant picks).
__global__ void pick_kernel(const char *sorted, u64 total, int parts, int D, char *out) {
  const int w = D / 4;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < (parts - 1) * w; x += gridDim.x * blockDim.x) {
    const int j = x / w, q = x % w;
    const u64 r = ((u64)(j + 1) * total) / (u64)parts - 1;
    reinterpret_cast<u32 *>(out)[(u64)j * w + q] = reinterpret_cast<const u32 *>(sorted + r * (u64)D)[q];
  }
}

}  // namespace ips4o
