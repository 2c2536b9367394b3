// common.cuh -- per-dtype traits and small device helpers of the sm_100a path.
// Product code; independent of oracle/.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace ips4o {

// ------------------------------------------------------------------ keys
// Keys live in an order-preserving unsigned space: comparisons are plain
// unsigned '<'.  The element BYTES are what gets moved; the key is only used
// to classify.

__host__ __device__ __forceinline__ u64 f64_to_key(u64 bits) {
  // negative doubles: flip all bits; non-negative: flip the sign bit
  return bits ^ ((u64)((i64)bits >> 63) | (1ull << 63));
}
__host__ __device__ __forceinline__ u64 key_to_f64(u64 k) {
  return k ^ ((u64)((i64)(~k) >> 63) | (1ull << 63));
}

__device__ __forceinline__ u32 bswap32(u32 x) { return __byte_perm(x, 0, 0x0123); }

// ------------------------------------------------------------------ 192-bit keys
// Quartet keys (a, b, c) compared lexicographically (Alg. 3) are
// the 192-bit number a*2^128 + b*2^64 + c; w[0] = c is the least significant.
struct K192 {
  u64 w[3];
  __host__ __device__ __forceinline__ K192() {}
  __host__ __device__ __forceinline__ K192(u64 x) : w{x, 0, 0} {}
  __host__ __device__ __forceinline__ K192(u64 lo, u64 mid, u64 hi) : w{lo, mid, hi} {}
  __host__ __device__ __forceinline__ explicit operator u64() const { return w[0]; }
  __host__ __device__ __forceinline__ explicit operator u32() const { return (u32)w[0]; }
};
__host__ __device__ __forceinline__ bool operator<(const K192 &x, const K192 &y) {
  if (x.w[2] != y.w[2]) return x.w[2] < y.w[2];
  if (x.w[1] != y.w[1]) return x.w[1] < y.w[1];
  return x.w[0] < y.w[0];
}
__host__ __device__ __forceinline__ bool operator>(const K192 &x, const K192 &y) { return y < x; }
__host__ __device__ __forceinline__ bool operator<=(const K192 &x, const K192 &y) { return !(y < x); }
__host__ __device__ __forceinline__ bool operator>=(const K192 &x, const K192 &y) { return !(x < y); }
__host__ __device__ __forceinline__ bool operator==(const K192 &x, const K192 &y) {
  return x.w[0] == y.w[0] && x.w[1] == y.w[1] && x.w[2] == y.w[2];
}
__host__ __device__ __forceinline__ bool operator!=(const K192 &x, const K192 &y) { return !(x == y); }
__host__ __device__ __forceinline__ K192 operator-(const K192 &x, const K192 &y) {
  K192 r;
  r.w[0] = x.w[0] - y.w[0];
  const u64 b0 = x.w[0] < y.w[0];
  const u64 t1 = x.w[1] - y.w[1];
  const u64 b1 = (x.w[1] < y.w[1]) | (t1 < b0);
  r.w[1] = t1 - b0;
  r.w[2] = x.w[2] - y.w[2] - b1;
  return r;
}
__host__ __device__ __forceinline__ K192 operator+(const K192 &x, const K192 &y) {
  K192 r;
  r.w[0] = x.w[0] + y.w[0];
  const u64 c0 = r.w[0] < x.w[0];
  const u64 t1 = x.w[1] + y.w[1];
  const u64 c1 = (t1 < x.w[1]) | ((t1 + c0) < t1);
  r.w[1] = t1 + c0;
  r.w[2] = x.w[2] + y.w[2] + c1;
  return r;
}
__host__ __device__ __forceinline__ K192 operator|(const K192 &x, const K192 &y) {
  return K192(x.w[0] | y.w[0], x.w[1] | y.w[1], x.w[2] | y.w[2]);
}
__host__ __device__ __forceinline__ K192 operator^(const K192 &x, const K192 &y) {
  return K192(x.w[0] ^ y.w[0], x.w[1] ^ y.w[1], x.w[2] ^ y.w[2]);
}
__host__ __device__ __forceinline__ K192 operator&(const K192 &x, const K192 &y) {
  return K192(x.w[0] & y.w[0], x.w[1] & y.w[1], x.w[2] & y.w[2]);
}
__host__ __device__ __forceinline__ K192 operator>>(const K192 &x, int s) {
  if (s <= 0) return x;
  if (s >= 192) return K192(0);
  const int q = s >> 6, r = s & 63;
  u64 in[3] = {x.w[0], x.w[1], x.w[2]};
  K192 o(0);
  for (int i = 0; i + q < 3; ++i) {
    const u64 lo = in[i + q];
    const u64 hi = (i + q + 1 < 3) ? in[i + q + 1] : 0;
    o.w[i] = r ? (lo >> r) | (hi << (64 - r)) : lo;
  }
  return o;
}
__host__ __device__ __forceinline__ K192 operator<<(const K192 &x, int s) {
  if (s <= 0) return x;
  if (s >= 192) return K192(0);
  const int q = s >> 6, r = s & 63;
  u64 in[3] = {x.w[0], x.w[1], x.w[2]};
  K192 o(0);
  for (int i = 2; i - q >= 0; --i) {
    const u64 hi = in[i - q];
    const u64 lo = (i - q - 1 >= 0) ? in[i - q - 1] : 0;
    o.w[i] = r ? (hi << r) | (lo >> (64 - r)) : hi;
  }
  return o;
}

template <int DT> struct Traits;

template <> struct Traits<DT_U64> {
  static constexpr int D = 8;
  using Key = u64;
  using Unit = u64;                 // copy unit (element alignment)
  static constexpr int B = 64;      // elements per block -> 512 B blocks
  static constexpr int KIDX = 256;  // bucket indices (buffer blocks) per CTA
  static constexpr int BASE_CAP = 24576;
  static constexpr int CLS_THREADS = 512;
  static constexpr int CLS_TILE = 2048;
  static constexpr int KEY_UNITS = 1;
  __device__ __forceinline__ static Key key(const char *e) { return *reinterpret_cast<const u64 *>(e); }
};

template <> struct Traits<DT_F64> {
  static constexpr int D = 8;
  using Key = u64;
  using Unit = u64;
  static constexpr int B = 64;
  static constexpr int KIDX = 256;
  static constexpr int BASE_CAP = 24576;
  static constexpr int CLS_THREADS = 512;
  static constexpr int CLS_TILE = 2048;
  static constexpr int KEY_UNITS = 1;
  __device__ __forceinline__ static Key key(const char *e) {
    return f64_to_key(*reinterpret_cast<const u64 *>(e));
  }
};

template <> struct Traits<DT_U32> {
  static constexpr int D = 4;
  using Key = u64;                  // zero-extended: the 64-bit key machinery applies
  using Unit = u32;
  static constexpr int B = 128;     // 512 B blocks
  static constexpr int KIDX = 256;
  static constexpr int BASE_CAP = 32768;
  static constexpr int CLS_THREADS = 512;
  static constexpr int CLS_TILE = 4096;
  static constexpr int KEY_UNITS = 1;
  __device__ __forceinline__ static Key key(const char *e) { return *reinterpret_cast<const u32 *>(e); }
};

template <> struct Traits<DT_QUARTET> {
  static constexpr int D = 32;       // {u64 a, b, c; u64 value}, key (a, b, c)
  using Key = K192;
  using Unit = uint4;
  static constexpr int B = 16;       // 512 B blocks
  static constexpr int KIDX = 256;
  static constexpr int BASE_CAP = 6144;
#ifndef IPS4O_QUA_CLS_THREADS
#define IPS4O_QUA_CLS_THREADS 1024  // (2^26: 512 5.44 ms, 1024 4.96 ms, 256 7.36 ms of classification)
#endif
#ifndef IPS4O_QUA_CLS_TILE
#define IPS4O_QUA_CLS_TILE 1024
#endif
  static constexpr int CLS_THREADS = IPS4O_QUA_CLS_THREADS;
  static constexpr int CLS_TILE = IPS4O_QUA_CLS_TILE;
  static constexpr int KEY_UNITS = 2;
  __device__ __forceinline__ static Key key(const char *e) {
    const u64 *q = reinterpret_cast<const u64 *>(e);
    return K192(q[2], q[1], q[0]);
  }
};

template <> struct Traits<DT_PAIR> {
  static constexpr int D = 16;
  using Key = u64;
  using Unit = uint4;
  static constexpr int B = 32;      // 512 B blocks
  static constexpr int KIDX = 256;
  static constexpr int BASE_CAP = 12288;
  static constexpr int CLS_THREADS = 512;
  static constexpr int CLS_TILE = 1024;
  static constexpr int KEY_UNITS = 1;
  __device__ __forceinline__ static Key key(const char *e) { return *reinterpret_cast<const u64 *>(e); }
};

template <> struct Traits<DT_REC100> {
  static constexpr int D = 100;
  using Key = u128;                 // 80-bit big-endian key in the low 80 bits
  using Unit = u32;
  static constexpr int B = 8;       // 800 B blocks = 25 x 32 B sectors
  static constexpr int KIDX = 128;
  static constexpr int BASE_CAP = 1792;
// (measured at 2^24: 256 threads / 256-record tiles 5.44 ms of classification,
// 512 / 512 3.47 ms, 128 / 256 8.7 ms)
#ifndef IPS4O_REC_CLS_THREADS
#define IPS4O_REC_CLS_THREADS 512
#endif
#ifndef IPS4O_REC_CLS_TILE
#define IPS4O_REC_CLS_TILE 512
#endif
  static constexpr int CLS_THREADS = IPS4O_REC_CLS_THREADS;
  static constexpr int CLS_TILE = IPS4O_REC_CLS_TILE;
  static constexpr int KEY_UNITS = 3;
  __device__ __forceinline__ static Key key(const char *e) {
    const u32 *w = reinterpret_cast<const u32 *>(e);
    u64 hi = ((u64)bswap32(w[0]) << 32) | (u64)bswap32(w[1]);
    u32 lo = bswap32(w[2]) >> 16;
    return ((u128)hi << 16) | (u128)lo;
  }
};

// ------------------------------------------------------------------ key helpers
template <class K> __host__ __device__ __forceinline__ K key_from_words(const u64 *w);
template <> __host__ __device__ __forceinline__ u64 key_from_words<u64>(const u64 *w) { return w[0]; }
template <> __host__ __device__ __forceinline__ u128 key_from_words<u128>(const u64 *w) {
  return ((u128)w[1] << 64) | (u128)w[0];
}
template <> __host__ __device__ __forceinline__ K192 key_from_words<K192>(const u64 *w) { return K192(w[0], w[1], w[2]); }
template <class K> __host__ __device__ __forceinline__ void key_to_words(K k, u64 *w);
template <> __host__ __device__ __forceinline__ void key_to_words<u64>(u64 k, u64 *w) {
  w[0] = k;
  w[1] = 0;
  w[2] = 0;
}
template <> __host__ __device__ __forceinline__ void key_to_words<u128>(u128 k, u64 *w) {
  w[0] = (u64)k;
  w[1] = (u64)(k >> 64);
  w[2] = 0;
}
template <> __host__ __device__ __forceinline__ void key_to_words<K192>(K192 k, u64 *w) {
  w[0] = k.w[0];
  w[1] = k.w[1];
  w[2] = k.w[2];
}

__device__ __forceinline__ int bitlen(u64 x) { return x ? 64 - __clzll((long long)x) : 0; }
__device__ __forceinline__ int bitlen(u128 x) {
  u64 h = (u64)(x >> 64);
  return h ? 128 - __clzll((long long)h) : bitlen((u64)x);
}
__device__ __forceinline__ u32 digit_of(u64 x, int shift, u32 mask) { return (u32)(x >> shift) & mask; }
__device__ __forceinline__ u32 digit_of(u128 x, int shift, u32 mask) { return (u32)(x >> shift) & mask; }
__device__ __forceinline__ int bitlen(const K192 &x) {
  return x.w[2] ? 128 + bitlen(x.w[2]) : x.w[1] ? 64 + bitlen(x.w[1]) : bitlen(x.w[0]);
}
__device__ __forceinline__ u32 digit_of(const K192 &x, int shift, u32 mask) { return (u32)(x >> shift) & mask; }

template <class K> __host__ __device__ __forceinline__ K key_max();
template <> __host__ __device__ __forceinline__ u64 key_max<u64>() { return ~0ull; }
template <> __host__ __device__ __forceinline__ u128 key_max<u128>() { return (((u128)1) << 80) - 1; }
template <> __host__ __device__ __forceinline__ K192 key_max<K192>() { return K192(~0ull, ~0ull, ~0ull); }

// ------------------------------------------------------------------ lookup table of starting leaves
// (P:4049-4050).  Slot q of a task's table covers [llo + q*2^ls, llo +
// (q+1)*2^ls) (slot 0 also every key below, the last slot every key above).
// A 16-bit entry holds either the final bucket (LUT_FIN, no splitter in the
// slot) or a = #{splitters < the slot's first key} (9 bits) and the number c
// of splitters inside it (6 bits, 63 = "63 or more").
constexpr int LUT_BITS = 14;
constexpr u32 LUT_SLOTS = 1u << LUT_BITS;
constexpr u32 LUT_FIN = 1u << 15;

// Slot of a key offset d = x - llo in a lookup table.  Linear (logm = 0):
// d >> ls.  Logarithmic (logm = M > 0): exact below 2^M, then 2^M slots per
// octave -- d in [2^e, 2^(e+1)) (e >= M) maps to 2^M (e - M) + (d >> (e - M)),
// monotone and contiguous (relative resolution 2^-M): dense at the low end of
// the range, for distributions whose splitters crowd there (Zipf).  The
// caller clamps to the table's last used slot.
__device__ __forceinline__ u32 lut_slot_of(u64 d, int ls, int logm) {
  if (logm == 0) return (u32)min(d >> ls, (u64)0xFFFFFFFFu);
  if (d < (2ull << logm)) return (u32)d;
  const int e = 63 - __clzll((long long)d);
  return (u32)(((u64)(e - logm) << logm) + (d >> (e - logm)));
}
// First offset of slot q (inverse of lut_slot_of on slot starts).
__device__ __forceinline__ u64 lut_slot_start(u32 q, int ls, int logm) {
  if (logm == 0) return (u64)q << ls;
  if (q < (2u << logm)) return q;
  const u32 j = q >> logm;  // >= 2: e = j + logm - 1
  const u64 t = (u64)q - ((u64)(j - 1) << logm);
  return t << (j - 1);
}

// ------------------------------------------------------------------ RNG (DESIGN R8)
constexpr u64 GAMMA = 0x9E3779B97F4A7C15ull;
__host__ __device__ __forceinline__ u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// index of sample j of the task (begin, size) at `level`
__device__ __forceinline__ u64 sample_index(u64 seed, u32 level, u64 begin, u64 size, u64 j) {
  u64 base = mix64(seed + GAMMA * ((u64)level + 1)) ^ mix64(begin + GAMMA * (size + 1));
  u64 u = mix64(base + GAMMA * (j + 1));
  return begin + __umul64hi(u, size);
}

// ------------------------------------------------------------------ memory helpers
__device__ __forceinline__ u64 ld_acquire_u64(const u64 *p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 ld_relaxed_u64(const u64 *p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  u32 s = (u32)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  u32 s = (u32)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// Bulk L2 prefetch of [p, p + bytes): a hint issued by threads tid < nthr in
// 16 KiB pieces; the range is shrunk to whole 16-byte units inside it, so the
// prefetch never touches memory outside [p, p + bytes).
__device__ __forceinline__ void prefetch_l2(const void *p, u64 bytes, int tid, int nthr) {
  uintptr_t a = ((uintptr_t)p + 15) & ~(uintptr_t)15;
  uintptr_t e = ((uintptr_t)p + bytes) & ~(uintptr_t)15;
  if (e <= a) return;
  constexpr u64 PIECE = 16384;
  const u64 n = (u64)(e - a);
  for (u64 off = (u64)tid * PIECE; off < n; off += (u64)nthr * PIECE) {
    const u32 sz = (u32)((n - off) < PIECE ? (n - off) : PIECE);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + off), "r"(sz) : "memory");
  }
}
// Bulk (TMA) copy shared -> global of `bytes` (multiple of 16, both addresses
// 16-byte aligned), issued by one thread after a barrier; the generic-proxy
// writes to shared memory are made visible to the async proxy first.
__device__ __forceinline__ void bulk_store_s2g(void *gdst, const void *ssrc, u32 bytes) {
  const u32 sa = (u32)__cvta_generic_to_shared(ssrc);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the source reads of the issued bulk stores are done (shared memory reusable)
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// the issued bulk stores are complete
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Copy bytes [g, g + nbytes) (g and nbytes multiples of 4) into shared memory
// at s + (g & 15) with 16-byte cp.async for the aligned body and 4-byte
// cp.async for the unaligned head/tail; returns the head offset (g & 15).
// Reads never leave [g & ~15, g + nbytes) rounded to 4 B, i.e. never past the
// end of the array.  Executed by `nthr` threads with index `tid`.
__device__ __forceinline__ int tile_load_async(char *s, const char *g, u64 nbytes, int tid, int nthr) {
  const uintptr_t a = (uintptr_t)g;
  const uintptr_t a0 = a & ~(uintptr_t)15;  // smem byte s[x - a0] holds global byte x
  const int head = (int)(a - a0);
  const uintptr_t end = a + nbytes;
  uintptr_t body0 = (a + 15) & ~(uintptr_t)15;
  uintptr_t body1 = end & ~(uintptr_t)15;
  if (body1 < body0) body1 = body0;  // tiny range: all of it is head/tail words
  // head words [a, min(body0, end))
  const uintptr_t hend = body0 < end ? body0 : end;
  const int nh = (int)((hend - a) >> 2);
  if (tid < nh) cp_async4(s + head + 4 * tid, (const void *)(a + 4 * tid));
  // body
  const u64 nb = (u64)((body1 - body0) >> 4);
  const u64 boff = (u64)(body0 - a0);
  for (u64 i = tid; i < nb; i += nthr) cp_async16(s + boff + 16 * i, (const void *)(body0 + 16 * i));
  // tail words [max(body1, hend), end)
  const uintptr_t t0 = body1 > hend ? body1 : hend;
  const int nt = end > t0 ? (int)((end - t0) >> 2) : 0;
  if (tid < nt) cp_async4(s + (t0 - a0) + 4 * tid, (const void *)(t0 + 4 * tid));
  return head;
}

// ------------------------------------------------------------------ checked build
// IPS4O_CHECKS: every guarded index is bounds-checked on the device; a failed
// check skips the access and raises ERR_CHECK (reported by the synchronising
// calls and ips4o_device_status).  Without it the guard is `true` (no code).
#ifdef IPS4O_CHECKS
#define IPS4O_GUARD(cond, errp) ((cond) ? true : (atomicOr((errp), (u32)ERR_CHECK), false))
#else
#define IPS4O_GUARD(cond, errp) true
#endif

// ------------------------------------------------------------------ key shuffles
template <class Key>
__device__ __forceinline__ Key shfl_key(Key v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}
template <>
__device__ __forceinline__ u128 shfl_key<u128>(u128 v, int src) {
  u64 lo = __shfl_sync(0xffffffffu, (u64)v, src);
  u64 hi = __shfl_sync(0xffffffffu, (u64)(v >> 64), src);
  return ((u128)hi << 64) | lo;
}
template <>
__device__ __forceinline__ K192 shfl_key<K192>(K192 v, int src) {
  return K192(__shfl_sync(0xffffffffu, v.w[0], src), __shfl_sync(0xffffffffu, v.w[1], src),
              __shfl_sync(0xffffffffu, v.w[2], src));
}
template <class Key>
__device__ __forceinline__ Key shfl_xor_key(Key v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
template <>
__device__ __forceinline__ K192 shfl_xor_key<K192>(K192 v, int m) {
  return K192(__shfl_xor_sync(0xffffffffu, v.w[0], m), __shfl_xor_sync(0xffffffffu, v.w[1], m),
              __shfl_xor_sync(0xffffffffu, v.w[2], m));
}
template <>
__device__ __forceinline__ u128 shfl_xor_key<u128>(u128 v, int m) {
  u64 lo = __shfl_xor_sync(0xffffffffu, (u64)v, m);
  u64 hi = __shfl_xor_sync(0xffffffffu, (u64)(v >> 64), m);
  return ((u128)hi << 64) | lo;
}

// ------------------------------------------------------------------ device timing
// Kernel durations without host events (the levels are launched from the
// device): the first thread of every CTA lowers the slot's start, lane 0 of
// every warp raises its end when it leaves the kernel (any return path).
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <int SLOT> struct KTimer {
  // holds a reference to the kernel parameter (no register kept live)
  unsigned long long *const &ts;
  __device__ __forceinline__ explicit KTimer(unsigned long long *const &tslots) : ts(tslots) {
    if (ts && threadIdx.x == 0) atomicMin(&ts[2 * SLOT], gtimer());
  }
  __device__ __forceinline__ ~KTimer() {
    if (ts && (threadIdx.x & 31) == 0) atomicMax(&ts[2 * SLOT + 1], gtimer());
  }
};
#define KTIMER(tslots, slot) KTimer<slot> ktimer_(tslots)

// ------------------------------------------------------------------ block scan
// Exclusive scan of one u32 per thread over the first `n` threads of a CTA of
// NT threads (n <= NT).  `ws` must hold NT/32 + 1 u32.  Returns the exclusive
// prefix; *total gets the sum.  Contains __syncthreads.
template <int NT>
__device__ __forceinline__ u32 block_exclusive_scan(u32 v, u32 *ws, u32 *total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u32 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    u32 w = lane < NT / 32 ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) ws[lane] = w;  // inclusive warp totals
    if (lane == NT / 32 - 1) ws[NT / 32] = w;
  }
  __syncthreads();
  u32 pre = (wid > 0 ? ws[wid - 1] : 0) + x - v;
  *total = ws[NT / 32];
  __syncthreads();
  return pre;
}

// Block-wide exclusive scan with ONE barrier: every warp scans the warp
// totals itself.  The caller must pass a barrier before `ws` is written again
// (block_exclusive_scan above ends with one for that).
template <int NT>
__device__ __forceinline__ u32 block_exclusive_scan_1b(u32 v, u32 *ws, u32 *total) {
  static_assert(NT / 32 <= 32, "one warp total per lane");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u32 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  const u32 w = lane < NT / 32 ? ws[lane] : 0u;
  u32 iw = w;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, iw, o);
    if (lane >= o) iw += y;
  }
  *total = __shfl_sync(0xffffffffu, iw, NT / 32 - 1);
  return __shfl_sync(0xffffffffu, iw - w, wid) + x - v;
}

}  // namespace ips4o
