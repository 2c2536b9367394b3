/*
 * oracle.c -- plain, slow, single-threaded CPU oracle (see oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / reference leg may use it.  It shares no code with
 * the CUDA path in paper_2009_13569_b200/ and neither includes the other.
 *
 * Everything here is written to be checked against the paper by eye; no
 * blocking, fusion or reordering beyond what the cited passage states.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- element model */

size_t orc_elem_bytes(int dtype)
{
    switch (dtype) {
    case ORC_U64: return 8;
    case ORC_F64: return 8;
    case ORC_PAIR: return 16;
    case ORC_REC100: return 100;
    case ORC_U32: return 4;
    case ORC_QUARTET: return 32;
    default: return 0;
    }
}

/* unsigned 64-bit '<' */
static int less_u64(const void *a, const void *b)
{
    uint64_t x, y;
    memcpy(&x, a, 8);
    memcpy(&y, b, 8);
    return x < y;
}

/* unsigned 32-bit '<' */
static int less_u32(const void *a, const void *b)
{
    uint32_t x, y;
    memcpy(&x, a, 4);
    memcpy(&y, b, 4);
    return x < y;
}

/* IEEE double '<' */
static int less_f64(const void *a, const void *b)
{
    double x, y;
    memcpy(&x, a, 8);
    memcpy(&y, b, 8);
    return x < y;
}

/* Pair: one 64-bit unsigned key + 64-bit payload, compared on the key */
static int less_pair(const void *a, const void *b)
{
    uint64_t x, y;
    memcpy(&x, a, 8);
    memcpy(&y, b, 8);
    return x < y;
}

/* Quartet: Alg. 3 -- a, then b, then c */
static int less_quartet(const void *l, const void *r)
{
    uint64_t x[3], y[3];
    memcpy(x, l, 24);
    memcpy(y, r, 24);
    if (x[0] != y[0]) return x[0] < y[0];
    if (x[1] != y[1]) return x[1] < y[1];
    return x[2] < y[2];
}

/* 100B: Alg. 4, key bytes k[0..9] compared as unsigned bytes */
static int less_rec100(const void *a, const void *b)
{
    const unsigned char *l = (const unsigned char *)a;
    const unsigned char *r = (const unsigned char *)b;
    for (int i = 0; i <= 9; i++) {
        if (l[i] != r[i]) return l[i] < r[i];
    }
    return 0;
}

typedef int (*less_fn)(const void *, const void *);

static less_fn less_of(int dtype)
{
    switch (dtype) {
    case ORC_U64: return less_u64;
    case ORC_F64: return less_f64;
    case ORC_PAIR: return less_pair;
    case ORC_REC100: return less_rec100;
    case ORC_U32: return less_u32;
    case ORC_QUARTET: return less_quartet;
    default: return 0;
    }
}

int orc_less(int dtype, const void *a, const void *b)
{
    less_fn f = less_of(dtype);
    return f ? f(a, b) : 0;
}

int64_t orc_check_input(int dtype, const void *p, uint64_t n)
{
    if (dtype != ORC_F64) return -1;
    const unsigned char *c = (const unsigned char *)p;
    for (uint64_t i = 0; i < n; i++) {
        double x;
        memcpy(&x, c + 8 * i, 8);
        if (isnan(x)) return (int64_t)i;
        if (x == 0.0 && signbit(x)) return (int64_t)i;
    }
    return -1;
}

/* ---------------------------------------------------------------- mergesort */

/* Sort p[lo, hi) using aux[lo, hi) as scratch.  Top-down: split in the
 * middle, sort both halves, merge into aux taking from the left run on ties,
 * copy back. */
static void msort_rec(unsigned char *p, unsigned char *aux, uint64_t lo, uint64_t hi,
                      size_t D, less_fn less)
{
    if (hi - lo < 2) return;
    uint64_t mid = lo + (hi - lo) / 2;
    msort_rec(p, aux, lo, mid, D, less);
    msort_rec(p, aux, mid, hi, D, less);
    uint64_t i = lo, j = mid, o = lo;
    while (i < mid && j < hi) {
        /* take from the right run only if it is strictly smaller */
        if (less(p + j * D, p + i * D)) {
            memcpy(aux + o * D, p + j * D, D);
            j++;
        } else {
            memcpy(aux + o * D, p + i * D, D);
            i++;
        }
        o++;
    }
    while (i < mid) {
        memcpy(aux + o * D, p + i * D, D);
        i++;
        o++;
    }
    while (j < hi) {
        memcpy(aux + o * D, p + j * D, D);
        j++;
        o++;
    }
    memcpy(p + lo * D, aux + lo * D, (hi - lo) * D);
}

int orc_mergesort(void *p, uint64_t n, int dtype)
{
    size_t D = orc_elem_bytes(dtype);
    less_fn less = less_of(dtype);
    if (!D || !less) return -1;
    if (n < 2) return 0;
    unsigned char *aux = (unsigned char *)malloc(n * D);
    if (!aux) return -1;
    msort_rec((unsigned char *)p, aux, 0, n, D, less);
    free(aux);
    return 0;
}

/* ---------------------------------------------------------------- brute force */

int orc_insertion_sort(void *p, uint64_t n, int dtype)
{
    size_t D = orc_elem_bytes(dtype);
    less_fn less = less_of(dtype);
    if (!D || !less) return -1;
    unsigned char *a = (unsigned char *)p;
    unsigned char tmp[128];
    for (uint64_t i = 1; i < n; i++) {
        memcpy(tmp, a + i * D, D);
        uint64_t j = i;
        while (j > 0 && less(tmp, a + (j - 1) * D)) {
            memcpy(a + j * D, a + (j - 1) * D, D);
            j--;
        }
        memcpy(a + j * D, tmp, D);
    }
    return 0;
}

int orc_is_sorted(const void *p, uint64_t n, int dtype)
{
    size_t D = orc_elem_bytes(dtype);
    less_fn less = less_of(dtype);
    const unsigned char *a = (const unsigned char *)p;
    for (uint64_t i = 1; i < n; i++)
        if (less(a + i * D, a + (i - 1) * D)) return 0;
    return 1;
}

/* ---------------------------------------------------------------- multiset hash */

/* Steele-Lea-Flood SplitMix64 finaliser, used here only as a hash mixer. */
static uint64_t orc_mix(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t elem_hash(const unsigned char *e, size_t D)
{
    uint64_t h = 0x0123456789ABCDEFULL ^ D;
    for (size_t off = 0; off < D; off += 8) {
        uint64_t w = 0;
        size_t c = D - off < 8 ? D - off : 8;
        memcpy(&w, e + off, c);
        h = orc_mix(h ^ w) + off;
    }
    return orc_mix(h);
}

uint64_t orc_multiset_hash(const void *p, uint64_t n, int dtype)
{
    size_t D = orc_elem_bytes(dtype);
    const unsigned char *a = (const unsigned char *)p;
    uint64_t s = 0;
    for (uint64_t i = 0; i < n; i++) s += elem_hash(a + i * D, D);
    return s;
}

/* ---------------------------------------------------------------- parity */

static int equal_keys(int dtype, const void *a, const void *b)
{
    return !orc_less(dtype, a, b) && !orc_less(dtype, b, a);
}

static size_t cmp_D;
static int cmp_bytes(const void *a, const void *b) { return memcmp(a, b, cmp_D); }

int64_t orc_parity_check(const void *g, const void *o, uint64_t n, int dtype)
{
    size_t D = orc_elem_bytes(dtype);
    const unsigned char *G = (const unsigned char *)g;
    const unsigned char *O = (const unsigned char *)o;
    if (dtype == ORC_U64 || dtype == ORC_F64 || dtype == ORC_U32) {
        for (uint64_t i = 0; i < n; i++)
            if (memcmp(G + i * D, O + i * D, D) != 0) return (int64_t)i;
        return -1;
    }
    /* (i) identical key sequence */
    for (uint64_t i = 0; i < n; i++)
        if (!equal_keys(dtype, G + i * D, O + i * D)) return (int64_t)i;
    /* (ii) identical record multisets inside every maximal run of equal keys */
    uint64_t i = 0;
    while (i < n) {
        uint64_t j = i + 1;
        while (j < n && equal_keys(dtype, O + i * D, O + j * D)) j++;
        if (j - i == 1) {
            if (memcmp(G + i * D, O + i * D, D) != 0) return (int64_t)i;
        } else {
            unsigned char *x = (unsigned char *)malloc((j - i) * D);
            unsigned char *y = (unsigned char *)malloc((j - i) * D);
            if (!x || !y) {
                free(x);
                free(y);
                return (int64_t)i;
            }
            memcpy(x, G + i * D, (j - i) * D);
            memcpy(y, O + i * D, (j - i) * D);
            cmp_D = D;
            qsort(x, j - i, D, cmp_bytes);
            qsort(y, j - i, D, cmp_bytes);
            int bad = memcmp(x, y, (j - i) * D) != 0;
            free(x);
            free(y);
            if (bad) return (int64_t)i;
        }
        i = j;
    }
    return -1;
}

/* ---------------------------------------------------------------- sampling */

#define ORC_GAMMA 0x9E3779B97F4A7C15ULL

/* DESIGN R8: base = mix(seed + GAMMA*(level+1)) ^ mix(begin + GAMMA*(size+1));
 * u_j = mix(base + GAMMA*(j+1)); index = begin + floor(u_j * size / 2^64). */
uint64_t orc_sample_index(uint64_t seed, uint32_t level, uint64_t task_begin,
                          uint64_t task_size, uint64_t j)
{
    uint64_t base = orc_mix(seed + ORC_GAMMA * ((uint64_t)level + 1)) ^
                    orc_mix(task_begin + ORC_GAMMA * (task_size + 1));
    uint64_t u = orc_mix(base + ORC_GAMMA * (j + 1));
    unsigned __int128 prod = (unsigned __int128)u * (unsigned __int128)task_size;
    return task_begin + (uint64_t)(prod >> 64);
}

static int next_pow2_int(int x)
{
    int p = 1;
    while (p < x) p *= 2;
    return p;
}

/* P:728 "k-1 splitters are picked equidistantly from the sorted sample",
 * P:729 "we check for and remove duplicates", P:733 equality buckets "when
 * there are several identical splitters" (R23: at least one duplicate).
 * R10: with equality buckets on, 2*(s+1) bucket indices must fit kidx_max.
 * If u unique splitters are too many, u - (kidx_max/2 - 1) of them are
 * dropped, fewest picks first (ties: the smaller), never two neighbours, k
 * unchanged; if that many cannot be dropped, k is halved (alpha doubled) and
 * the pick repeated. */
int orc_select_splitters(const void *sorted_sample, uint64_t m, int k, int kidx_max,
                         int dtype, void *out_splitters, int *equality, int *k_final)
{
    size_t D = orc_elem_bytes(dtype);
    const unsigned char *S = (const unsigned char *)sorted_sample;
    unsigned char *out = (unsigned char *)out_splitters;
    for (;;) {
        uint64_t alpha = m / (uint64_t)k;
        int u = 0;
        int dup = 0;
        int picks[512];          /* picks per unique splitter (k <= 512) */
        for (int j = 0; j < k - 1; j++) {
            const unsigned char *c = S + ((uint64_t)(j + 1) * alpha - 1) * D;
            if (u > 0 && equal_keys(dtype, out + (size_t)(u - 1) * D, c)) {
                dup = 1;
                picks[u - 1]++;
                continue;
            }
            memcpy(out + (size_t)u * D, c, D);
            picks[u] = 1;
            u++;
        }
        int leaves = next_pow2_int(u + 1);
        int need = dup ? 2 * leaves : leaves;
        int keep_n = kidx_max / 2 - 1;
        if (dup && need > kidx_max && kidx_max >= 4 && u > keep_n) {
            /* DESIGN R10 (round 2, revised again): drop u - keep_n unique
             * splitters, one at a time: the one with the fewest picks
             * (smaller index first) among those whose neighbours in splitter
             * order are both still kept -- so the open bucket that absorbs a
             * dropped splitter's keys spans at most two former buckets.  If
             * fewer can be dropped that way, k is halved (below). */
            int drop_n = u - keep_n, got = 0;
            char dropped[512];
            memset(dropped, 0, sizeof dropped);
            while (got < drop_n) {
                int best = -1;
                for (int i = 0; i < u; i++) {
                    if (dropped[i] || (i > 0 && dropped[i - 1]) || (i + 1 < u && dropped[i + 1])) continue;
                    if (best < 0 || picks[i] < picks[best]) best = i;
                }
                if (best < 0) break;
                dropped[best] = 1;
                got++;
            }
            if (got == drop_n) {
                int w = 0;
                for (int i = 0; i < u; i++) {
                    if (dropped[i]) continue;
                    memmove(out + (size_t)w * D, out + (size_t)i * D, D);
                    w++;
                }
                u = w;
                leaves = next_pow2_int(u + 1);
                need = 2 * leaves;
            }
        }
        if (need <= kidx_max || k <= 2) {
            *equality = dup;
            *k_final = k;
            return u;
        }
        k /= 2;
    }
}

/* a_1 = s_{k/2-1}, children of a_i are a_{2i}, a_{2i+1}; the tree
 * over s = 2^l - 1 splitters is complete, so node i at depth d, position p
 * holds the splitter with in-order rank (2p+1)*2^(l-1-d) - 1.
 * pad with the largest splitter; splitter[s] = splitter[s-1]. */
int orc_build_tree(const void *splitters, int u, int dtype, void *tree, void *splitter)
{
    size_t D = orc_elem_bytes(dtype);
    const unsigned char *sp = (const unsigned char *)splitters;
    unsigned char *T = (unsigned char *)tree;
    unsigned char *S = (unsigned char *)splitter;
    int leaves = next_pow2_int(u + 1);
    int s = leaves - 1;
    int l = 0;
    while ((1 << l) < leaves) l++;
    for (int i = 0; i < s; i++) memcpy(S + (size_t)i * D, sp + (size_t)(i < u ? i : u - 1) * D, D);
    memcpy(S + (size_t)s * D, S + (size_t)(s - 1) * D, D);
    memset(T, 0, D);
    for (int i = 1; i <= s; i++) {
        int d = 0;
        while ((2 << d) <= i) d++;
        int p = i - (1 << d);
        int rank = (2 * p + 1) * (1 << (l - 1 - d)) - 1;
        memcpy(T + (size_t)i * D, S + (size_t)rank * D, D);
    }
    return l;
}

/* P:392-394 + P:432-437 by definition: i = #{j < s : s_j < e}. */
int orc_classify_linear(const void *splitter, int l, int equality, int dtype, const void *e)
{
    size_t D = orc_elem_bytes(dtype);
    const unsigned char *S = (const unsigned char *)splitter;
    int s = (1 << l) - 1;
    int i = 0;
    for (int j = 0; j < s; j++)
        if (orc_less(dtype, S + (size_t)j * D, e)) i++;
    if (!equality) return i;
    return 2 * i + 1 - orc_less(dtype, e, S + (size_t)i * D);
}

/* Alg. 1, read per R4: l tree steps, then the equality step with
 * splitter[b - k/2], output b - k (k = 2^{l+1}); without equality b - k/2. */
int orc_classify_tree(const void *tree, const void *splitter, int l, int equality,
                      int dtype, const void *e)
{
    size_t D = orc_elem_bytes(dtype);
    const unsigned char *T = (const unsigned char *)tree;
    const unsigned char *S = (const unsigned char *)splitter;
    int k = 1 << (l + 1);
    int b = 1;
    for (int r = 0; r < l; r++) b = 2 * b + orc_less(dtype, T + (size_t)b * D, e);
    if (equality) {
        b = 2 * b + 1 - orc_less(dtype, e, S + (size_t)(b - k / 2) * D);
        return b - k;
    }
    return b - k / 2;
}

/* ---------------------------------------------------------------- IPS2Ra digit */

uint32_t orc_radix_digit(int dtype, const void *e, int shift, int bits)
{
    const unsigned char *c = (const unsigned char *)e;
    if (dtype == ORC_QUARTET) {
        /* key = a*2^128 + b*2^64 + c (Alg. 3 order); bit q of it */
        uint64_t w[3];
        memcpy(w, c, 24); /* w[0] = a (most significant), w[2] = c */
        uint32_t d = 0;
        for (int t = bits - 1; t >= 0; t--) {
            int q = shift + t;
            int bit = (int)((w[2 - q / 64] >> (q % 64)) & 1);
            d = 2 * d + (uint32_t)bit;
        }
        return d;
    }
    if (dtype == ORC_REC100) {
        /* key = sum_i k[i] * 256^(9-i); bit q lives in byte 9 - q/8 */
        uint32_t d = 0;
        for (int t = bits - 1; t >= 0; t--) {
            int q = shift + t;
            int bit = (c[9 - q / 8] >> (q % 8)) & 1;
            d = 2 * d + (uint32_t)bit;
        }
        return d;
    }
    uint64_t key;
    if (dtype == ORC_U32) {
        uint32_t k32;
        memcpy(&k32, c, 4);
        key = k32;
    } else {
        memcpy(&key, c, 8);
    }
    if (dtype == ORC_F64) {
        /* Non-negative doubles order like their magnitude bits and come after
         * all negatives: key = 2^63 + mag.  Negative doubles order by
         * decreasing magnitude: key = 2^63 - 1 - mag. */
        double x;
        memcpy(&x, c, 8);
        uint64_t mag = key & 0x7FFFFFFFFFFFFFFFULL;
        key = signbit(x) ? (0x7FFFFFFFFFFFFFFFULL - mag) : (0x8000000000000000ULL + mag);
    }
    uint64_t d = 0;
    for (int t = bits - 1; t >= 0; t--) d = 2 * d + ((key >> (shift + t)) & 1);
    return (uint32_t)d;
}

/* Logarithmic digit of the sample-adaptive IPS2Ra extractor (P:4042-4047 asks
 * for an extractor adapted to the input distribution; the mapping itself is
 * DESIGN.md reading R33): the offset d of a key from its task's lower bound
 * maps to itself while d < 2^(M+1); an offset with leading bit e > M (2^e <=
 * d < 2^(e+1)) maps into the octave's 2^M equal slots: the slots of octave e
 * start at 2^M (e - M + 1) and the offset takes slot number floor((d - 2^e) /
 * 2^(e-M)) of them.  Monotone, and consecutive slots are contiguous. */
uint32_t orc_log_digit(uint64_t d, int M)
{
    if (d < ((uint64_t)2 << M)) return (uint32_t)d;
    int e = 0;
    while (e < 63 && (d >> (e + 1)) != 0) e++; /* leading bit */
    uint64_t first = ((uint64_t)1 << M) * (uint64_t)(e - M + 1);
    uint64_t width = (uint64_t)1 << (e - M);
    return (uint32_t)(first + (d - ((uint64_t)1 << e)) / width);
}

/* ---------------------------------------------------------------- boundaries */

void orc_boundaries(const uint64_t *count, int k, uint64_t b, uint64_t *E, uint64_t *d)
{
    E[0] = 0;
    for (int j = 0; j < k; j++) E[j + 1] = E[j] + count[j];
    for (int j = 0; j <= k; j++) d[j] = (E[j] + b - 1) / b * b;
}

void orc_histogram(const void *p, uint64_t n, int dtype, const void *splitter, int l,
                   int equality, uint64_t *hist)
{
    size_t D = orc_elem_bytes(dtype);
    const unsigned char *a = (const unsigned char *)p;
    int K = equality ? (1 << (l + 1)) : (1 << l);
    for (int j = 0; j < K; j++) hist[j] = 0;
    for (uint64_t i = 0; i < n; i++) hist[orc_classify_linear(splitter, l, equality, dtype, a + i * D)]++;
}
