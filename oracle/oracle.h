/*
 * oracle.h -- plain, slow, single-threaded CPU oracle for the IPS4o / IPS2Ra
 * in-place partitioning step (arXiv 2009.13569).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load, call or link this
 * code.  The product path (paper_2009_13569_b200/) never touches it, and it
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line (section named next
 * to it); "S:<line>" = SPEC.md line.  Readings of ambiguous passages are the
 * numbered items of DESIGN.md "Readings of the paper".
 *
 * Element types (Alg. 3/4 P:1822-1855):
 *   ORC_U64    8-byte unsigned integer, compared with unsigned '<'
 *   ORC_F64    IEEE-754 double, compared with '<' (precondition: no NaN, no -0.0)
 *   ORC_PAIR   16 bytes {uint64 key; uint64 value}, compared on key only
 *   ORC_REC100 100 bytes, key = bytes 0..9 compared lexicographically as
 *              UNSIGNED bytes (Alg. 4; DESIGN reading R1)
 *   ORC_U32    4-byte unsigned integer, compared with unsigned '<'
 *   ORC_QUARTET 32 bytes {uint64 a, b, c; uint64 value}, key (a, b, c) compared
 *              lexicographically (Alg. 3)
 *
 * Pinning status: every function below is pinned by
 * a -m "not gpu" test against something other than itself (brute force,
 * Python's sorted(), numpy, closed forms, SPEC/SURVEY worked vectors).
 */
#ifndef IPS4O_ORACLE_H
#define IPS4O_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_U64 = 0, ORC_F64 = 1, ORC_PAIR = 2, ORC_REC100 = 3, ORC_U32 = 4, ORC_QUARTET = 5 };

/* Element size in bytes, 0 for an unknown dtype. */
size_t orc_elem_bytes(int dtype);

/* Strict weak order of the dtype: 1 iff a < b. */
int orc_less(int dtype, const void *a, const void *b);

/* Input precondition (DESIGN R2): F64 input must hold no NaN and no -0.0.
 * Returns -1 if fine, else the index of the first offending element. */
int64_t orc_check_input(int dtype, const void *p, uint64_t n);

/* THE oracle (P:328-331 problem statement: output is the input array in
 * sorted order): top-down recursive mergesort, stable, one auxiliary buffer of
 * n elements, merges take from the left run on ties.  Returns 0, or -1 on
 * allocation failure / bad dtype. */
int orc_mergesort(void *p, uint64_t n, int dtype);

/* Brute force used only to pin the mergesort on tiny inputs: O(n^2)
 * insertion sort written independently of orc_mergesort. */
int orc_insertion_sort(void *p, uint64_t n, int dtype);

/* 1 iff p[0..n) is non-decreasing under orc_less. */
int orc_is_sorted(const void *p, uint64_t n, int dtype);

/* Order-independent multiset hash: wrapping sum over elements of a 64-bit
 * mixer applied to the element's bytes. */
uint64_t orc_multiset_hash(const void *p, uint64_t n, int dtype);

/* Parity checker.  U64/F64: byte equality.
 * PAIR/REC100: identical key sequence AND, inside every maximal run of equal
 * keys, identical record multisets.  Returns -1 when g matches o, else the
 * first index where they disagree. */
int64_t orc_parity_check(const void *g, const void *o, uint64_t n, int dtype);

/* ---- sub-oracles for one partitioning step --------------------------------
 * Keys below are passed as raw elements of the dtype (for REC100 only the
 * first 10 bytes of each 'splitter' element matter).  No order-preserving
 * transform is used anywhere in the oracle. */

/* Sample draw (DESIGN R8): index of sample j of a task, from the
 * counter-based generator written out in DESIGN.md R8. */
uint64_t orc_sample_index(uint64_t seed, uint32_t level, uint64_t task_begin,
                          uint64_t task_size, uint64_t j);

/* Splitter selection from a SORTED sample of m = alpha*k elements
 * (DESIGN R8/R10/R23).  Writes the u unique splitters (elements)
 * to out_splitters (capacity k-1 elements), returns u and sets *equality and
 * *k_final (k after the equality-budget halving of R10).  kidx_max is the
 * bucket-index budget (number of buffer blocks per CTA). */
int orc_select_splitters(const void *sorted_sample, uint64_t m, int k, int kidx_max,
                         int dtype, void *out_splitters, int *equality, int *k_final);

/* Decision tree (Fig. 2): pad u unique
 * splitters with the largest to s = 2^l - 1, tree[1..s] breadth-first
 * (tree[0] is a dummy, zero-filled), splitter[0..s] sorted with
 * splitter[s] = splitter[s-1].  Returns l (= log2(s+1)).  tree and splitter
 * need room for 2^l elements each. */
int orc_build_tree(const void *splitters, int u, int dtype, void *tree, void *splitter);

/* Classification by the definition P:392-394 / P:432-437: leaf i with
 * s_{i-1} < e <= s_i found by a linear scan over splitter[0..s); with
 * equality buckets the bucket is 2i + 1 - [e < s_i]. */
int orc_classify_linear(const void *splitter, int l, int equality, int dtype, const void *e);

/* Classification literally as Alg. 1 (DESIGN R4): walk the
 * breadth-first tree l levels, then the equality step, then subtract k. */
int orc_classify_tree(const void *tree, const void *splitter, int l, int equality,
                      int dtype, const void *e);

/* IPS2Ra radix extractor: bits [shift, shift+bits) of the unsigned
 * key of e.  The key of F64 is obtained by the oracle's own IEEE-754 order
 * argument (DESIGN R20), of REC100 as the 80-bit big-endian number. */
uint32_t orc_radix_digit(int dtype, const void *e, int shift, int bits);
/* Logarithmic digit of an offset d (sample-adaptive IPS2Ra extractor, DESIGN R33). */
uint32_t orc_log_digit(uint64_t d, int M);

/* Bucket boundaries: E[j] = sum_{i<j} count[i] (exact, E[0]=0),
 * d[j] = ceil(E[j]/b)*b (block-rounded delimiters), j = 0..k. */
void orc_boundaries(const uint64_t *count, int k, uint64_t b, uint64_t *E, uint64_t *d);

/* Full-array helpers used by tests: histogram of orc_classify_linear over
 * p[0..n) into hist[0..2^(l+1)) (or 2^l without equality). */
void orc_histogram(const void *p, uint64_t n, int dtype, const void *splitter, int l,
                   int equality, uint64_t *hist);

#ifdef __cplusplus
}
#endif
#endif
