/*
 * ips4o.h -- C ABI of the B200-native in-place samplesort partitioning step
 * (IPS4o, with the IPS2Ra radix classifier) from Axtmann, Witt, Ferizovic,
 * Sanders, "Engineering In-place (Shared-memory) Sorting Algorithms",
 * arXiv 2009.13569.  Citations "P:<line>" refer to the paper's LaTeX source
 * (PAPER.md line, section named next to it).
 *
 * Problem statement (Sec. 2): the input is an array A[0..n-1] of n
 * elements and the output is stored in the input array.  "In-place" means
 * sub-linear additional space; here the auxiliary DEVICE memory is
 * O(k*b) per CTA plus O(#tasks) task records, reported by
 * ips4o_scratch_bytes() and ips4o_stats.scratch_bytes.
 *
 * All entry points are plain C: raw pointers, sizes, and a cudaStream_t passed
 * as void*.  No PyTorch or C++ types cross this boundary.  Every call returns
 * an int status (0 = success, negative = IPS4O_ERR_*) and never throws.
 */
#ifndef IPS4O_H
#define IPS4O_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- element types
 * P:1877-1886 (data types of the experiments) and Alg. 3/4.
 *   IPS4O_U64           8 B, unsigned 64-bit key, ascending unsigned order.
 *   IPS4O_F64           8 B IEEE-754 double, ascending '<'.  Precondition: no
 *                       NaN; if both -0.0 and +0.0 occur their relative order
 *                       is unspecified (-0.0 sorts first).
 *   IPS4O_PAIR_U64_U64  16 B {uint64 key; uint64 value}, ordered by key only.
 *   IPS4O_REC100_KEY10  100 B record, key = bytes 0..9 compared
 *                       lexicographically as unsigned bytes (Alg. 4), payload
 *                       bytes 10..99 carried along.
 *   IPS4O_U32           4 B, unsigned 32-bit key, ascending unsigned order
 *                       ("32-bit unsigned integers").
 *   IPS4O_QUARTET       32 B {uint64 a, b, c; uint64 value}, key (a, b, c)
 *                       compared lexicographically (Alg. 3, P:1824-1836;
 *                       P:1878).
 * The sort is NOT stable (the block permutation P:840-922 moves whole blocks
 * in arbitrary order; DESIGN R3): for PAIR and REC100 the order inside a run
 * of equal keys is unspecified. */
enum ips4o_dtype {
    IPS4O_U64 = 0,
    IPS4O_F64 = 1,
    IPS4O_PAIR_U64_U64 = 2,
    IPS4O_REC100_KEY10 = 3,
    IPS4O_U32 = 4,
    IPS4O_QUARTET = 5
};

/* Classifier of the partitioning step. */
enum ips4o_algo {
    IPS4O_ALGO_TREE = 0,  /* IPS4o: sample + branchless splitter tree with
                             equality buckets        */
    IPS4O_ALGO_DIGIT = 1  /* IPS2Ra: MSB digit extractor     */
};

/* Status codes. */
enum ips4o_status {
    IPS4O_OK = 0,
    IPS4O_ERR_INVALID = -1, /* NULL ptr with n > 0, unknown dtype/algo, misaligned
                               ptr (4 B for U32, 8 B for U64/F64, 16 B otherwise),
                               n >= 2^32, bad option                               */
    IPS4O_ERR_NOMEM = -2,   /* device scratch (or pinned host) allocation failed  */
    IPS4O_ERR_CUDA = -3,    /* a CUDA launch or runtime call failed, or (calls that
                               synchronise) the device reported an error flag; the
                               text is kept for ips4o_status_string()              */
    IPS4O_ERR_NOGPU = -4    /* no CUDA device / device is not sm_100             */
};

/* Options of ips4o_sort_ex (NULL = defaults).  Zero in a field = default. */
typedef struct ips4o_options {
    int32_t algo;          /* enum ips4o_algo (default TREE)                          */
    int32_t k_max;         /* max leaves/digits per partitioning step (k=256),
                              power of two in [2, 256] ([4, 256] for TREE: >= 3
                              splitters guarantee progress); default per dtype       */
    uint64_t seed;         /* sampling seed (DESIGN R8); default 0x1F4A2C7            */
    int32_t alpha_min;     /* lower bound of the oversampling factor alpha; the paper
                              uses alpha = 0.2 log2 n, default max(that, 64) */
    int32_t base_cap;      /* base-case capacity M (elements per one-CTA sort);
                              default and maximum per dtype (DESIGN "Base case")      */
    int32_t max_levels;    /* stop after this many partitioning levels (debug);
                              0 = unlimited.  With a limit the array is PARTITIONED,
                              not sorted, unless all buckets reached the base case.  */
    int32_t skip_prepass;  /* 1 = do not run the easy-input pre-pass   */
    int32_t skip_basecase; /* 1 = do not run the base case (debug; leaves buckets
                              unsorted)                                               */
    int32_t timing;        /* 1 = record per-kernel device times into ips4o_stats
                              (device globaltimer stamps per kernel; needs `out`)    */
    int32_t arena_mb;      /* level arena in MiB (0 = sized for the first two levels;
                              at least the root level's plan); a level that does not
                              fit runs in several rounds                            */
    int32_t reserved[6];
} ips4o_options;

#define IPS4O_MAX_LEVELS_REPORTED 16
#define IPS4O_NUM_KERNELS 12

/* Statistics (optional output of ips4o_sort_ex; a non-NULL pointer implies a
 * stream synchronisation before return). */
typedef struct ips4o_stats {
    uint64_t scratch_bytes;           /* device scratch allocated by this call        */
    int32_t levels;                   /* partitioning rounds executed (= levels unless
                                         the arena deferred tasks to a later round)   */
    int32_t easy_input;               /* 0 none, 1 sorted, 2 reverse-sorted (reversed),
                                         3 all keys equal                             */
    uint64_t tasks_per_level[IPS4O_MAX_LEVELS_REPORTED];
    uint64_t elems_per_level[IPS4O_MAX_LEVELS_REPORTED]; /* sum of task sizes      */
    uint64_t basecase_tasks;          /* number of one-CTA base-case sorts            */
    uint64_t basecase_elems;          /* elements sorted by the base case             */
    uint64_t equal_elems;             /* elements left in terminal equality buckets   */
    float kernel_ms[IPS4O_NUM_KERNELS]; /* per kernel family, when opt->timing, summed
                                         over launches (earliest CTA start to latest
                                         warp end, device globaltimer):
                                         0 prepass (+ entry), 1 sample (+ IPS2Ra range
                                         measure), 2 classify, 3 boundaries + schedule,
                                         4 stripe-fix, 5 permute, 6 cleanup, 7 unused
                                         (the scheduler runs inside 3), 8 base case,
                                         9 reverse, 10 device planner, 11 total device
                                         time of the sort (first start to last end)   */
    uint64_t kernel_launches;         /* kernels launched by this call (round 0 by the
                                         host, the rest by the device planner)        */
    uint64_t deferred_tasks;          /* tasks a round deferred because the arena was
                                         full (they ran in a later round)             */
    float round_kernel_ms[IPS4O_MAX_LEVELS_REPORTED][4]; /* per round, when opt->timing:
                                         0 classify, 1 permute, 2 base case (+ split),
                                         3 every other kernel of the round            */
} ips4o_stats;

/* Sort the n elements at DEVICE pointer ptr ascending, in place, unstably,
 * stream-ordered on `stream` (a cudaStream_t, or NULL for the legacy default
 * stream).  ptr alignment: 4 B (U32), 8 B (U64, F64), 16 B (PAIR, REC100,
 * QUARTET).  The caller owns ptr and keeps it alive until the stream work
 * completes.
 * Asynchronous like a kernel launch: the call enqueues a stream-ordered
 * scratch allocation (from a memory pool the library owns per device), ONE
 * kernel, and the scratch free, and returns; every partitioning level is
 * planned and launched by the device (recursion on the device, P:1119-1163,
 * DESIGN "Device planner").  The enqueued work can be captured into a CUDA
 * graph (stream capture) once the device has been initialised by an earlier
 * call (the first call per device creates the pool and a status word).
 * Errors: IPS4O_ERR_INVALID, IPS4O_ERR_NOMEM, IPS4O_ERR_CUDA, IPS4O_ERR_NOGPU
 * are returned for what the host can see; an error the device detects later
 * (an internal invariant) is ORed into the device's status word
 * (ips4o_device_status) and reported by the synchronising calls.
 * n <= 1 returns 0 without device work. */
int ips4o_sort(void *ptr, uint64_t n, int dtype, void *stream);

/* As ips4o_sort with options (NULL = defaults) and optional statistics
 * (non-NULL `out` synchronises `stream` and reads the device's control block
 * back; such a call is not capturable). */
int ips4o_sort_ex(void *ptr, uint64_t n, int dtype, void *stream,
                  const ips4o_options *opt, ips4o_stats *out);

/* End-to-end call on HOST memory: copies host_ptr[0..n) to the device (through
 * pinned staging), sorts it with ips4o_sort_ex, copies the result back into
 * host_ptr, and synchronises.  host_ptr needs 16-byte alignment; if it is
 * already page-locked (cudaHostAlloc/cudaHostRegister) it is used directly.
 * Device memory for the array is allocated and freed inside the call. */
int ips4o_sort_host(void *host_ptr, uint64_t n, int dtype,
                    const ips4o_options *opt, ips4o_stats *out);

/* The device scratch bytes ips4o_sort_ex allocates for (n, dtype, opt)
 * ("the scratch bytes are reported"): a control block, two task lists of
 * n/(M+1)+2 records, and the level arena sized for the first two levels
 * (O(G*k*b*D) per level plus 3 bytes per block; larger levels run in
 * several rounds instead of growing it). */
uint64_t ips4o_scratch_bytes(uint64_t n, int dtype, const ips4o_options *opt);

/* Error flags device code raised on `device` since the last clear (bit 0
 * cleanup invariant, 1 task-list overflow, 2 a task without progress, 3 a
 * device-side launch failure, 4 arena too small for one task).  Read it after
 * synchronising the streams that ran sorts.  clear != 0 resets it. */
int ips4o_device_status(int device, uint32_t *flags, int clear);

/* Return the library's pooled scratch memory on `device` to the driver. */
int ips4o_release_memory(int device);

/* Human-readable text of a status code (for IPS4O_ERR_CUDA: the last CUDA
 * error string seen by this thread). */
const char *ips4o_status_string(int status);

/* Per-dtype parameters the library uses (for tests and reports). */
typedef struct ips4o_dtype_info {
    int32_t elem_bytes;    /* D                                                      */
    int32_t block_elems;   /* b: elements per block (DESIGN "H1")     */
    int32_t kidx_max;      /* bucket indices per CTA (buffer blocks in shared memory)*/
    int32_t base_cap;      /* base-case capacity M                                   */
    int32_t key_bytes;     /* bytes of a key in ips4o_step_info arrays (8 or 16)      */
} ips4o_dtype_info;
int ips4o_get_dtype_info(int dtype, ips4o_dtype_info *out);

/* ---------------------------------------------------------------- distributed samplesort
 * The three local steps of the multi-GPU samplesort (the paper
 * names IPS4o as the local step of distributed-memory sorting, P:3952-3953;
 * the splitter rule is the paper's own).  One process per GPU;
 * the exchange of samples and buckets between the GPUs is NCCL's (the Python
 * package paper_2009_13569_b200.distributed composes the calls):
 *   1. ips4o_sample              m samples of the local shard;
 *   2. (all-gather of the samples) ips4o_select_splitters: p - 1 splitters;
 *   3. ips4o_partition_splitters in-place partition of the shard into p ranges;
 *   4. (all-to-all of the ranges) ips4o_sort of the received elements.
 *
 * ips4o_sample: writes m elements of the DEVICE array ptr[0..n) to DEVICE
 * pointer out[0..m): out[j] = ptr[i_j] with i_j the counter-based draw of
 * DESIGN R8 for the task (level 0, begin 0, size n) and `seed` (use a
 * different seed per rank).  Sampling with replacement.
 * Asynchronous on `stream`.  ptr and out need 4-byte alignment.
 * Errors: IPS4O_ERR_INVALID (unknown dtype, n = 0 with m > 0, NULL pointers);
 * m = 0 does nothing. */
int ips4o_sample(const void *ptr, uint64_t n, int dtype, void *stream,
                 uint64_t m, uint64_t seed, void *out);

/* ips4o_select_splitters: sorts the DEVICE array samples[0..total) in place
 * (ips4o_sort) and writes the parts - 1 equidistant picks
 * out[j] = samples[((j + 1) * total) / parts - 1], j < parts - 1, to DEVICE
 * pointer out.  Asynchronous.  parts = 1 does nothing; total < parts is
 * IPS4O_ERR_INVALID. */
int ips4o_select_splitters(void *samples, uint64_t total, int dtype, void *stream,
                           int parts, void *out);

/* ips4o_partition_splitters: partitions the DEVICE array ptr[0..n) in place
 * into nspl + 1 ranges by the nspl given splitters S_0 <= ... <= S_{nspl-1}
 * (DEVICE pointer, elements of `dtype`, sorted ascending by key): range r =
 * [bounds[r], bounds[r+1]) holds the elements e with S_{r-1} < e <= S_r (S_-1
 * = -inf, S_nspl = +inf; the bucket rule of P:392-394).  One partitioning
 * step (sampling replaced by the given splitters; branchless tree with
 * equality buckets when splitters repeat, block permutation, cleanup; no
 * recursion), so each range is NOT sorted.  bounds is a HOST array of
 * nspl + 2 uint64.  Synchronous (the caller needs the range sizes for the
 * exchange).  1 <= nspl <= kidx_max/2 - 1 (127 for 8/16-byte elements).
 * Errors: IPS4O_ERR_INVALID (bad arguments, splitters not sorted),
 * IPS4O_ERR_NOMEM, IPS4O_ERR_CUDA. */
int ips4o_partition_splitters(void *ptr, uint64_t n, int dtype, void *stream,
                              const void *splitters, int nspl, uint64_t *bounds);

/* ---------------------------------------------------------------- test hooks
 * One partitioning step (Sec. 4.1: sampling, classification,
 * block permutation, cleanup) over the whole array A[0..n), with NO recursion
 * and no base case.  Afterwards A is partitioned into buckets
 * [E[j], E[j+1]), j < num_buckets.  The classifier actually used is returned
 * in raw KEY form (not the internal order-preserving form):
 *   key_bytes = 8 : U64/PAIR key as uint64, F64 as the double's bit pattern;
 *   key_bytes = 16: REC100 key bytes 0..9 followed by 6 zero bytes.
 * tree[1..s] / splitter[0..s] with s = 2^l - 1 (tree[0] unused, zero) follow
 * P:402-406.  For IPS4O_ALGO_DIGIT, tree/splitter are untouched and
 * `shift`, `l` (= digit bits) describe the extractor (key >> shift) & (2^l - 1)
 * over the order-preserving 64-bit (or 80-bit) key; with lut_log = M > 0 the
 * sample-adaptive extractor (DESIGN R33) is in use instead: the
 * bucket of a key is the logarithmic digit of (key - smallest key of A) with
 * M mantissa bits (offsets below 2^(M+1) map to themselves, every octave
 * above to 2^M equal slots), shift = 0.
 * Host arrays are caller-owned: E needs room for kidx_max+1 uint64,
 * tree and splitter for kidx_max keys of key_bytes each.  Synchronous. */
typedef struct ips4o_step_info {
    int32_t algo;
    int32_t num_buckets;   /* K: bucket indices (2^l, or 2^(l+1) with equality)   */
    int32_t l;             /* log2 leaves (tree) / digit bits (radix)             */
    int32_t equality;      /* equality buckets enabled                */
    int32_t shift;         /* radix shift (DIGIT)                                 */
    int32_t k_req;         /* k requested by the level planner (power of two)     */
    int32_t k_used;        /* k after the equality budget rule (DESIGN R10)       */
    int32_t samples;       /* m = alpha * k samples drawn (TREE)                  */
    int32_t kidx_budget;   /* bucket-index budget of the equality rule (R10)      */
    int32_t level;         /* sampling level argument (0 here)                    */
    uint64_t seed;         /* seed used                                           */
    uint64_t *E;           /* [num_buckets + 1] exact bucket boundaries (out)     */
    void *tree;            /* [2^l] keys (out, TREE)                              */
    void *splitter;        /* [2^l] keys (out, TREE)                              */
    int32_t lut_log;       /* lookup table of starting leaves (TREE, keys <= 16 B):
                              0 = linear slots, M > 0 = logarithmic slots with M
                              mantissa bits (DESIGN "Classification"); DIGIT:
                              M > 0 = logarithmic digit (see above)             */
    int32_t reserved0;
} ips4o_step_info;
int ips4o_partition_step(void *ptr, uint64_t n, int dtype, void *stream,
                         const ips4o_options *opt, ips4o_step_info *info);

/* Classify n elements at DEVICE pointer elems with the branchless tree of
 * P:432-437 built from the u sorted, unique splitter keys at HOST pointer
 * splitters (raw key form, key_bytes each); equality buckets if `equality`.
 * Writes one uint32 bucket index per element to DEVICE pointer out.  This is
 * the device tree walk (Alg. 1) that the record/quartet classifier runs and
 * that the 4/8/16-byte classifier's lookup table of starting leaves
 * must agree with -- parity of whole partition steps checks the
 * latter (test hook).  Synchronous. */
int ips4o_classify(const void *elems, uint64_t n, int dtype, const void *splitters,
                   int u, int equality, uint32_t *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* IPS4O_H */
