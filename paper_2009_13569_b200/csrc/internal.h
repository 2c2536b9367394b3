// internal.h -- data structures shared by the host driver and the kernels.
// Product code: never includes anything from oracle/.
#pragma once
#include <cstdint>

namespace ips4o {

typedef unsigned long long u64;
typedef unsigned int u32;
typedef long long i64;
typedef unsigned __int128 u128;

enum { DT_U64 = 0, DT_F64 = 1, DT_PAIR = 2, DT_REC100 = 3, DT_U32 = 4, DT_QUARTET = 5 };
constexpr int KEY_WORDS = 3;  // internal keys up to 192 bits (Quartet), [0] = least significant
enum { ALGO_TREE = 0, ALGO_DIGIT = 1 };

// Flags of a task.
enum : u32 {
  TF_NONE = 0,
  TF_LOOSE = 1,   // [lo, hi] are valid bounds but may be loose (the root when the
                  // pre-pass was skipped: [0, max]; K6 passes the flag on to the
                  // children whose bound is the parent's); the base case measures
                  // the exact key range of such a bucket before taking its digit
  TF_MEASURE = 2, // DIGIT: the parent's digit left more than half of it in this
                  // bucket; K0m measures the exact key range before the digit setup
};

// A task T[l, r): the subarray [begin, begin+size) of the input, with
// inclusive bounds [lo, hi] on its keys in the internal order-preserving key
// space (u64 for U64/F64/PAIR, 80-bit for REC100; stored as two u64 words).
struct TaskDesc {
  u64 begin;
  u64 size;
  u64 lo[KEY_WORDS];  // [0] = low 64 bits, [1], [2] = higher bits
  u64 hi[KEY_WORDS];
  u32 level;
  u32 flags;
};

// Per-task record of one partitioning level.  The host fills the plan part;
// the kernels fill the result part.
struct LevelTask {
  TaskDesc t;
  // ---- plan (host)
  u32 k_req;         // requested leaves (TREE) / max digits (DIGIT), power of 2
  u32 kidx;          // capacity of this task's per-bucket arrays (>= K)
  u32 m;             // samples to draw (TREE), m = alpha * k_req
  u32 stripe_first;  // first stripe of this task in the level's stripe list
  u32 nstripes;
  u32 perm_first;    // first permute CTA
  u32 nperm;         // permute CTAs
  u32 pad0;
  u64 stripe_elems;  // elements per stripe (multiple of b); last stripe shorter
  u64 bucket_off;    // offset (in bucket slots) into per-task-bucket arrays
  u64 blk_off;       // offset (in block slots) into the level's read-done flags
  u64 sbk_off;       // offset (in stripe-bucket slots) of this task's first stripe;
                     // stripe s uses slots [sbk_off + (s - stripe_first) * kidx, +kidx)
  // ---- results (device)
  u32 K;             // number of bucket indices of the classifier
  u32 l;             // log2(leaves) (TREE) or digit bits (DIGIT)
  u32 equality;      // equality buckets on (TREE)
  int shift;         // digit shift (DIGIT)
  u32 k_used;        // k after the equality-budget rule (DESIGN R10)
  u32 lut_log;       // lookup-table slot mapping: 0 linear, M > 0 logarithmic (lut_slot_of)
  u64 lut_lo[KEY_WORDS];  // key range of the sample (TREE); after K1: the first key of
  u64 lut_hi[KEY_WORDS];  // the lookup table's slot 1 grid (llo) and the sample maximum
  u32 lut_ls;             // lookup table (K1 builds it once per task): slot of key x =
  u32 lut_n;              //   min((x - llo) >> lut_ls, lut_n - 1) (x >= llo), else 0
  u32 lut_span;           // the table spans the task's bounds (no clamping needed)
  u32 lut_bits;           // the table has 2^lut_bits slots (planner: from the bucket count)
  u64 lut_off;            // its offset (in slots) in the level's table array
};

// Device pointers of one level's scratch arrays (all in one arena).
struct LevelArgs {
  char *base;                 // the input array
  LevelTask *tasks;           // [ntasks]
  u32 ntasks;
  u32 nstripes;
  u32 nperm;                  // permute CTAs in total
  u32 algo;
  const u32 *stripe_task;     // [nstripes] -> task index
  const u32 *perm_task;       // [nperm] -> task index
  void *trees;                // [ntasks][2][KIDX] keys (tree | splitter)
  unsigned short *luts;       // [lut_off + q] lookup tables of starting leaves (K1 -> K2)
  u32 *counts;                // [stripe-bucket slot] elements per bucket per stripe
  u32 *pfill;                 // [stripe-bucket slot] elements left in partial buffers
  u32 *pcum;                  // [stripe-bucket slot] exclusive prefix over the task's stripes of pfill
  u32 *ptot;                  // [bucket_off + j] partial-buffer elements of bucket j (all stripes)
  u32 *fullblocks;            // [nstripes] full blocks flushed per stripe
  u32 *fcum;                  // [nstripes] exclusive prefix of fullblocks within the task
  char *partials;             // [stripe-bucket slot][b*D] partial buffer contents
  u64 *E;                     // [bucket_off + j], j <= K: exact boundaries (relative)
  u32 *fblk;                  // [bucket_off + j]: full block POSITIONS in region j after
                              // classification (blocks of any bucket)
  u64 *wr;                    // [bucket_off + j] * 8 words: packed (w, r) at [0], readers at [4]
  char *overlap;              // [bucket_off + j][b*D] saved overlaps (cleanup phase a)
  char *overflow;             // [ntasks][b*D] overflow blocks
  u32 *ovf_used;              // [ntasks] bucket that wrote the overflow block, or ~0
  unsigned char *rdone;       // [blk_off + x] block x of the task has been read (K4)
  unsigned short *bid;        // [blk_off + x] bucket of the full block at x (K2 writes,
                              // K3 moves with the block, K4 reads)
  u32 *task_done;             // [ntasks] no block of the task can be fetched any more (K4)
  // scheduler outputs
  TaskDesc *next_tasks;       // pending list of the next round (tasks of the next level)
  u32 *next_count;            // its length (atomic append; the planner preset it to the
                              // number of tasks it deferred, DESIGN "Device planner")
  TaskDesc *base_tasks;       // base-case tasks of this level
  TaskDesc *split_tasks;      // base-case tasks of M < size <= 2M (split in two passes)
  u32 *counters;              // [1] base count, [8] split count (per round); [2..3] equal
                              // elems, [6..7] base elems (whole sort)
  u32 *err;                   // error flags of the sort (ERR_*), never cleared
  unsigned long long *tslot;  // device timing slots of this round [KS_COUNT][2] or null
  u32 next_cap;
  u32 base_cap_tasks;
  u32 capture;                // test hook ips4o_partition_step: no scheduling
  u32 bc_grid;                // base-case CTAs
  void *ctl;                  // the sort's control block (SortCtl, k_plan.cuh)
  const u32 *go;              // round 0 (host-launched): run only if *go != 0 (not an easy input)
  u32 stages;                 // bit s set: stage s of this round runs (enum Stage)
  u32 nmparts, nmtasks;       // K0m parts and tasks of this round (IPS2Ra)
  u64 base_cap_elems;         // base-case capacity M (elements)
  u64 base_split_elems;       // buckets up to this size go to the base case (2M when it can split)
  char *bc_scratch;           // K7 split scratch: [grid][M] items
  u64 seed;
  u32 dbg_one_agent;          // debug: a single permutation agent per task
  u32 sample_p;               // K1 shared layout: sample slots (pow2 >= every task's m)
  const u32 *measure_part;    // [2 * nmeasure_parts]: task, part | nparts << 16 (K0m)
  const u32 *measure_task;    // [3 * nmeasure]: task, first part, nparts (K0m)
  void *measure_out;          // [nmeasure_parts] PrepassPart: per-part key min/max
  // count-first finish of narrow-range key-only tasks (k_count.cuh; K6 appends)
  TaskDesc *count_tasks;      // [count_cap] tasks (counters[9] appended this round)
  u32 *count_off;             // [count_cap] offset of the task's counters in count_hist
  u32 *count_hist;            // [CNT_POOL] per-value counts (counters[10] reserved)
  u32 *count_pre;             // [count_cap + 1] exclusive prefix of the tasks' chunk counts
  u32 *count_work;            // [2] work counters of K9b, K9c
  u32 count_cap;
  u32 count_grid;             // persistent CTAs of K9b / K9c
  const char *ext_spl;        // round 0 of ips4o_partition_splitters: the given splitters
                              // (ext_n elements, sorted) replace the sample's picks
  u32 ext_n;
  u32 pad_ext;
};

// The packed per-bucket permutation word: high 32
// bits = write pointer w (block index), low 32 bits = read pointer r + RBIAS
// (r is the inclusive index of the last unprocessed block; it may fall below
// w by at most the number of agents, hence the bias).
constexpr u64 RBIAS = 1ull << 31;
#ifndef IPS4O_WR_STRIDE
#define IPS4O_WR_STRIDE 4  // one 32-byte sector per bucket (8: 6.50 ms, 4: 6.37 ms, 16: 6.90 ms permute at 2^30)
#endif
constexpr int WR_STRIDE = IPS4O_WR_STRIDE;  // u64 words per bucket slot: [0] = packed (w, r), [1] = prefix end

// Error flags a sort can raise on the device (SortCtl::error, and the
// per-device status word behind ips4o_device_status).
enum : u32 {
  ERR_CLEANUP = 1,        // cleanup invariant: holes != overlap + partial buffers
  ERR_LIST_OVERFLOW = 2,  // a task list was full (cannot happen with the planner's bounds)
  ERR_NO_PROGRESS = 4,    // a child task equal to its parent (dropped, never looped on)
  ERR_LAUNCH = 8,         // a device-side kernel launch failed
  ERR_ARENA = 16,         // a single task does not fit the level arena
  ERR_CHECK = 32,         // checked build (IPS4O_CHECKS): an index failed its bounds check
};

// Device timing slots (globaltimer, ns) per round: [slot][0] = earliest CTA
// start, [slot][1] = latest warp end.  Host folds them into kernel families.
enum KSlot {
  KS_PRESAMPLE = 0, KS_PREPASS, KS_PREREDUCE, KS_MEASURE, KS_MEASURE_RED, KS_SAMPLE, KS_CLASSIFY,
  KS_BOUND, KS_FIX, KS_PERM, KS_CSAVE, KS_CFILL, KS_BASE, KS_SPLIT, KS_REV, KS_PLAN, KS_NARROW, KS_COUNT
};

// The kernels of one round, in launch order (k_plan.cuh launch_stage).
enum Stage {
  ST_MEAS = 0, ST_MEASRED, ST_SAMPLE, ST_CLASSIFY, ST_BOUND, ST_FIX, ST_PERM, ST_CSAVE, ST_CFILL, ST_CSETUP,
  ST_CCOUNT, ST_CWRITE, ST_BASE, ST_SPLIT, ST_NEXT, ST_N
};

struct PrepassOut {
  u32 nondecreasing;  // all adjacent pairs a[i] <= a[i+1]
  u32 nonincreasing;  // all adjacent pairs a[i] >= a[i+1]
  u64 minkey[KEY_WORDS];
  u64 maxkey[KEY_WORDS];
};

}  // namespace ips4o
