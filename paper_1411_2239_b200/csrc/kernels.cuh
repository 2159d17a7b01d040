// kernels.cuh -- launch parameter blocks and launchers of the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"

namespace ltl4c {

#ifndef LTL4C_PART_THREADS
#define LTL4C_PART_THREADS 512
#endif
constexpr int kPartThreads = LTL4C_PART_THREADS;  // partition CTA: 16 warps (or 32)
constexpr int kTileEv = 8 * kPartThreads;         // events per partition tile: 8 rounds x 32 lanes per warp
constexpr int kMaxDigitBits = 9;     // <= 512 digits per stable partition pass
constexpr int kMaxDigits = 1 << kMaxDigitBits;
constexpr int kMaxPasses = 3;        // bucket bits <= 27
constexpr int kSegW = 256;           // events per heavy-path segment (one warp each)
constexpr int kCap = 2048;           // events per bucket chunk held in shared memory (CTA paths)
constexpr int kBucketThreads = 256;
#ifndef LTL4C_WARP_CAP
#define LTL4C_WARP_CAP 256
#endif
#ifndef LTL4C_UNIT_TARGET
#define LTL4C_UNIT_TARGET 192
#endif
constexpr int kWarpCap = LTL4C_WARP_CAP;        // events per warp-processed unit
#ifndef LTL4C_WARP_CAP_BIG
#define LTL4C_WARP_CAP_BIG 1024
#endif
constexpr int kWarpCapBig = LTL4C_WARP_CAP_BIG;  // events per warp-processed medium bucket
constexpr int kUnitTarget = LTL4C_UNIT_TARGET;  // events per bucket_warp work unit (consecutive buckets)

// The stable LSD partition of a batch by bucket = top `bits` bits of hash(k0)
// (a1 + a2).  Per pass p (digit bits [lo[p], lo[p] + width[p])): count per
// tile, scan per digit, stable scatter.
struct PartPlan {
  const uint32_t *in_key[kMaxLevels];   // the batch (pass 0 input)
  const uint8_t *in_let;
  uint32_t *buf_key[2][kMaxLevels];     // ping-pong outputs
  uint8_t *buf_let[2];
  unsigned long long n;                 // events in the batch
  uint32_t n_tiles;                     // ceil(n / kTileEv)
  int K, bits, passes;
  int n_sms;                            // persistent grids: resident CTAs = n_sms x per-SM occupancy
  int hk;                               // key column hashed for the bucket (0; K-1 in online mode)
  const uint32_t *hcol[2];              // that column in buf_key[0] / buf_key[1]
  const uint32_t *dense_key;            // K = 1 hot path (hot.cu): pass 0 reads the dense cold stream
  const uint8_t *dense_let;             //   (dense_key, dense_let) of *dense_n events
  const unsigned long long *dense_n;    //   instead of the batch
  const uint32_t *dense_flag;           //   when *dense_flag != 0 (some key is hot); null: never
  const uint32_t *skip_flag;            // passes >= 1 do nothing when *skip_flag != 0 (one-pass mode), or null
  uint32_t salt;                        // kBucketSalt (buckets) or kOwnerSalt (ranks)
  int lo[kMaxPasses], width[kMaxPasses];
  uint32_t *digit_hist;                 // [kMaxPasses][kMaxDigits] digit totals (bound events)
  uint32_t *counts;                     // [kMaxDigits][n_tiles] tile counts, scanned in place
  int rank_ballot;                      // stable rank by per-bit ballots instead of match.any
  uint32_t let_mask;                    // (1 << n_atoms) - 1: pass 0 drops letter bits of no atom
  unsigned long long *nvalid;           // bound events of this batch
  DevAcc *acc;
};

__device__ __forceinline__ bool first_dense(const PartPlan &pl) { return pl.dense_flag && *pl.dense_flag; }
__device__ __forceinline__ unsigned long long first_n(const PartPlan &pl) { return first_dense(pl) ? *pl.dense_n : pl.n; }
__device__ __forceinline__ bool pass_skipped(const PartPlan &pl, int pass) { return pass > 0 && pl.skip_flag && *pl.skip_flag; }

// Heavy hitters of single-level properties (hot.cu): the most frequent keys are
// composed in trace order where they lie; only the other events are partitioned.
#ifndef LTL4C_HOT_SLOTS
#define LTL4C_HOT_SLOTS 4096
#endif
constexpr int kHotSlotsMax = LTL4C_HOT_SLOTS;  // hot-table slots (2-way buckets) for 1-byte maps; / 4 for 8-byte maps
#ifndef LTL4C_HOT_SAMPLES
#define LTL4C_HOT_SAMPLES (1 << 18)
#endif
constexpr int kHotSamplesMax = LTL4C_HOT_SAMPLES;  // evenly spaced sample of the batch
constexpr int kHotCountCap = 1 << 20;  // sample-count table slots (at most; 2 x the samples, rounded up)
constexpr int kHotMinCount = 4;        // a hot key was sampled at least this often
constexpr int kHotCtaWarps = 8;
constexpr double kOnePassKeys = 768.0 * 1024;  // cold keys (Chao1 estimate) for the one-pass mode
struct HotParams {
  const uint32_t *k0;                   // the batch's key column (K = 1)
  const uint8_t *let;
  unsigned long long n;
  uint32_t n_samples;
  int mapk;                             // 0: 2-bit packed maps (nq <= 4, <= 16 letters); 1: byte maps (nq <= 8)
  int slots;                            // hot-table slots (hot_slots(mapk))
  uint32_t let_mask;
  uint32_t *cnt_key, *cnt_val;          // [cnt_cap] sample counts (key = ABSENT: empty)
  uint32_t cnt_cap;                     // power of two >= 2 x n_samples
  uint32_t *slot_key;                   // [slots] hot key of each slot (ABSENT: empty) = dense id
  uint32_t *nhot;                       // [0] hot keys, [1] their samples, [2] dense, [3] one pass; [8 + c] keys sampled c times
  void *partial;                        // [n_chunks][slots] per-warp-chunk maps
  uint32_t *cold_key;                   // scratch [n]: chunk c's cold events at its own range
  uint8_t *cold_let;
  uint32_t *dense_key;                  // [n] the cold events in trace order
  uint8_t *dense_let;
  uint32_t *chunk_cold;                 // [n_chunks] cold events per chunk
  uint32_t *chunk_pre;                  // [n_chunks] their exclusive prefix (dense offset)
  unsigned long long *n_cold;           // total cold events (zeroed)
  unsigned long long chunk_ev;          // events per chunk (multiple of 512)
  int n_chunks;                         // warps of hot_compose
  int force_onepass;                    // LTL4C_FORCE_ONEPASS (tests): one-pass mode whatever the estimate
  const DevProg *prog;
  DevAcc *acc;
};

// Carried / per-verify global tables of the global (chunked) bucket path.
struct DevTables {
  uint32_t epoch;
  unsigned long long leaf_cap;          // power of two
  uint4 *leaf_slot;                     // {tag, k0, k1, k2}; tag = epoch << 1 | ready
  uint8_t *leaf_state;
  unsigned long long node_cap[kMaxLevels];
  uint4 *node_slot[kMaxLevels];         // level l in [1, n-1]
  uint32_t *node_verdict[kMaxLevels];   // 4 x u8 packed, 0xFF = none
  uint32_t *node_hist[kMaxLevels];      // [cap][F][6]
  uint32_t *leaf_aux;                   // heavy path: dense leaf id per slot
  uint32_t *node_aux[kMaxLevels];       // heavy path: dense node id per slot
};

// Heavy path (buckets larger than one shared-memory chunk, offline): segments of
// kCap events are processed in parallel; each emits, per leaf, the ordered
// composition of its transition maps (a "partial"); partials are grouped by leaf
// and composed in segment order (the segmented transition-map scan of SURVEY
// §8(a) a4); leaves and nodes are then aggregated through the global tables.
struct HeavyParams {
  const uint32_t *key[kMaxLevels];
  const uint8_t *let;
  const uint32_t *bucket_off;
  const uint32_t *list;                 // oversize buckets
  const unsigned long long *list_len;
  const DevProg *prog;
  DevAcc *acc;
  DevTables tab;
  uint32_t *seg_base;                   // [list_len + 1]
  uint32_t *ctr;                        // [8] work counters (zeroed)
  uint4 *part;                          // {dense leaf, segment item, map lo, map hi}
  unsigned long long *n_part;
  unsigned long long *n_leaves;
  uint32_t *leaf_slot_of;               // dense leaf -> table slot
  uint32_t *leaf_npart;                 // [dense] (zeroed)
  uint32_t *leaf_off;                   // [dense] exclusive scan of leaf_npart
  uint32_t *leaf_fill;                  // [dense] (zeroed)
  uint4 *lists;                         // partials grouped by leaf
  uint32_t *long_list;                  // dense leaves with > 32 partials
  uint32_t *node_list[kMaxLevels];      // dense node -> slot, per level
  unsigned long long *n_nodes;          // [kMaxLevels]
  uint32_t *scan_tmp;                   // block sums of the leaf_npart scan
  unsigned long long cap_leaves;        // upper bound of dense leaves (host)
};

struct BucketParams {
  const uint32_t *key[kMaxLevels];      // partitioned events (bucket order, stable)
  const uint8_t *let;
  const uint32_t *bucket_off;           // [n_buckets + 1]
  int warps_per_cta;
  uint32_t warp_hdr;                    // warp kernels: CTA header bytes (bucket_warp_hdr)
  uint32_t n_buckets;
  const uint32_t *list;                 // if set: CTA i processes bucket list[i]
  const unsigned long long *list_len;   // number of entries in list
  uint32_t *oversize_list;              // fast path: buckets larger than kCap
  uint32_t *medium_list;                // warp path: buckets larger than kWarpCap
  uint32_t *spill_list;                 // warp paths: buckets that do not fit go here
  unsigned long long *spill_len;
  uint32_t *bucket_counter;             // warp path: dynamic unit scheduler
  const uint32_t *unit_start;           // warp path: [n_units + 1] first bucket of each unit
  uint32_t n_units;                     // for the batch's N events (host)
  uint32_t unit_target;                 // events per unit (unit_start's target)
  const uint32_t *gate;                 // K = 1 hot batches: the kernel runs iff (*gate != 0) == gate_want
  int gate_want;
  const uint32_t *coarse_hist;          // one-pass mode: the first pass's digit totals (coarse bucket sizes)
  const unsigned long long *nvalid;     // bound events (device): units past nvalid / kUnitTarget + 1 are empty
  const DevProg *prog;
  DevAcc *acc;
  DevTables tab;
};

// Online mode: the bucket parameters plus the per-batch touched-node lists.
struct OnlineParams {
  BucketParams b;
  uint32_t bid;                         // batch id (!= 0), the touch mark of this batch
  const uint32_t *bid_dev;              // if set: the batch id is read here (graph replays: set per batch)
  uint32_t *tlist[kMaxLevels];          // touched node slots per depth (capacity node_cap)
  uint32_t *tcnt;                       // [kMaxLevels] entries in tlist (zeroed per batch)
};

// Everything the host reads back after a verify (one D2H copy).
struct DevOut {
  DevResult res[kMaxFormulas];
  unsigned long long oversize_buckets, oversize_events, table_overflow, leaves;
  unsigned long long nodes[kMaxLevels + 1];
  unsigned long long onepass;           // the batch took the one-pass mode (oversize buckets are coarse)
};

struct Launcher {
  cudaStream_t stream;
  void (*before)(void *ctx, int kernel_id);
  void (*after)(void *ctx, int kernel_id);
  void *ctx;
};

enum KernelId {
  kKPartCount = 0,
  kKPartScan,
  kKPartScatter,
  kKBucketBounds,
  kKBucketWarp,
  kKBucketFast,
  kKFinalize,
  kKRehash,
  kKHeavy,
  kKUnitStart,
  kKBucketWarpBig,
  kKOnlineLeaf,
  kKOnlineNodes,
  kKHot,
  kKHotCompose,
  kKNumKernels
};
extern const char *const kKernelNames[kKNumKernels];

cudaError_t launch_part_count(const PartPlan &p, int pass, const Launcher &L);
cudaError_t launch_part_scan(const PartPlan &p, int pass, const Launcher &L);
// a batch of <= kTinyBatch events as ONE bucket: its bound events compacted in trace
// order into the final partition buffers, the bucket offsets (all events in bucket 0)
// and the bound count -- instead of the count / scan / scatter passes and mu
constexpr int kTinyBatch = 256;
cudaError_t launch_tiny_stage(const PartPlan &p, uint32_t *off, uint32_t n_buckets, const Launcher &L);
cudaError_t launch_part_scatter(const PartPlan &p, int pass, const Launcher &L);
cudaError_t launch_bucket_bounds(const PartPlan &p, uint32_t *off, uint32_t n_buckets, const Launcher &L,
                                 const uint32_t *gate = nullptr, int want = 0);
cudaError_t launch_bucket_fast(const BucketParams &p, int K, int nf, int n_sms, const Launcher &L);
cudaError_t launch_unit_start(const uint32_t *off, uint32_t nb, uint32_t *ustart, uint32_t n_units, const Launcher &L,
                              uint32_t target = kUnitTarget, const uint32_t *gate = nullptr, int want = 0);
cudaError_t launch_bucket_warp(const BucketParams &p, int K, int nf, uint32_t grid, const Launcher &L);
// {warps per CTA, CTAs per SM} of the unit kernel (cfg[0..1]) and of the
// medium-bucket kernel (cfg[2..3])
cudaError_t bucket_warp_config(int K, int nf, int nq, int na, int *cfg);
uint32_t bucket_warp_hdr(int nq, int na);  // CTA header bytes of the warp kernels
cudaError_t launch_heavy(const HeavyParams &h, int K, int nf, int nq, int n_sms, const Launcher &L);
cudaError_t launch_online_leaf(const OnlineParams &p, int K, int nf, uint32_t grid, const Launcher &L);
cudaError_t launch_online_nodes(const OnlineParams &p, int nf, int l, uint32_t grid, const Launcher &L);
cudaError_t online_leaf_config(int K, int nf, int nq, int na, int *cfg);  // {warps/CTA, CTAs/SM}
cudaError_t launch_rehash(const DevTables &from, const DevTables &to, int n_levels, int nf,
                          unsigned long long *overflow, const Launcher &L);
cudaError_t launch_finalize(const DevProg *prog, const DevAcc *acc, DevOut *out, const Launcher &L);
cudaError_t launch_set_u32(uint32_t *p, uint32_t v, const Launcher &L);  // *p = v (stream-ordered)
// zero acc (if set), *nvalid and totals[0 .. ntot) (if set) in one launch
cudaError_t launch_reset(DevAcc *acc, unsigned long long *nvalid, uint32_t *totals, int ntot, const Launcher &L);
// K = 1 offline units: segmented map scans through warp tables (seg.cu)
cudaError_t launch_bucket_seg(const BucketParams &p, int nq, int nf, uint32_t grid, const Launcher &L);
int bucket_seg_ctas_per_sm(int nq);
// one-pass mode of a K = 1 hot batch (<= 4 states, <= 16 letters): CTA per coarse bucket (seg.cu)
constexpr int kCoarseBits = 9;
cudaError_t launch_bucket_coarse(const BucketParams &p, int nf, uint32_t grid, const Launcher &L);
int bucket_coarse_ctas_per_sm();

cudaError_t launch_hot_select(const HotParams &hp, const Launcher &L);
cudaError_t launch_hot_compose(const HotParams &hp, const Launcher &L);  // + gather of the cold stream
cudaError_t launch_hot_finish(const HotParams &hp, const Launcher &L);
int hot_ctas_per_sm(int mapk);  // resident hot_compose CTAs
int hot_slots(int mapk);
int hot_map_bytes(int mapk);

}  // namespace ltl4c
