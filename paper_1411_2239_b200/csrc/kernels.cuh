// kernels.cuh -- launch parameter blocks and launchers of the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"

namespace ltl4c {

constexpr int kTileEv = 4096;        // events per partition tile
constexpr int kPartThreads = 256;    // 8 warps x 16 rounds x 32 lanes
constexpr int kMaxDigitBits = 8;     // <= 256 digits per stable partition pass
constexpr int kCap = 2048;           // events per bucket chunk held in shared memory
constexpr int kBucketThreads = 256;
constexpr int kWarpCap = 512;        // events per warp-processed bucket
constexpr int kLeafSlots = 1024;     // warp leaf table (load <= 1/2)
constexpr int kNodeSlots = 512;      // warp node table per inner level (<= 512 nodes: never full)
constexpr int kWarpsPerCta = 4;

// One stable LSD pass of the hash(k0) bucket partition (a2, SortTrace).
struct PartParams {
  const uint32_t *in_key[kMaxLevels];
  const uint8_t *in_let;
  uint32_t *out_key[kMaxLevels];
  uint8_t *out_let;
  unsigned long long n;                 // input events (upper bound)
  const unsigned long long *n_dev;      // if set: input events = min(n, *n_dev)
  int K, bits, lo, width;               // bucket bits; digit = bits [lo, lo + width)
  int first;                            // pass 0: epsilon filter + bucket histogram
  uint32_t n_tiles;
  uint32_t *counts;                     // [1 << width][n_tiles], scanned in place
  uint32_t *totals;                     // [1 << width]
  uint32_t *bucket_count;               // [1 << bits] (pass 0)
  DevAcc *acc;
  unsigned long long *nvalid;           // per-verify count of bound events (pass 0 adds)
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
};

struct BucketParams {
  const uint32_t *key[kMaxLevels];      // partitioned events (bucket order, stable)
  const uint8_t *let;
  const uint32_t *bucket_off;           // [n_buckets + 1]
  uint32_t n_buckets;
  const uint32_t *list;                 // if set: CTA i processes bucket list[i]
  const unsigned long long *list_len;   // number of entries in list
  uint32_t *oversize_list;              // fast path: buckets larger than kCap
  uint32_t *medium_list;                // warp path: buckets larger than kWarpCap
  uint32_t *bucket_counter;             // warp path: dynamic bucket scheduler
  const DevProg *prog;
  DevAcc *acc;
  DevTables tab;
};

// Everything the host reads back after a verify (one D2H copy).
struct DevOut {
  DevResult res[kMaxFormulas];
  unsigned long long oversize_buckets, oversize_events, table_overflow, leaves;
  unsigned long long nodes[kMaxLevels + 1];
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
  kKBucketScan,
  kKBucketFast,
  kKBucketGlobal,
  kKFinalize,
  kKRehash,
  kKBucketWarp,
  kKNumKernels
};
extern const char *const kKernelNames[kKNumKernels];

cudaError_t launch_part_count(const PartParams &p, const Launcher &L);
cudaError_t launch_part_scan(const PartParams &p, const Launcher &L);
cudaError_t launch_part_scatter(const PartParams &p, const Launcher &L);
cudaError_t launch_bucket_scan(const uint32_t *count, uint32_t *off, uint32_t n, const Launcher &L);
cudaError_t launch_bucket_fast(const BucketParams &p, int K, int nf, uint32_t grid, const Launcher &L);
cudaError_t launch_bucket_warp(const BucketParams &p, int K, int nf, uint32_t grid, const Launcher &L);
size_t bucket_warp_smem(int K, int nf);
cudaError_t launch_bucket_global(const BucketParams &p, int K, int nf, uint32_t grid, const Launcher &L);
cudaError_t launch_rehash(const DevTables &from, const DevTables &to, int n_levels, int nf,
                          unsigned long long *overflow, const Launcher &L);
cudaError_t launch_finalize(const DevProg *prog, const DevAcc *acc, DevOut *out, const Launcher &L);

}  // namespace ltl4c
