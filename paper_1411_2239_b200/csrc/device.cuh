// device.cuh -- shared device-side definitions for the sm_100a kernels.
//
// Hot path of arXiv:1411.2239 Alg. 1:
//   a1 epsilon + a2 SortTrace  -> stable hash(k0) partition   (kernels.cu: part_*)
//   a3 SpawnMonitors / dedup   -> shared-memory hash per bucket (bucket kernels)
//   a4 Distribute/UpdateMonitor-> delta table in smem, lane / warp per leaf
//   a5 ApplyQuantifiers        -> per-level grouping + Def. 6 rule, integer only
//   a6 result                  -> finalize kernel
#pragma once
#include <cstdint>

namespace ltl4c {

constexpr int kMaxLevels = 3;
constexpr int kMaxFormulas = 4;
constexpr int kMaxStates = 16;
constexpr int kMaxLetters = 256;
constexpr uint32_t kAbsent = 0xFFFFFFFFu;

// Program tables as the kernels read them (one copy in device memory).
struct DevProg {
  uint32_t nf, nl, na, nq, q0;
  uint32_t pad;
  uint64_t map[kMaxLetters];                // packed nibble map q -> delta[q][a]
  uint8_t delta[kMaxStates][kMaxLetters];   // delta[q][a]
  uint8_t lab[kMaxFormulas][kMaxStates];    // lambda_f(q) in B6 codes
  int32_t qkind[kMaxFormulas][kMaxLevels];
  int32_t qcmp[kMaxFormulas][kMaxLevels];
  uint64_t qnum[kMaxFormulas][kMaxLevels];
  uint64_t qden[kMaxFormulas][kMaxLevels];
};

// Accumulators of one verify / of the carried online state (device memory).
// hist[f][l][v] = # depth-l nodes of formula f with verdict v (signed deltas
// are applied as two's-complement adds in online mode).
struct DevAcc {
  unsigned long long hist[kMaxFormulas][kMaxLevels + 1][6];
  unsigned long long events_seen;
  unsigned long long events_bound;
  unsigned long long medium_buckets;
  unsigned long long large_buckets;
  unsigned long long oversize_buckets;
  unsigned long long oversize_events;
  unsigned long long table_overflow;
  unsigned long long leaves;  // distinct leaves inserted in the carried table
  unsigned long long nodes[kMaxLevels + 1];
  unsigned long long onepass;  // K = 1 hot batch in one-pass mode (seg.cu: bucket_coarse)
};

// Result as written by the finalize kernel (mirrors ltl4c_result, per formula).
struct DevResult {
  int32_t verdict;
  uint32_t n_levels;
  unsigned long long hist[kMaxLevels + 1][6];
  unsigned long long events_seen;
  unsigned long long events_bound;
};

__host__ __device__ inline uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

// bucket of an event: top `bits` bits of a hash of its level-0 key
constexpr uint32_t kBucketSalt = 0x9e3779b9u;
constexpr uint32_t kOwnerSalt = 0x5bd1e995u;  // multi-GPU owner rank (independent of buckets)
__host__ __device__ inline uint32_t salted_bucket(uint32_t k0, int bits, uint32_t salt) {
  return bits == 0 ? 0u : fmix32(k0 ^ salt) >> (32 - bits);
}
__host__ __device__ inline uint32_t bucket_of(uint32_t k0, int bits) { return salted_bucket(k0, bits, kBucketSalt); }

// Def. 6 node verdict from the child histogram (readings A1-A3, A9; DESIGN.md
// "Node rule").  Integer only: A compares count*den ~ num*N (num/den reduced,
// den <= 10^6, N < 2^40 -> products < 2^60).
__host__ __device__ inline bool cmp_u64(int cmp, unsigned long long a, unsigned long long b) {
  switch (cmp) {
    case 0: return a < b;
    case 1: return a <= b;
    case 2: return a > b;
    case 3: return a >= b;
    default: return a == b;
  }
}

template <class C>
__host__ __device__ inline int node_verdict(int kind, int cmp, unsigned long long c,
                                            unsigned long long den, const C *h) {
  unsigned long long N = 0, up[6];
  unsigned long long run = 0;
  for (int v = 5; v >= 0; --v) { run += (unsigned long long)h[v]; up[v] = run; }
  N = run;
  auto S = [&](int t) {  // constraint on the up-set {v >= t} (Eq. S)
    return kind == 0 ? cmp_u64(cmp, up[t] * den, c * N) : cmp_u64(cmp, up[t], c);
  };
  const unsigned long long h0 = (unsigned long long)h[0], h5 = (unsigned long long)h[5];
  // permanence (forall-v clauses, Table 1 P:703-713 for E; P:690 and the same
  // argument for A): only h0 (#F children) and h5 (#T children) are permanent.
  bool top, bot;
  if (kind == 1) {
    top = (cmp == 2 && h5 > c) || (cmp == 3 && h5 >= c);
    bot = (cmp == 4 && h5 > c) || (cmp == 0 && h5 >= c) || (cmp == 1 && h5 > c);
  } else {
    const bool one = (c == den), zero = (c == 0);
    top = (cmp == 3 && zero) || (cmp == 1 && one) || (cmp == 2 && zero && h5 >= 1) ||
          (cmp == 0 && one && h0 >= 1);
    bot = ((cmp == 4 || cmp == 3) && one && h0 >= 1) || ((cmp == 4 || cmp == 1) && zero && h5 >= 1) ||
          (cmp == 2 && one) || (cmp == 0 && zero);
  }
  if (top && S(5)) return 5;
  if (bot && !S(1)) return 0;
  if (S(4)) return 4;
  if (S(3)) return 3;
  if (S(2)) return 2;
  return 1;
}

}  // namespace ltl4c
