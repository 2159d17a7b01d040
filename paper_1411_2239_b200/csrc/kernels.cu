// kernels.cu -- sm_100a kernels of the LTL4-C verification hot path.
//
// arXiv:1411.2239, Algorithm 1, re-designed for B200:
//
//  (partition.cu: part_count / part_scan / part_scatter / bucket_bounds --
//      a1 epsilon fused with a2 SortTrace: a stable LSD partition of the bound
//      events by bucket = top bits of hash(k0), so a bucket holds whole level-0
//      subtrees and every slice u^D stays in trace order (reading A15).)
//  unit_start
//      work units = runs of consecutive buckets of ~kUnitTarget events.
//  bucket_fast
//      one CTA per bucket, everything in shared memory:
//        a3 SpawnMonitors: dedup of value vectors (smem hash) = leaves
//        a4 Distribute / UpdateMonitor: each leaf steps the LTL4 monitor delta
//           over its slice in order (Def. 5); lane per short slice,
//           warp per long slice (ordered composition of transition maps)
//        a5 ApplyQuantifiers: level by level, group children by parent prefix
//           (P), histogram B, rule Def. 6
//  bucket_warp / bucket_warp_big
//      warp per work unit (runs of consecutive buckets) with warp-private
//      shared-memory tables; the CTA path above takes what does not fit.
//  heavy
//      oversized buckets: segmented transition-map scan through global tables.
//  online_leaf / online_nodes
//      online mode: carried global tables, verdict deltas propagated
//      level by level through touched nodes.
//  finalize
//      root verdict from the depth-1 histogram, result record.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "util.cuh"

namespace ltl4c {

const char *const kKernelNames[kKNumKernels] = {"part_count", "part_scan", "part_scatter", "bucket_bounds",
                                                "bucket_warp", "bucket_fast",
                                                "finalize", "rehash", "heavy", "unit_start",
                                                "bucket_warp_big", "online_leaf", "online_nodes", "hot", "hot_compose"};

namespace {

// ------------------------------------------------------------------ buckets
struct Smem {
  uint32_t *key[kMaxLevels];  // [kCap] each
  uint8_t *let;               // [kCap]
  uint16_t *cls;              // class of each item
  uint16_t *rep;              // rep event of each class
  uint16_t *item_rep;         // rep event of each item
  uint16_t *htab;             // [2 * kCap]
  uint16_t *owner;            // [kCap]
  uint32_t *scan;             // [kCap + 1]
  uint32_t *cur;              // [kCap + 1]
  uint16_t *perm;             // [kCap]
  uint8_t *state;             // [kCap]
  uint8_t *iv;                // [kMaxFormulas][kCap] item verdicts (new)
  uint8_t *ov;                // [kMaxFormulas][kCap] item verdicts (old, global path)
  uint8_t *nv;                // [kMaxFormulas][kCap] node verdicts
  uint8_t *nov;               // [kMaxFormulas][kCap] node old verdicts (global path)
  uint8_t *delta;             // [kMaxStates * 256]
  unsigned long long *map;    // [256]
  uint8_t *lab;               // [kMaxFormulas * kMaxStates]
  int *acc;                   // [kMaxFormulas][kMaxLevels + 1][6] signed
  uint32_t *misc;             // [64]
};

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Shared-memory plan of a bucket CTA: K key words and nf formulas; the global
// path additionally keeps the old verdicts (ov, nov).
__host__ __device__ inline size_t smem_bytes(int K, int nf, int mode) {
  const bool global = mode == 1;
  const size_t fv = align16((size_t)nf * kCap);
  return align16(sizeof(uint32_t) * kCap) * K + align16(kCap) + 3 * align16(2 * kCap) +
         align16(2 * 2 * kCap) + align16(2 * kCap) + 2 * align16(4 * (kCap + 1)) + align16(2 * kCap) +
         align16(kCap) + (global ? 4 : 2) * fv + align16(kMaxStates * 256) +
         align16(8 * 256) + align16(kMaxFormulas * kMaxStates) +
         align16(4 * kMaxFormulas * (kMaxLevels + 1) * 6) + align16(4 * 64);
}

__device__ Smem carve(uint8_t *base, int K, int nf, int mode) {
  Smem s;
  const bool global = mode == 1;
  uint8_t *p = base;
  auto take = [&](size_t bytes) { uint8_t *r = p; p += align16(bytes); return r; };
  for (int i = 0; i < kMaxLevels; ++i) s.key[i] = i < K ? (uint32_t *)take(sizeof(uint32_t) * kCap) : nullptr;
  s.let = take(kCap);
  s.cls = (uint16_t *)take(2 * kCap);
  s.rep = (uint16_t *)take(2 * kCap);
  s.item_rep = (uint16_t *)take(2 * kCap);
  s.htab = (uint16_t *)take(2 * 2 * kCap);
  s.owner = (uint16_t *)take(2 * kCap);
  s.scan = (uint32_t *)take(4 * (kCap + 1));
  s.cur = (uint32_t *)take(4 * (kCap + 1));
  s.perm = (uint16_t *)take(2 * kCap);
  s.state = take(kCap);
  s.iv = take((size_t)nf * kCap);
  s.nv = take((size_t)nf * kCap);
  s.ov = global ? take((size_t)nf * kCap) : nullptr;
  s.nov = global ? take((size_t)nf * kCap) : nullptr;
  s.delta = take(kMaxStates * 256);
  s.map = (unsigned long long *)take(8 * 256);
  s.lab = take(kMaxFormulas * kMaxStates);
  s.acc = (int *)take(4 * kMaxFormulas * (kMaxLevels + 1) * 6);
  s.misc = (uint32_t *)take(4 * 64);
  return s;
}

template <int K>
__device__ __forceinline__ uint32_t hash_prefix(const Smem &s, int e, int m) {
  uint32_t h = 0x2545F491u;
#pragma unroll
  for (int i = 0; i < K; ++i)
    if (i < m) h = fmix32(h ^ s.key[i][e]) + 0x9e3779b9u * (i + 1);
  return h;
}

template <int K>
__device__ __forceinline__ bool same_prefix(const Smem &s, int a, int b, int m) {
  bool eq = true;
#pragma unroll
  for (int i = 0; i < K; ++i)
    if (i < m) eq &= s.key[i][a] == s.key[i][b];
  return eq;
}

// Group n items (rep event item_rep[i]) by the first m keys of their rep.
// Out: s.cls[i] = dense class id, s.rep[c] = rep event of class c. Returns #classes.
template <int K>
__device__ int dedup(const Smem &s, int n, int m) {
  const int tid = threadIdx.x, nt = blockDim.x;
  constexpr int TS = 2 * kCap;
  for (int i = tid; i < TS; i += nt) s.htab[i] = 0xFFFF;
  __syncthreads();
  for (int i = tid; i < n; i += nt) {
    const int r = s.item_rep[i];
    uint32_t slot = hash_prefix<K>(s, r, m) & (TS - 1);
    while (true) {
      unsigned short old = ((volatile uint16_t *)s.htab)[slot];
      if (old == 0xFFFF) old = atomicCAS(&s.htab[slot], (unsigned short)0xFFFF, (unsigned short)i);
      if (old == 0xFFFF) { s.owner[i] = (uint16_t)i; break; }
      if (same_prefix<K>(s, s.item_rep[old], r, m)) { s.owner[i] = old; break; }
      slot = (slot + 1) & (TS - 1);
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += nt) s.scan[i] = s.owner[i] == i;
  __syncthreads();
  const int C = (int)block_exclusive_scan(s.scan, n, s.misc);
  for (int i = tid; i < n; i += nt)
    if (s.owner[i] == i) s.rep[s.scan[i]] = s.item_rep[i];
  __syncthreads();
  for (int i = tid; i < n; i += nt) s.cls[i] = (uint16_t)s.scan[s.owner[i]];
  __syncthreads();
  return C;
}

// Counting sort of n items by class (C classes): s.perm = items grouped by
// class, s.scan[c] .. s.scan[c+1] = segment of class c.  Unstable.
__device__ void group_by_class(const Smem &s, int n, int C) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int c = tid; c <= C; c += nt) s.scan[c] = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += nt) {  // warp-aggregated: one atomic per (warp, class)
    const int i = i0 + tid;
    const bool act = i < n;
    const uint32_t c = act ? s.cls[i] : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, c);
    const int lead = __ffs(peers) - 1;
    uint32_t base = 0;
    if (act && (tid & 31) == lead) base = atomicAdd(&s.scan[c], (uint32_t)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, lead);
    if (act) s.owner[i] = (uint16_t)(base + __popc(peers & lanemask_lt()));
  }
  __syncthreads();
  block_exclusive_scan(s.scan, C + 1, s.misc);  // scan[C] = n
  for (int i = tid; i < n; i += nt) s.perm[s.scan[s.cls[i]] + s.owner[i]] = (uint16_t)i;
  __syncthreads();
}

// Make every SHORT class segment (<= 32 events) of s.perm ascending (trace
// order, reading A15) by insertion sort.  Long classes are never sorted: their
// transition maps are composed in position order by long_class_map().
__device__ void order_segments(const Smem &s, int n, int C) {
  (void)n;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int c = tid; c < C; c += nt) {
    const int a = s.scan[c], b = s.scan[c + 1];
    if (b - a > 32) continue;
    for (int i = a + 1; i < b; ++i) {
      const uint16_t x = s.perm[i];
      int j = i - 1;
      while (j >= a && s.perm[j] > x) { s.perm[j + 1] = s.perm[j]; --j; }
      s.perm[j + 1] = x;
    }
  }
  __syncthreads();
}

// (g o f) for monitors of at most NQB states (compile-time bound: the loop unrolls,
// and maps of <= 8 states are 32-bit nibble vectors)
template <int NQB>
__device__ __forceinline__ unsigned long long map_apply_t(unsigned long long g, unsigned long long f) {
  if constexpr (NQB <= 8) {
    // byte permutes (PRMT): g's 8 nibbles spread to 8 bytes, f's nibbles (images < 8)
    // are the selectors, the selected bytes packed back to nibbles
    const uint32_t g32 = (uint32_t)g, f32 = (uint32_t)f;
    const uint32_t ge = g32 & 0x0F0F0F0Fu, go = (g32 >> 4) & 0x0F0F0F0Fu;  // nibbles 0,2,4,6 / 1,3,5,7
    const uint32_t glo = __byte_perm(ge, go, 0x5140), ghi = __byte_perm(ge, go, 0x7362);  // g[0..3], g[4..7]
    const uint32_t rlo = __byte_perm(glo, ghi, f32 & 0xFFFFu), rhi = __byte_perm(glo, ghi, f32 >> 16);
    const uint32_t r = __byte_perm(rlo, rhi, 0x6420) | __byte_perm(rlo, rhi, 0x7531) << 4;
    return NQB == 8 ? r : r & ((1u << (4 * NQB)) - 1u);
  } else {
    unsigned long long r = 0;
#pragma unroll
    for (int q = 0; q < NQB; ++q) {
      const int fq = (int)((f >> (4 * q)) & 15ull);
      r |= ((g >> (4 * fq)) & 15ull) << (4 * q);
    }
    return r;
  }
}

__device__ __forceinline__ unsigned long long map_apply(unsigned long long g, unsigned long long f, int nq) {
  // (g o f)[q] = g[f[q]]
  unsigned long long r = 0;
  for (int q = 0; q < nq; ++q) {
    const int fq = (int)((f >> (4 * q)) & 15ull);
    r |= ((g >> (4 * fq)) & 15ull) << (4 * q);
  }
  return r;
}

// One warp: the ordered composition of the transition maps of class c's events
// (events of the chunk are in trace order; lane l takes positions
// [l * P, (l + 1) * P), then the 32 lane maps are composed in lane order).
// Valid in every lane.
__device__ unsigned long long long_class_map(const Smem &s, int n, int c, int nq, unsigned long long ident) {
  const int lane = threadIdx.x & 31;
  const int per = (n + 31) / 32;
  const int lo = min(n, lane * per), hi = min(n, lo + per);
  unsigned long long m = ident;
  for (int i = lo; i < hi; ++i)
    if (s.cls[i] == c) m = map_apply(s.map[s.let[i]], m, nq);
  unsigned long long total = ident;
  for (int l = 0; l < 32; ++l) total = map_apply(__shfl_sync(0xffffffffu, m, l), total, nq);
  return total;
}

// Step every leaf class over its (ordered) segment from start state st0[c]
// (kept in s.state on entry, replaced by the final state).
__device__ void step_leaves(const Smem &s, int C, int nq, int na_letters) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  // short slices: one lane per leaf, delta in shared memory (Def. 5)
  for (int c = tid; c < C; c += nt) {
    const int a = s.scan[c], b = s.scan[c + 1];
    if (b - a > 32) continue;
    int q = s.state[c];
    for (int i = a; i < b; ++i) q = s.delta[q * na_letters + s.let[s.perm[i]]];
    s.state[c] = (uint8_t)q;
  }
  // long slices: one warp per leaf composes the leaf's transition maps in trace
  // order (associativity), then applies the result to the start state
  unsigned long long ident = 0;
  for (int q = 0; q < nq; ++q) ident |= (unsigned long long)q << (4 * q);
  for (int c = wid; c < C; c += nw) {
    if (s.scan[c + 1] - s.scan[c] <= 32) continue;
    const unsigned long long total = long_class_map(s, s.misc[60], c, nq, ident);
    if (lane == 0) s.state[c] = (uint8_t)((total >> (4 * s.state[c])) & 15ull);
    __syncwarp();
  }
  __syncthreads();
}

__device__ void load_prog(const Smem &s, const DevProg *prog) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int A = 1 << prog->na;
  for (int i = tid; i < (int)prog->nq * A; i += nt) s.delta[i] = prog->delta[i / A][i % A];
  for (int i = tid; i < A; i += nt) s.map[i] = prog->map[i];
  for (int i = tid; i < kMaxFormulas * kMaxStates; i += nt) s.lab[i] = prog->lab[i / kMaxStates][i % kMaxStates];
  for (int i = tid; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += nt) s.acc[i] = 0;
}

__device__ __forceinline__ int acc_idx(int f, int l, int v) { return (f * (kMaxLevels + 1) + l) * 6 + v; }

__device__ void flush_acc(const Smem &s, DevAcc *acc, int nf, int nl) {
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) {
    const int v = s.acc[i];
    const int f = i / ((kMaxLevels + 1) * 6), l = (i / 6) % (kMaxLevels + 1), b = i % 6;
    if (v != 0 && f < nf && l >= 1 && l <= nl)
      atomicAdd(&acc->hist[f][l][b], (unsigned long long)(long long)v);
  }
}

template <int K>
__device__ int load_chunk(const Smem &s, const BucketParams &p, uint32_t start, int cnt) {
  if (threadIdx.x == 0) s.misc[60] = (uint32_t)cnt;
  for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
#pragma unroll
    for (int i = 0; i < K; ++i) s.key[i][e] = p.key[i][start + e];
    s.let[e] = p.let[start + e];
    s.item_rep[e] = (uint16_t)e;
  }
  __syncthreads();
  return cnt;
}

// ----------------------------------------------- fast path (offline, fits)
template <int K>
__global__ void __launch_bounds__(kBucketThreads) bucket_fast_kernel(BucketParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  if (blockIdx.x >= *p.list_len) return;  // (uniform per CTA) nothing for this CTA
  const DevProg *prog = p.prog;
  const int nf = prog->nf, nl = prog->nl, nq = prog->nq, A = 1 << prog->na;
  const Smem s = carve(smem_raw, K, nf, 0);
  load_prog(s, prog);
  const int tid = threadIdx.x, nt = blockDim.x;
  const unsigned long long len = *p.list_len;
  for (unsigned long long it = blockIdx.x; it < len; it += gridDim.x) {
    const uint32_t b = p.list[it];
    const uint32_t start = p.bucket_off[b], cnt = p.bucket_off[b + 1] - start;
    if (cnt > (uint32_t)kCap) {
      if (tid == 0) {
        const unsigned long long i = atomicAdd(&p.acc->oversize_buckets, 1ull);
        p.oversize_list[i] = b;
        atomicAdd(&p.acc->oversize_events, (unsigned long long)cnt);
      }
      continue;
    }
    __syncthreads();
    const int n = load_chunk<K>(s, p, start, (int)cnt);
    // a3: leaves = distinct value vectors D of the bucket (Eq. D)
    const int L = dedup<K>(s, n, K);
    group_by_class(s, n, L);
    order_segments(s, n, L);
    // a4: every leaf starts at q0 (offline) and steps over u^D
    for (int c = tid; c < L; c += nt) s.state[c] = (uint8_t)prog->q0;
    __syncthreads();
    step_leaves(s, L, nq, A);
    // leaf verdicts lambda_f (Def. 5) and the depth-n histogram
    for (int c = tid; c < L; c += nt) {
      s.item_rep[c] = s.rep[c];
      for (int f = 0; f < nf; ++f) {
        const uint8_t v = s.lab[f * kMaxStates + s.state[c]];
        s.iv[f * kCap + c] = v;
        atomicAdd(&s.acc[acc_idx(f, nl, v)], 1);
      }
    }
    __syncthreads();
    // a5: ApplyQuantifiers for depth nl-1 .. 1 (depth 0, the root, in finalize)
    int items = L;
    for (int l = nl - 1; l >= 1; --l) {
      const int C = dedup<K>(s, items, l);
      group_by_class(s, items, C);
      for (int x = tid; x < C; x += nt) {
        const int a = s.scan[x], e = s.scan[x + 1];
        for (int f = 0; f < nf; ++f) {
          uint32_t h[6] = {0, 0, 0, 0, 0, 0};
          for (int i = a; i < e; ++i) h[s.iv[f * kCap + s.perm[i]]]++;
          const int v = node_verdict(prog->qkind[f][l], prog->qcmp[f][l], prog->qnum[f][l],
                                     prog->qden[f][l], h);
          s.nv[f * kCap + x] = (uint8_t)v;
          atomicAdd(&s.acc[acc_idx(f, l, v)], 1);
        }
      }
      __syncthreads();
      for (int x = tid; x < C; x += nt) {
        s.item_rep[x] = s.rep[x];
        for (int f = 0; f < nf; ++f) s.iv[f * kCap + x] = s.nv[f * kCap + x];
      }
      __syncthreads();
      items = C;
    }
  }
  flush_acc(s, p.acc, nf, nl);
}

// ----------------------------------------------- warp-per-unit path (offline)
// One warp owns one work unit (a run of consecutive buckets = whole level-0
// subtrees, <= CAP events); no block barriers.  The unit is staged into
// warp-private shared memory with cp.async (16-byte chunks); the NEXT unit is
// resolved one step ahead and its byte ranges are prefetched into L2 with one
// bulk (TMA) prefetch per array.  Events are consumed in windows of 32 x kIlp
// in trace order:
//   a3  every lane find-or-inserts the value vectors of its kIlp events in the
//       warp's leaf table (keys in registers, compared against the staged keys
//       of the slot's representative event); a new leaf resolves its ancestors
//       (depths 1 .. K-1, P) right away in the node tables;
//   a4  a window whose touched slots are all new steps each of them once from
//       q0; otherwise it is replayed as kIlp sub-rounds of 32 in which lanes
//       sharing a slot are grouped (__match_any_sync) and their leader applies
//       the letters in lane order -- every slice u^D is stepped in trace order;
//   a5  leaf verdicts (Def. 5) -> per-node child histograms (B) with
//       per-lane run-length aggregation, then Def. 6 level by level.
// Table slots carry a per-unit epoch (tag = epoch << 16 | rep event + 1), so no
// table is cleared between units.
#ifndef LTL4C_ILP
#define LTL4C_ILP 4
#endif
#ifndef LTL4C_UNIT_BATCH
#define LTL4C_UNIT_BATCH 1  // units taken per atomic by a warp of bucket_warp
#endif
#ifndef LTL4C_STATIC_UNITS
#define LTL4C_STATIC_UNITS 0
#endif
#ifndef LTL4C_LS_MUL
#define LTL4C_LS_MUL 2
#endif
constexpr int kIlp = LTL4C_ILP;         // events per lane per window
// CTA header: sacc [kMaxFormulas][kMaxLevels + 1][6] u32, lab [kMaxFormulas][kMaxStates],
// then delta [nq][2^na] (sized by the program: warp_hdr_bytes)
constexpr int kWarpHdrFixed = 4 * kMaxFormulas * (kMaxLevels + 1) * 6 + kMaxFormulas * kMaxStates;
__host__ __device__ inline uint32_t warp_hdr_bytes(uint32_t nq, uint32_t na) {
  return (uint32_t)align16(kWarpHdrFixed + (size_t)nq * (1u << na));
}

__host__ __device__ constexpr int pow2ceil(int x) { return x <= 1 ? 1 : 2 * pow2ceil((x + 1) / 2); }

template <int K, int NF, int CAP>
struct alignas(16) WarpTab {
  static constexpr int NL = K > 1 ? K - 1 : 1;        // inner levels 1 .. K-1 (index l - 1)
  static constexpr int NSL = pow2ceil(CAP / 4);       // node slots per inner level (claims <= NSL / 2)
  static constexpr int NS = K > 1 ? NSL : 1;
  static constexpr int LS = pow2ceil(LTL4C_LS_MUL * CAP);  // leaf slots (load <= 1/2)
  uint32_t key[K][CAP + 4];             // staged keys; event i at [i + (start & 3)]
  uint8_t let[CAP + 32];                // staged letters; event i at [i + (start & 15)]
  uint32_t ltag[LS];                    // epoch << 16 | rep event + 1 (other epochs = empty)
  uint8_t lnode[K > 1 ? LS : 1];        // depth-(K-1) ancestor slot of the leaf
  uint8_t lstate[LS];                   // state | 0x80 once the leaf's verdict is counted
  int pleaf[NF * 6];                    // pending leaf-verdict deltas of the unit (replayed windows)
  uint32_t ntag[NL][NS];                // as ltag
  uint32_t nhist[NL][NS][NF * 3];       // two u16 counters per word: h[2x] | h[2x+1] << 16
  uint16_t nlist[NL][NS];
  uint16_t npar[NL][NS];                // parent slot (depth l - 1), l >= 2
  uint32_t ncnt[4];                     // claimed node slots per level
  alignas(8) unsigned long long mbar;   // staging barrier (stage_bulk)
};

// TMA bulk staging of a work unit into warp-private shared memory: lane 0 arms
// the warp's mbarrier with the byte count and issues one cp.async.bulk (global ->
// shared, UBLKCP) per key column and one for the letters; every lane then waits on
// the barrier's phase (complete_tx).  Sources are the 16-byte aligned addresses at
// or below the unit's first event: event i lands at key[k][i + (start & 3)] and
// let[i + (start & 15)]; the buffers hold the rounded-up sizes.
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n"
               "fence.mbarrier_init.release.cluster;" ::"r"(smem_u32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *mb, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n"
               "LTL4C_WAIT_%=:\n"
               " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra LTL4C_WAIT_%=;\n}" ::"r"(smem_u32(mb)), "r"(parity) : "memory");
}
template <int K>
__device__ __forceinline__ void stage_bulk(uint32_t *key0, int row, uint8_t *let, const uint32_t *const *gkey,
                                           const uint8_t *glet, uint32_t start, uint32_t cnt,
                                           unsigned long long *mbar, uint32_t &parity) {
  __syncwarp();  // every lane is done with the previous unit's staged data
  if ((threadIdx.x & 31) == 0) {
    const uint32_t koff = start & 3u, loff = start & 15u;
    const uint32_t kb = ((koff + cnt) * 4u + 15u) & ~15u, lb = (loff + cnt + 15u) & ~15u;
    const uint32_t mb = smem_u32(mbar);
    asm volatile("fence.proxy.async.shared::cta;\n"
                 "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(K * kb + lb) : "memory");
#pragma unroll
    for (int k = 0; k < K; ++k)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(key0 + k * row)), "l"(gkey[k] + (start - koff)), "r"(kb), "r"(mb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(let)), "l"(glet + (start - loff)), "r"(lb), "r"(mb) : "memory");
  }
  mbar_wait(mbar, parity);
  parity ^= 1u;
}

// TMA bulk prefetch of [p, p + bytes) into L2 (16-byte granules)
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, uint32_t bytes) {
  const uintptr_t a = (uintptr_t)p & ~uintptr_t(15);
  const uint32_t n = (uint32_t)((((uintptr_t)p + bytes + 15) & ~uintptr_t(15)) - a);
  if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
}

template <int K>
__device__ __forceinline__ uint32_t key_hash(const uint32_t (&kv)[K], int m) {
  uint32_t h = 0;
#pragma unroll
  for (int i = 0; i < K; ++i)
    if (i < m) h += kv[i] * (0x9E3779B1u + 0x7F4A7C16u * i);
  return fmix32(h);
}

// find-or-insert of the m-key prefix of kv (event e) in a node table of the
// current epoch; returns the slot, -1 when `limit` claims are exceeded
// (overflow -> the next path).  A new slot's histogram words are zeroed.
template <int K, int NF, int NSL>
__device__ __forceinline__ int node_probe(uint32_t *tag, uint32_t (*hist)[NF * 3], const uint32_t *const (&kb)[K],
                                          const uint32_t (&kv)[K], int e, int m, uint32_t ep, bool *isnew,
                                          uint32_t *claims, uint32_t limit, uint16_t *list) {
  constexpr int shift = 32 - __builtin_ctz((unsigned)NSL);
  uint32_t h = key_hash<K>(kv, m) >> shift;
  volatile uint32_t *vt = tag;
  while (true) {
    uint32_t t = vt[h];
    if ((t >> 16) != ep) {
      if (*(volatile uint32_t *)claims >= limit) return -1;
      const uint32_t o = atomicCAS(&tag[h], t, ep << 16 | (uint32_t)(e + 1));
      if (o == t) {
        *isnew = true;
#pragma unroll
        for (int x = 0; x < NF * 3; ++x) hist[h][x] = 0;
        list[atomicAdd(claims, 1u)] = (uint16_t)h;
        return (int)h;
      }
      t = o;
    }
    const int rep = (int)(t & 0xFFFFu) - 1;
    bool eq = true;
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (i < m) eq &= kb[i][rep] == kv[i];
    if (eq) { *isnew = false; return (int)h; }
    h = (h + 1) & (uint32_t)(NSL - 1);
  }
}

#ifndef LTL4C_WARP_MINB
#define LTL4C_WARP_MINB 4  // <= 64 registers: the shared-memory plan keeps up to 30 warps resident
#endif
template <int K, int NF, int CAP>
__global__ void __launch_bounds__(256, LTL4C_WARP_MINB) bucket_warp_kernel(BucketParams p) {
  using Tab = WarpTab<K, NF, CAP>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const DevProg *prog = p.prog;
  const int nq = prog->nq, A = 1 << prog->na;
  uint32_t *sacc = reinterpret_cast<uint32_t *>(smem_raw);
  uint8_t *slab = smem_raw + 4 * kMaxFormulas * (kMaxLevels + 1) * 6;
  uint8_t *sdelta = slab + kMaxFormulas * kMaxStates;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Tab &w = reinterpret_cast<Tab *>(smem_raw + warp_hdr_bytes(nq, prog->na))[wid];
  for (int i = threadIdx.x; i < nq * A; i += blockDim.x) sdelta[i] = prog->delta[i / A][i % A];
  for (int i = threadIdx.x; i < kMaxFormulas * kMaxStates; i += blockDim.x)
    slab[i] = prog->lab[i / kMaxStates][i % kMaxStates];
  for (int i = threadIdx.x; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) sacc[i] = 0;
  for (int i = lane; i < Tab::LS; i += 32) w.ltag[i] = 0;
  for (int i = lane; i < Tab::NL * Tab::NS; i += 32) (&w.ntag[0][0])[i] = 0;
  for (int i = lane; i < NF * 6; i += 32) w.pleaf[i] = 0;
  if (lane == 0) mbar_init(&w.mbar);
  uint32_t mpar = 0;  // phase parity of w.mbar
  __syncthreads();
  const uint32_t q0 = prog->q0;
  const uint32_t node_limit = Tab::NSL / 2;
  // per-lane leaf verdict counts, 16-bit fields j = 0..3 for v = 0, 2, 3, 5
  unsigned long long lcp[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) lcp[f] = 0;
  uint32_t since = 0;                   // leaves counted into lcp since its last flush (warp-uniform)
  auto flush_lcp = [&]() {
#pragma unroll
    for (int f = 0; f < NF; ++f) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t c = __reduce_add_sync(0xffffffffu, (uint32_t)(lcp[f] >> (16 * j)) & 0xFFFFu);
        if (lane == 0 && c) atomicAdd(&sacc[(f * (kMaxLevels + 1) + K) * 6 + (j == 0 ? 0 : j + 1 + (j == 3))], c);
      }
      lcp[f] = 0;
    }
  };

  // work: units [unit_start[u], unit_start[u+1]) (or the buckets of p.list),
  // taken dynamically; unit u+1 is resolved and prefetched while u is processed.
  // A unit above CAP events is split back into its buckets; a bucket above CAP
  // (or overflowing the node tables) is spilled to the next path's list.
  const bool listed = p.list != nullptr;
  const uint32_t n_items = listed ? (uint32_t)*p.list_len
                                  : min(p.n_units, (uint32_t)(*p.nvalid / kUnitTarget) + 2u);
  auto item = [&](uint32_t u, uint32_t &lo, uint32_t &hi) {
    if (listed) { lo = p.list[u]; hi = lo + 1; }
    else { lo = p.unit_start[u]; hi = p.unit_start[u + 1]; }
  };
#if LTL4C_STATIC_UNITS
  // static round-robin over the warps of the grid (units are balanced by construction)
  uint32_t snext = blockIdx.x * (blockDim.x >> 5) + wid;
  const uint32_t sstep = gridDim.x * (blockDim.x >> 5);
  auto take = [&]() { const uint32_t u = snext; snext += sstep; return u; };
#else
  // dynamic: LTL4C_UNIT_BATCH consecutive units per atomic on the shared counter (lane 0
  // keeps the rest of its batch)
  uint32_t bnext = 0, bleft = 0;
  auto take = [&]() {
    uint32_t u = 0;
    if (lane == 0) {
      if (bleft == 0) { bnext = atomicAdd(p.bucket_counter, (uint32_t)LTL4C_UNIT_BATCH); bleft = LTL4C_UNIT_BATCH; }
      u = bnext++;
      --bleft;
    }
    return u;
  };
#endif
  uint32_t nraw = take();
  uint32_t cu = __shfl_sync(0xffffffffu, nraw, 0);
  uint32_t cbl = 0, cbh = 0, cs0 = 0, cs1 = 0;
  if (cu < n_items) {
    item(cu, cbl, cbh);
    cs0 = p.bucket_off[cbl];
    cs1 = p.bucket_off[cbh];
  }
  nraw = take();
  uint32_t ep = 0;
  while (cu < n_items) {
    const uint32_t nu = __shfl_sync(0xffffffffu, nraw, 0);
    uint32_t nbl = 0, nbh = 0, ns0 = 0, ns1 = 0;
    if (nu < n_items) item(nu, nbl, nbh);
    nraw = take();
    bool nres = false;
    auto resolve_next = [&]() {   // next unit's event range + L2 prefetch of its bytes
      if (nres) return;
      nres = true;
      if (nu >= n_items) return;
      ns0 = p.bucket_off[nbl];
      ns1 = p.bucket_off[nbh];
      if (lane <= K && ns1 > ns0 && ns1 - ns0 <= (uint32_t)CAP) {
        if (lane < K) bulk_prefetch_l2(p.key[lane] + ns0, 4 * (ns1 - ns0));
        else bulk_prefetch_l2(p.let + ns0, ns1 - ns0);
      }
    };
    const bool split = cs1 - cs0 > (uint32_t)CAP && cbh - cbl > 1;
    for (uint32_t b = cbl;;) {
      uint32_t bl, bh, start, cnt;
      if (!split) {
        bl = cbl; bh = cbh; start = cs0; cnt = cs1 - cs0;
      } else {
        if (b >= cbh) break;
        bl = b; bh = b + 1;
        start = p.bucket_off[b];
        cnt = p.bucket_off[b + 1] - start;
        ++b;
      }
      if (cnt > (uint32_t)CAP) {
        if (lane == 0) p.spill_list[atomicAdd(p.spill_len, 1ull)] = bl;
      } else if (cnt > 0) {
        // a new epoch: every slot of the previous unit reads as empty
        if (++ep == 0x10000u) {
          for (int i = lane; i < Tab::LS; i += 32) w.ltag[i] = 0;
          for (int i = lane; i < Tab::NL * Tab::NS; i += 32) (&w.ntag[0][0])[i] = 0;
          ep = 1;
        }
        if (lane < 4) w.ncnt[lane] = 0;
        // stage the unit (TMA bulk copies, one per column)
        const uint32_t koff = start & 3u, loff = start & 15u;
        stage_bulk<K>(&w.key[0][0], CAP + 4, w.let, p.key, p.let, start, cnt, &w.mbar, mpar);
        const uint32_t *kb[K];
#pragma unroll
        for (int k = 0; k < K; ++k) kb[k] = &w.key[k][koff];
        const uint8_t *lb = &w.let[loff];
        // a3 + a4 over windows of 32 x kIlp events; verdicts are counted as they
        // change (a new leaf adds its verdict, a replayed leaf moves old -> new):
        // per-lane pending counts (pl) and child counts of the lane's current
        // ancestor (hv, flushed when the ancestor changes) -- committed only if the
        // unit does not overflow the node tables
        bool ovf = false;
        int cslot = -1;                 // per-lane cache: deepest ancestor of the last new leaf
        uint32_t ck[K > 1 ? K - 1 : 1];
#pragma unroll
        for (int i = 0; i < (K > 1 ? K - 1 : 1); ++i) ck[i] = 0;
        int cur = -1;
        unsigned long long hv[NF], pl[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) hv[f] = pl[f] = 0;
        auto flush_hv = [&]() {
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            if (hv[f] && cur >= 0) {
              uint32_t *hw = w.nhist[K > 1 ? K - 2 : 0][cur] + f * 3;
              const uint32_t f0 = (uint32_t)hv[f] & 0xFFFFu, f1 = (uint32_t)(hv[f] >> 16) & 0xFFFFu;
              const uint32_t f2 = (uint32_t)(hv[f] >> 32) & 0xFFFFu, f3 = (uint32_t)(hv[f] >> 48);
              if (f0) atomicAdd(&hw[0], f0);
              if (f1 | f2) atomicAdd(&hw[1], f1 | f2 << 16);
              if (f3) atomicAdd(&hw[2], f3 << 16);
            }
            hv[f] = 0;
          }
        };
        for (uint32_t base = 0; base < cnt; base += 32 * kIlp) {
          int slot[kIlp], par[kIlp];
          bool fresh[kIlp];
#pragma unroll
          for (int r = 0; r < kIlp; ++r) {
            const int e = (int)(base + 32 * r + lane);
            slot[r] = -1;
            par[r] = -1;
            fresh[r] = false;
            if (e < (int)cnt) {
              uint32_t kv[K];
#pragma unroll
              for (int i = 0; i < K; ++i) kv[i] = kb[i][e];
              constexpr int shift = 32 - __builtin_ctz((unsigned)Tab::LS);
              uint32_t h = key_hash<K>(kv, K) >> shift;
              volatile uint32_t *vt = w.ltag;
              while (true) {
                uint32_t t = vt[h];
                if ((t >> 16) != ep) {
                  const uint32_t o = atomicCAS(&w.ltag[h], t, ep << 16 | (uint32_t)(e + 1));
                  if (o == t) { fresh[r] = true; break; }
                  t = o;
                }
                const int rep = (int)(t & 0xFFFFu) - 1;
                bool eq = true;
#pragma unroll
                for (int i = 0; i < K; ++i) eq &= kb[i][rep] == kv[i];
                if (eq) break;
                h = (h + 1) & (uint32_t)(Tab::LS - 1);
              }
              slot[r] = (int)h;
              if (K > 1 && fresh[r] && !ovf) {
                // ancestors of the new leaf (depths 1 .. K-1), cached per lane
                bool hit = cslot >= 0;
#pragma unroll
                for (int i = 0; i < K - 1; ++i) hit &= ck[i] == kv[i];
                if (!hit) {
                  int parent = -1;
                  for (int l = 1; l < K; ++l) {
                    bool isnew = false;
                    const int ns = node_probe<K, NF, Tab::NSL>(w.ntag[l - 1], w.nhist[l - 1], kb, kv, e, l, ep, &isnew,
                                                     &w.ncnt[l], node_limit, w.nlist[l - 1]);
                    if (ns < 0) { ovf = true; break; }
                    if (isnew && l > 1) w.npar[l - 1][ns] = (uint16_t)parent;
                    parent = ns;
                  }
                  cslot = ovf ? -1 : parent;
#pragma unroll
                  for (int i = 0; i < K - 1; ++i) ck[i] = kv[i];
                }
                if (!ovf) w.lnode[h] = (uint8_t)cslot;
                par[r] = ovf ? -1 : cslot;
              }
            }
          }
          bool old = false;
#pragma unroll
          for (int r = 0; r < kIlp; ++r) old |= slot[r] >= 0 && !fresh[r];
          if (!__any_sync(0xffffffffu, old)) {
            // every touched slot is new and touched once: one step from q0, and the
            // leaf's verdict is counted
#pragma unroll
            for (int r = 0; r < kIlp; ++r) {
              if (slot[r] < 0) continue;
              const uint32_t q1 = sdelta[q0 * A + lb[base + 32 * r + lane]];
              w.lstate[slot[r]] = (uint8_t)(q1 | 0x80u);
              if (K > 1 && par[r] != cur) { flush_hv(); cur = par[r]; }
#pragma unroll
              for (int f = 0; f < NF; ++f) {
                const int v = slab[f * kMaxStates + q1];
                const unsigned long long inc = 1ull << (16 * ((v + 1) >> 1));  // v = 0, 2, 3, 5 -> field 0..3
                pl[f] += inc;
                if (K > 1) hv[f] += inc;
              }
            }
          } else {
#pragma unroll
            for (int r = 0; r < kIlp; ++r)
              if (fresh[r]) w.lstate[slot[r]] = (uint8_t)q0;
            __syncwarp();
#pragma unroll
            for (int r = 0; r < kIlp; ++r) {
              if (base + 32 * r >= cnt) break;
              const bool act = slot[r] >= 0;
              const uint32_t am = __ballot_sync(0xffffffffu, act);
              if (act) {
                const uint32_t peers = __match_any_sync(am, (uint32_t)slot[r]);
                if ((peers & lanemask_lt()) == 0) {  // leader: lowest lane of its group
                  const uint32_t raw = w.lstate[slot[r]];
                  const uint32_t qo = raw & 0x7Fu;
                  uint32_t q = qo;
                  uint32_t m = peers;
                  while (m) {
                    const int i = __ffs(m) - 1;
                    m &= m - 1;
                    q = sdelta[q * A + lb[base + 32 * r + i]];
                  }
                  w.lstate[slot[r]] = (uint8_t)(q | 0x80u);
                  const int pn = K > 1 ? (int)w.lnode[slot[r]] : 0;
                  uint32_t *hw = w.nhist[K > 1 ? K - 2 : 0][pn < Tab::NS ? pn : 0];
#pragma unroll
                  for (int f = 0; f < NF; ++f) {
                    const int vn = slab[f * kMaxStates + q], vo = slab[f * kMaxStates + qo];
                    if (!(raw & 0x80u)) {
                      atomicAdd(&w.pleaf[f * 6 + vn], 1);
                      if (K > 1) atomicAdd(&hw[f * 3 + (vn >> 1)], 1u << (16 * (vn & 1)));
                    } else if (vo != vn) {
                      atomicAdd(&w.pleaf[f * 6 + vo], -1);
                      atomicAdd(&w.pleaf[f * 6 + vn], 1);
                      if (K > 1) {
                        atomicAdd(&hw[f * 3 + (vn >> 1)], 1u << (16 * (vn & 1)));
                        atomicSub(&hw[f * 3 + (vo >> 1)], 1u << (16 * (vo & 1)));
                      }
                    }
                  }
                }
              }
              __syncwarp();
            }
          }
          __syncwarp();
        }
        resolve_next();
        if (K > 1) flush_hv();
        ovf = __any_sync(0xffffffffu, ovf);
        __syncwarp();
        if (ovf) {
          // too many distinct prefixes for the warp tables: hand the buckets on
          for (uint32_t x = bl + lane; x < bh; x += 32)
            if (p.bucket_off[x + 1] > p.bucket_off[x]) p.spill_list[atomicAdd(p.spill_len, 1ull)] = x;
        } else {
          // a5 (i): commit the unit's leaf-verdict counts
#pragma unroll
          for (int f = 0; f < NF; ++f) lcp[f] += pl[f];
          for (int i = lane; i < NF * 6; i += 32) {
            const int v = w.pleaf[i];
            if (v) atomicAdd(&sacc[((i / 6) * (kMaxLevels + 1) + K) * 6 + i % 6], (uint32_t)v);
          }
          since += CAP / 32;  // a lane adds at most CAP / 32 leaves per unit (16-bit fields)
          if (since > 60000u) { flush_lcp(); since = 0; }
          // a5 (ii): node verdicts by Def. 6, depth K-1 .. 1
          for (int l = K - 1; l >= 1; --l) {
            const uint32_t nn = w.ncnt[l];
            for (uint32_t i = lane; i < nn; i += 32) {
              const int s = w.nlist[l - 1][i];
#pragma unroll
              for (int f = 0; f < NF; ++f) {
                const uint32_t *hw = w.nhist[l - 1][s] + f * 3;
                uint32_t h[6];
#pragma unroll
                for (int x = 0; x < 6; ++x) h[x] = (hw[x >> 1] >> (16 * (x & 1))) & 0xFFFFu;
                const int v = node_verdict(prog->qkind[f][l], prog->qcmp[f][l], prog->qnum[f][l], prog->qden[f][l], h);
                atomicAdd(&sacc[(f * (kMaxLevels + 1) + l) * 6 + v], 1u);
                if (l > 1) atomicAdd(&w.nhist[l - 2][w.npar[l - 1][s]][f * 3 + (v >> 1)], 1u << (16 * (v & 1)));
              }
            }
            __syncwarp();
          }
        }
        for (int i = lane; i < NF * 6; i += 32) w.pleaf[i] = 0;
        __syncwarp();
      }
      if (!split) break;
    }
    resolve_next();
    cu = nu; cbl = nbl; cbh = nbh; cs0 = ns0; cs1 = ns1;
  }
  flush_lcp();
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) {
    const uint32_t v = sacc[i];
    const int f = i / ((kMaxLevels + 1) * 6), l = (i / 6) % (kMaxLevels + 1), bb = i % 6;
    if (v && f < NF && l >= 1 && l <= K) atomicAdd(&p.acc->hist[f][l][bb], (unsigned long long)v);
  }
}

// ----------------------------------------------- work units for bucket_warp
// unit u = buckets [unit_start[u], unit_start[u+1]): the buckets whose first event
// lies in [u * target, (u + 1) * target) (target = kUnitTarget; seg_unit for bucket_seg).  Lane per bucket c: the units
// whose boundary u * kUnitTarget lies in (off[c-1], off[c]] start at c (c = nb,
// the end: every remaining unit); the warp writes each lane's range together
// (a skewed bucket can own thousands of unit boundaries).
__global__ void unit_start_kernel(const uint32_t *off, uint32_t nb, uint32_t *ustart, uint32_t n_units, uint32_t target,
                                  const uint32_t *gate, int want) {
  if (gate && ((*gate != 0) != (want != 0))) return;
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  uint32_t u0 = 1, u1 = 0;  // empty
  if (c <= nb) {
    if (c == 0) { u0 = 0; u1 = 0; }
    else {
      u0 = off[c - 1] / target + 1;
      u1 = c == nb ? n_units : min(n_units, off[c] / target);
    }
  }
  uint32_t todo = __ballot_sync(0xffffffffu, u0 <= u1);
  while (todo) {
    const int l = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint32_t a = __shfl_sync(0xffffffffu, u0, l), b = __shfl_sync(0xffffffffu, u1, l);
    const uint32_t cc = __shfl_sync(0xffffffffu, c, l);
    for (uint32_t u = a + lane; u <= b; u += 32) ustart[u] = cc;
  }
}

// ----------------------------------------------- global tables
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// find-or-insert of an m-key vector in an epoch-tagged open-addressing table.
// Returns the slot; *inserted = 1 if the vector was not present.
__device__ unsigned long long table_find_insert(uint4 *slots, unsigned long long cap, uint32_t epoch,
                                                const uint32_t *k, int m, int *inserted,
                                                unsigned long long *overflow) {
  const uint32_t ready = (epoch << 1) | 1u, busy = epoch << 1;
  uint32_t h = 0x7F4A7C15u;
  for (int i = 0; i < m; ++i) h = fmix32(h ^ k[i]) + 0x632BE5ABu * (i + 1);
  unsigned long long slot = h & (cap - 1);
  for (unsigned long long probes = 0; probes < cap; ++probes) {
    uint32_t *tag = &slots[slot].x;
    uint32_t t = ld_acquire(tag);
    while (t == busy) t = ld_acquire(tag);
    if (t == ready) {
      const uint4 s = slots[slot];
      const bool eq = s.y == k[0] && (m < 2 || s.z == k[1]) && (m < 3 || s.w == k[2]);
      if (eq) { *inserted = 0; return slot; }
      slot = (slot + 1) & (cap - 1);
      continue;
    }
    // empty or stale (older epoch): claim it
    if (atomicCAS(tag, t, busy) == t) {
      slots[slot].y = k[0];
      slots[slot].z = m > 1 ? k[1] : 0u;
      slots[slot].w = m > 2 ? k[2] : 0u;
      *inserted = 1;
      return slot;  // caller initialises payload then publishes with table_publish
    }
    // lost the race: re-examine the same slot
  }
  atomicAdd(overflow, 1ull);
  *inserted = -1;
  return 0;
}

// st.release.gpu orders this thread's earlier writes (the slot's keys and the
// payload it initialised) before the tag: no separate fence is needed
__device__ __forceinline__ void table_publish(uint4 *slots, unsigned long long slot, uint32_t epoch) {
  st_release(&slots[slot].x, (epoch << 1) | 1u);
}

// ----------------------------------------------- online path (carried state)
// Online mode (§3.3): the submonitor set 𝔻 and every node of
// the quantifier tree persist across batches in global tables.  A batch is
// partitioned by the DEEPEST key (all events of a leaf share it, so a leaf's
// events land in one bucket, in trace order, and buckets stay balanced even
// when level-0 keys are few), then:
//   online_leaf   warp per unit (or per <= CAP-event chunk of a larger bucket, in
//                 order): leaves deduplicated in shared memory; a leaf seen for
//                 the first time in the chunk is found-or-inserted in the global
//                 leaf table (new leaves start at q0, existing ones resume --
//                 "merged"); its events are stepped in trace order;
//                 the state is written back; a verdict change old -> new moves
//                 one child of its depth-(K-1) node (h[old]--, h[new]++) and
//                 marks that node touched;
//   online_nodes  depth K-1 .. 1: every touched node re-evaluates Def. 6 from
//                 its histogram; a change moves one child of its parent.
// The per-level histograms (acc) receive the same signed deltas; the root rule
// is applied to the depth-1 histogram by finalize.
constexpr uint8_t kNewLeaf = 0xFF;

template <int K>
struct alignas(16) OnlineTab {
  static constexpr int CAP = kWarpCap;
  static constexpr int LS = 2 * CAP;
  uint32_t key[K][CAP + 4];             // staged keys; event i at [i + (start & 3)]
  uint8_t let[CAP + 32];                // staged letters; event i at [i + (start & 15)]
  uint32_t ltag[LS];                    // epoch << 16 | rep event + 1
  uint32_t lg[LS];                      // global leaf slot
  uint8_t lstate[LS];
  uint8_t linit[LS];                    // state at chunk start, kNewLeaf for a leaf created now
  uint16_t llist[CAP];
  uint32_t tstage[CAP];                 // nodes touched first by this chunk (appended together)
  uint32_t tn;
  alignas(8) unsigned long long mbar;   // staging barrier (stage_bulk)
};

// node of depth l (keys k[0..l-1]) in the carried tables; a new node starts with
// an empty histogram and no verdict
__device__ __forceinline__ unsigned long long online_node(const OnlineParams &p, int l, const uint32_t *k,
                                                          bool *ok) {
  const DevTables &T = p.b.tab;
  int ins;
  const unsigned long long s = table_find_insert(T.node_slot[l], T.node_cap[l], T.epoch, k, l, &ins,
                                                 &p.b.acc->table_overflow);
  if (ins == 1) {
    for (int x = 0; x < kMaxFormulas * 6; ++x) T.node_hist[l][s * kMaxFormulas * 6 + x] = 0;
    T.node_verdict[l][s] = 0xFFFFFFFFu;
    table_publish(T.node_slot[l], s, T.epoch);
    atomicAdd(&p.b.acc->nodes[l], 1ull);
  }
  *ok = ins >= 0;
  return s;
}

__device__ __forceinline__ void online_touch(const OnlineParams &p, uint32_t bid, int l, unsigned long long s) {
  if (atomicExch(&p.b.tab.node_aux[l][s], bid) != bid) p.tlist[l][atomicAdd(&p.tcnt[l], 1u)] = (uint32_t)s;
}

template <int K, int NF>
__global__ void __launch_bounds__(256) online_leaf_kernel(OnlineParams op) {
  const uint32_t bid = op.bid_dev ? *op.bid_dev : op.bid;  // (the params stay in the constant bank)
  using Tab = OnlineTab<K>;
  constexpr int CAP = Tab::CAP;
  const BucketParams &p = op.b;
  const DevTables &T = p.tab;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const DevProg *prog = p.prog;
  const int nq = prog->nq, A = 1 << prog->na;
  int *sacc = reinterpret_cast<int *>(smem_raw);
  uint8_t *slab = smem_raw + 4 * kMaxFormulas * (kMaxLevels + 1) * 6;
  uint8_t *sdelta = slab + kMaxFormulas * kMaxStates;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Tab &w = reinterpret_cast<Tab *>(smem_raw + warp_hdr_bytes(nq, prog->na))[wid];
  for (int i = threadIdx.x; i < nq * A; i += blockDim.x) sdelta[i] = prog->delta[i / A][i % A];
  for (int i = threadIdx.x; i < kMaxFormulas * kMaxStates; i += blockDim.x)
    slab[i] = prog->lab[i / kMaxStates][i % kMaxStates];
  for (int i = threadIdx.x; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) sacc[i] = 0;
  for (int i = lane; i < Tab::LS; i += 32) w.ltag[i] = 0;
  if (lane == 0) mbar_init(&w.mbar);
  uint32_t mpar = 0;  // phase parity of w.mbar
  __syncthreads();
  const uint32_t q0 = prog->q0;
  uint32_t newleaves = 0;  // leaves this lane inserted in the carried table
  int lacc[NF][6];  // per-lane leaf-level verdict deltas
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int v = 0; v < 6; ++v) lacc[f][v] = 0;
  uint32_t ep = 0;
  const uint32_t n_units = min(p.n_units, (uint32_t)(*p.nvalid / kUnitTarget) + 2u);
  while (true) {
    uint32_t u = 0;
    if (lane == 0) u = atomicAdd(p.bucket_counter, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= n_units) break;
    const uint32_t ubl = p.unit_start[u], ubh = p.unit_start[u + 1];
    if (ubh <= ubl) continue;
    const uint32_t us = p.bucket_off[ubl], ue = p.bucket_off[ubh];
    // pieces: the whole unit, or each bucket in chunks of <= CAP events (in order)
    const bool split = ue - us > (uint32_t)CAP;
    uint32_t b = ubl, pos = us, bend = split ? us : ue;
    while (true) {
      uint32_t start, cnt;
      if (!split) {
        if (pos >= ue) break;
        start = us;
        cnt = ue - us;
        pos = ue;
      } else {
        while (pos >= bend && b < ubh) { pos = p.bucket_off[b]; bend = p.bucket_off[b + 1]; ++b; }
        if (pos >= bend) break;
        start = pos;
        cnt = min((uint32_t)CAP, bend - pos);
        pos += cnt;
      }
      if (++ep == 0x10000u) {
        for (int i = lane; i < Tab::LS; i += 32) w.ltag[i] = 0;
        ep = 1;
      }
      const uint32_t koff = start & 3u, loff = start & 15u;
      stage_bulk<K>(&w.key[0][0], Tab::CAP + 4, w.let, p.key, p.let, start, cnt, &w.mbar, mpar);
      const uint32_t *kb[K];
#pragma unroll
      for (int k = 0; k < K; ++k) kb[k] = &w.key[k][koff];
      const uint8_t *lb = &w.let[loff];
      uint32_t nleaf = 0;
      for (uint32_t base = 0; base < cnt; base += 32 * kIlp) {
        int slot[kIlp];
        bool fresh[kIlp];
        uint32_t qs[kIlp];
#pragma unroll
        for (int r = 0; r < kIlp; ++r) {
          const int e = (int)(base + 32 * r + lane);
          slot[r] = -1;
          fresh[r] = false;
          qs[r] = 0;
          if (e < (int)cnt) {
            uint32_t kv[K];
#pragma unroll
            for (int i = 0; i < K; ++i) kv[i] = kb[i][e];
            constexpr int shift = 32 - __builtin_ctz((unsigned)Tab::LS);
            uint32_t h = key_hash<K>(kv, K) >> shift;
            volatile uint32_t *vt = w.ltag;
            while (true) {
              uint32_t t = vt[h];
              if ((t >> 16) != ep) {
                const uint32_t o = atomicCAS(&w.ltag[h], t, ep << 16 | (uint32_t)(e + 1));
                if (o == t) { fresh[r] = true; break; }
                t = o;
              }
              const int rep = (int)(t & 0xFFFFu) - 1;
              bool eq = true;
#pragma unroll
              for (int i = 0; i < K; ++i) eq &= kb[i][rep] == kv[i];
              if (eq) break;
              h = (h + 1) & (uint32_t)(Tab::LS - 1);
            }
            slot[r] = (int)h;
            if (fresh[r]) {
              // first sight in this chunk: the carried leaf (or a new one at q0)
              uint32_t k3[kMaxLevels] = {kv[0], K > 1 ? kv[1 % K] : 0u, K > 2 ? kv[2 % K] : 0u};
              int ins;
              const unsigned long long g = table_find_insert(T.leaf_slot, T.leaf_cap, T.epoch, k3, K, &ins,
                                                             &p.acc->table_overflow);
              uint32_t q = q0;
              if (ins == 1) {
                // publish at once: a lane of this warp probing through the slot spins
                // on its busy tag (a deferred publish could deadlock the warp)
                T.leaf_state[g] = (uint8_t)q0;
                table_publish(T.leaf_slot, g, T.epoch);
                ++newleaves;
              } else if (ins == 0) {
                q = T.leaf_state[g];
              }
              w.lg[h] = (uint32_t)g;
              w.linit[h] = ins == 0 ? (uint8_t)q : kNewLeaf;
              w.lstate[h] = (uint8_t)q;
              qs[r] = q;
            }
          }
        }
#pragma unroll
        for (int r = 0; r < kIlp; ++r) {  // append new leaves (warp-uniform count)
          const uint32_t nm = __ballot_sync(0xffffffffu, fresh[r]);
          if (fresh[r]) w.llist[nleaf + __popc(nm & lanemask_lt())] = (uint16_t)slot[r];
          nleaf += __popc(nm);
        }
        bool old = false;
#pragma unroll
        for (int r = 0; r < kIlp; ++r) old |= slot[r] >= 0 && !fresh[r];
        if (!__any_sync(0xffffffffu, old)) {
#pragma unroll
          for (int r = 0; r < kIlp; ++r)
            if (slot[r] >= 0) w.lstate[slot[r]] = sdelta[qs[r] * A + lb[base + 32 * r + lane]];
        } else {
          __syncwarp();
#pragma unroll
          for (int r = 0; r < kIlp; ++r) {
            if (base + 32 * r >= cnt) break;
            const bool act = slot[r] >= 0;
            const uint32_t am = __ballot_sync(0xffffffffu, act);
            if (act) {
              const uint32_t peers = __match_any_sync(am, (uint32_t)slot[r]);
              if ((peers & lanemask_lt()) == 0) {
                uint32_t q = w.lstate[slot[r]];
                uint32_t m = peers;
                while (m) {
                  const int i = __ffs(m) - 1;
                  m &= m - 1;
                  q = sdelta[q * A + lb[base + 32 * r + i]];
                }
                w.lstate[slot[r]] = (uint8_t)q;
              }
            }
            __syncwarp();
          }
        }
        __syncwarp();
      }
      // write back, verdict deltas, parent histogram deltas (lane-contiguous runs:
      // a lane's leaves mostly share a parent, looked up once)
      const uint32_t per = (nleaf + 31) >> 5;
      const uint32_t i0 = min(nleaf, lane * per), i1 = min(nleaf, i0 + per);
      long long pslot = -1;
      bool pok = false;
      uint32_t pk[kMaxLevels] = {0, 0, 0};
      if (lane == 0) w.tn = 0;
      __syncwarp();
      for (uint32_t i = i0; i < i1; ++i) {
        const int s = w.llist[i];
        const uint32_t qn = w.lstate[s], qi = w.linit[s];
        T.leaf_state[w.lg[s]] = (uint8_t)qn;
        int vo[NF], vn[NF];
        bool any = false;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          vn[f] = slab[f * kMaxStates + qn];
          vo[f] = qi == kNewLeaf ? -1 : (int)slab[f * kMaxStates + qi];
          if (vo[f] != vn[f]) {
            any = true;
#pragma unroll
            for (int v = 0; v < 6; ++v) lacc[f][v] += (vn[f] == v) - (vo[f] == v);
          }
        }
        if (K > 1 && any) {
          const int rep = (int)(w.ltag[s] & 0xFFFFu) - 1;
          uint32_t k[kMaxLevels] = {0, 0, 0};
          bool same = pslot >= 0;
#pragma unroll
          for (int x = 0; x < K - 1; ++x) {
            k[x] = kb[x][rep];
            same &= k[x] == pk[x];
          }
          if (!same) {
            pslot = (long long)online_node(op, K - 1, k, &pok);
#pragma unroll
            for (int x = 0; x < K - 1; ++x) pk[x] = k[x];
            if (pok && atomicExch(&T.node_aux[K - 1][pslot], bid) != bid)
              w.tstage[atomicAdd(&w.tn, 1u)] = (uint32_t)pslot;  // first touch this batch
          }
          if (pok) {
            uint32_t *hist = T.node_hist[K - 1] + (unsigned long long)pslot * kMaxFormulas * 6;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
              if (vo[f] != vn[f]) {
                if (vo[f] >= 0) atomicAdd(&hist[f * 6 + vo[f]], 0xFFFFFFFFu);
                atomicAdd(&hist[f * 6 + vn[f]], 1u);
              }
            }
          }
        }
      }
      __syncwarp();
      if (K > 1) {
        // the chunk's newly touched nodes: one global append for the warp
        const uint32_t tn = w.tn;
        uint32_t tb = 0;
        if (lane == 0 && tn) tb = atomicAdd(&op.tcnt[K - 1], tn);
        tb = __shfl_sync(0xffffffffu, tb, 0);
        for (uint32_t i = lane; i < tn; i += 32) op.tlist[K - 1][tb + i] = w.tstage[i];
        __syncwarp();
      }
    }
  }
  {
    const uint32_t c = __reduce_add_sync(0xffffffffu, newleaves);
    if (lane == 0 && c) atomicAdd(&p.acc->leaves, (unsigned long long)c);
  }
  // leaf-level verdict deltas: warp sums, then the CTA's
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int v = 0; v < 6; ++v) {
      const int c = __reduce_add_sync(0xffffffffu, lacc[f][v]);
      if (lane == 0 && c) atomicAdd(&sacc[(f * (kMaxLevels + 1) + K) * 6 + v], c);
    }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) {
    const int v = sacc[i];
    if (v) atomicAdd(&p.acc->hist[0][0][0] + i, (unsigned long long)(long long)v);
  }
}

// depth-l touched nodes: Def. 6 from the carried histogram; a changed verdict moves
// one child of the parent (depth l-1), or of the root's histogram for l = 1
template <int NF>
__global__ void __launch_bounds__(256) online_nodes_kernel(OnlineParams op, int l) {
  const uint32_t bid = op.bid_dev ? *op.bid_dev : op.bid;  // (the params stay in the constant bank)
  __shared__ int sacc[kMaxFormulas * 6];
  const BucketParams &p = op.b;
  const DevTables &T = p.tab;
  const DevProg *prog = p.prog;
  for (int i = threadIdx.x; i < kMaxFormulas * 6; i += blockDim.x) sacc[i] = 0;
  __syncthreads();
  const uint32_t n = op.tcnt[l];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t s = op.tlist[l][i];
    const uint32_t *hist = T.node_hist[l] + (unsigned long long)s * kMaxFormulas * 6;
    const uint32_t packed = T.node_verdict[l][s];
    uint32_t np = packed;
    int vo[NF], vn[NF];
    bool any = false;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      uint32_t h[6];
#pragma unroll
      for (int v = 0; v < 6; ++v) h[v] = hist[f * 6 + v];
      vn[f] = node_verdict(prog->qkind[f][l], prog->qcmp[f][l], prog->qnum[f][l], prog->qden[f][l], h);
      const uint32_t o = (packed >> (8 * f)) & 0xFFu;
      vo[f] = o == 0xFFu ? -1 : (int)o;
      if (vo[f] != vn[f]) {
        any = true;
        if (vo[f] >= 0) atomicAdd(&sacc[f * 6 + vo[f]], -1);
        atomicAdd(&sacc[f * 6 + vn[f]], 1);
        np = (np & ~(0xFFu << (8 * f))) | ((uint32_t)vn[f] << (8 * f));
      }
    }
    if (!any) continue;
    T.node_verdict[l][s] = np;
    if (l >= 2) {
      const uint4 ks = T.node_slot[l][s];
      const uint32_t k[kMaxLevels] = {ks.y, ks.z, ks.w};
      bool ok;
      const unsigned long long ps = online_node(op, l - 1, k, &ok);
      if (!ok) continue;
      online_touch(op, bid, l - 1, ps);
      uint32_t *ph = T.node_hist[l - 1] + ps * kMaxFormulas * 6;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        if (vo[f] != vn[f]) {
          if (vo[f] >= 0) atomicAdd(&ph[f * 6 + vo[f]], 0xFFFFFFFFu);
          atomicAdd(&ph[f * 6 + vn[f]], 1u);
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxFormulas * 6; i += blockDim.x) {
    const int v = sacc[i];
    if (v) atomicAdd(&p.acc->hist[i / 6][l][i % 6], (unsigned long long)(long long)v);
  }
}

// ----------------------------------------------- rehash (online tables grow)
__global__ void rehash_kernel(DevTables from, DevTables to, int nl, int nf, unsigned long long *overflow) {
  const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t ready = (from.epoch << 1) | 1u;
  // blockIdx.y = 0: leaves (m = nl keys), y = l in [1, nl-1]: nodes of depth l
  const int l = blockIdx.y;
  if (l == 0) {
    if (i >= from.leaf_cap) return;
    const uint4 s = from.leaf_slot[i];
    if (s.x != ready) return;
    const uint32_t k[3] = {s.y, s.z, s.w};
    int ins;
    const unsigned long long j = table_find_insert(to.leaf_slot, to.leaf_cap, to.epoch, k, nl, &ins, overflow);
    if (ins < 0) return;
    to.leaf_state[j] = from.leaf_state[i];
    table_publish(to.leaf_slot, j, to.epoch);
  } else {
    if (l >= nl || i >= from.node_cap[l]) return;
    const uint4 s = from.node_slot[l][i];
    if (s.x != ready) return;
    const uint32_t k[3] = {s.y, s.z, s.w};
    int ins;
    const unsigned long long j = table_find_insert(to.node_slot[l], to.node_cap[l], to.epoch, k, l, &ins, overflow);
    if (ins < 0) return;
    to.node_verdict[l][j] = from.node_verdict[l][i];
    for (int x = 0; x < kMaxFormulas * 6; ++x)
      to.node_hist[l][j * kMaxFormulas * 6 + x] = from.node_hist[l][i * kMaxFormulas * 6 + x];
    table_publish(to.node_slot[l], j, to.epoch);
  }
}


// ----------------------------------------------- heavy path (offline, skewed buckets)
// H0: segments per oversize bucket -> seg_base (exclusive scan), total in ctr[1]
__global__ void __launch_bounds__(1024) heavy_plan_kernel(HeavyParams h) {
  __shared__ uint32_t buf[1024];
  __shared__ uint32_t wt[32];
  const uint32_t L = (uint32_t)*h.list_len;
  uint32_t carry = 0;
  for (uint32_t o = 0; o < L; o += 1024) {
    const uint32_t i = o + threadIdx.x;
    uint32_t v = 0;
    if (i < L) {
      const uint32_t b = h.list[i];
      v = (h.bucket_off[b + 1] - h.bucket_off[b] + kSegW - 1) / kSegW;
    }
    buf[threadIdx.x] = v;
    __syncthreads();
    const uint32_t tot = block_exclusive_scan(buf, 1024, wt);
    if (i < L) h.seg_base[i] = buf[threadIdx.x] + carry;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) { h.seg_base[L] = carry; h.ctr[1] = carry; }
}

// H1: segments of kSegW events, one warp each.  The segment is
// staged into warp-private shared memory; its value vectors are deduplicated in
// an epoch-tagged warp table; every leaf's transition maps are composed in trace
// order (a window whose slots are all new and touched once takes the letter's
// map; otherwise lanes sharing a slot are grouped and the leader composes in
// lane order); one partial {dense leaf, segment, map} per leaf of the segment.

template <int K>
struct alignas(16) SegTab {
  static constexpr int LS = 2 * kSegW;
  uint32_t key[K][kSegW + 4];
  uint8_t let[kSegW + 32];
  uint32_t ltag[LS];
  unsigned long long lmap[LS];
  uint16_t llist[kSegW];
  alignas(8) unsigned long long mbar;   // staging barrier (stage_bulk)
};

template <int K, int NQB>
__global__ void __launch_bounds__(256) heavy_segw_kernel(HeavyParams h) {
  using Tab = SegTab<K>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  unsigned long long *smap = reinterpret_cast<unsigned long long *>(smem_raw);  // [256]
  const DevProg *prog = h.prog;
  const int nq = prog->nq, A = 1 << prog->na;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Tab &w = reinterpret_cast<Tab *>(smem_raw + 8 * kMaxLetters)[wid];
  for (int i = threadIdx.x; i < A; i += blockDim.x) smap[i] = prog->map[i];
  for (int i = lane; i < Tab::LS; i += 32) w.ltag[i] = 0;
  if (lane == 0) mbar_init(&w.mbar);
  uint32_t mpar = 0;  // phase parity of w.mbar
  __syncthreads();
  const DevTables &T = h.tab;
  unsigned long long ident = 0;
  for (int q = 0; q < nq; ++q) ident |= (unsigned long long)q << (4 * q);
  const uint32_t L = (uint32_t)*h.list_len;
  const uint32_t n_items = h.ctr[1];
  uint32_t ep = 0;
  while (true) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(&h.ctr[0], 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    // bucket of the item: last i with seg_base[i] <= item
    uint32_t lo = 0, hi = L;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (h.seg_base[mid] <= item) lo = mid; else hi = mid;
    }
    const uint32_t b = h.list[lo];
    const uint32_t j = item - h.seg_base[lo];
    const uint32_t boff = h.bucket_off[b], bcnt = h.bucket_off[b + 1] - boff;
    const uint32_t start = boff + j * kSegW;
    const uint32_t cnt = min((uint32_t)kSegW, bcnt - j * kSegW);
    if (++ep == 0x10000u) {
      for (int i = lane; i < Tab::LS; i += 32) w.ltag[i] = 0;
      ep = 1;
    }
    const uint32_t koff = start & 3u, loff = start & 15u;
    stage_bulk<K>(&w.key[0][0], kSegW + 4, w.let, h.key, h.let, start, cnt, &w.mbar, mpar);
    const uint32_t *kb[K];
#pragma unroll
    for (int k = 0; k < K; ++k) kb[k] = &w.key[k][koff];
    const uint8_t *lb = &w.let[loff];
    uint32_t nleaf = 0;
    for (uint32_t base = 0; base < cnt; base += 32 * kIlp) {
      int slot[kIlp];
      bool fresh[kIlp];
#pragma unroll
      for (int r = 0; r < kIlp; ++r) {
        const int e = (int)(base + 32 * r + lane);
        slot[r] = -1;
        fresh[r] = false;
        if (e < (int)cnt) {
          uint32_t kv[K];
#pragma unroll
          for (int i = 0; i < K; ++i) kv[i] = kb[i][e];
          constexpr int shift = 32 - __builtin_ctz((unsigned)Tab::LS);
          uint32_t hh = key_hash<K>(kv, K) >> shift;
          volatile uint32_t *vt = w.ltag;
          while (true) {
            uint32_t t = vt[hh];
            if ((t >> 16) != ep) {
              const uint32_t o = atomicCAS(&w.ltag[hh], t, ep << 16 | (uint32_t)(e + 1));
              if (o == t) { fresh[r] = true; break; }
              t = o;
            }
            const int rep = (int)(t & 0xFFFFu) - 1;
            bool eq = true;
#pragma unroll
            for (int i = 0; i < K; ++i) eq &= kb[i][rep] == kv[i];
            if (eq) break;
            hh = (hh + 1) & (uint32_t)(Tab::LS - 1);
          }
          slot[r] = (int)hh;
        }
      }
#pragma unroll
      for (int r = 0; r < kIlp; ++r) {
        const uint32_t nm = __ballot_sync(0xffffffffu, fresh[r]);
        if (fresh[r]) w.llist[nleaf + __popc(nm & lanemask_lt())] = (uint16_t)slot[r];
        nleaf += __popc(nm);
      }
      bool old = false;
#pragma unroll
      for (int r = 0; r < kIlp; ++r) old |= slot[r] >= 0 && !fresh[r];
      if (!__any_sync(0xffffffffu, old)) {
#pragma unroll
        for (int r = 0; r < kIlp; ++r)
          if (slot[r] >= 0) w.lmap[slot[r]] = smap[lb[base + 32 * r + lane]];
      } else {
#pragma unroll
        for (int r = 0; r < kIlp; ++r)
          if (fresh[r]) w.lmap[slot[r]] = ident;
        __syncwarp();
#pragma unroll
        for (int r = 0; r < kIlp; ++r) {
          if (base + 32 * r >= cnt) break;
          const bool act = slot[r] >= 0;
          const int s0 = __shfl_sync(0xffffffffu, slot[r], 0);
          if (__all_sync(0xffffffffu, !act || slot[r] == s0)) {
            // one leaf in the whole round (a skewed key): ordered tree composition
            // of the 32 lanes' maps (lane order = trace order), 5 steps
            unsigned long long m = act ? smap[lb[base + 32 * r + lane]] : ident;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const unsigned long long o = __shfl_down_sync(0xffffffffu, m, d);
              if ((lane & (2 * d - 1)) == 0) m = map_apply_t<NQB>(o, m);
            }
            if (lane == 0) w.lmap[s0] = map_apply_t<NQB>(m, w.lmap[s0]);
          } else {
            const uint32_t am = __ballot_sync(0xffffffffu, act);
            if (act) {
              const uint32_t peers = __match_any_sync(am, (uint32_t)slot[r]);
              if ((peers & lanemask_lt()) == 0) {
                unsigned long long m = w.lmap[slot[r]];
                uint32_t pm = peers;
                while (pm) {
                  const int i = __ffs(pm) - 1;
                  pm &= pm - 1;
                  m = map_apply_t<NQB>(smap[lb[base + 32 * r + i]], m);
                }
                w.lmap[slot[r]] = m;
              }
            }
          }
          __syncwarp();
        }
      }
      __syncwarp();
    }
    // one partial per leaf of the segment
    unsigned long long pbase = 0;
    if (lane == 0) pbase = atomicAdd(h.n_part, (unsigned long long)nleaf);
    pbase = __shfl_sync(0xffffffffu, pbase, 0);
    for (uint32_t i = lane; i < nleaf; i += 32) {
      const int s = w.llist[i];
      const int rep = (int)(w.ltag[s] & 0xFFFFu) - 1;
      uint32_t k[kMaxLevels] = {0, 0, 0};
#pragma unroll
      for (int x = 0; x < K; ++x) k[x] = kb[x][rep];
      int ins;
      const unsigned long long slot = table_find_insert(T.leaf_slot, T.leaf_cap, T.epoch, k, K, &ins, &h.acc->table_overflow);
      // dense ids of the new leaves: one counter update per group of converged lanes
      uint32_t dense = 0;
      const unsigned am = __activemask();
      const unsigned nm = __ballot_sync(am, ins == 1);
      if (nm) {
        const int leader = __ffs(nm) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(h.n_leaves, (unsigned long long)__popc(nm));
        base = __shfl_sync(am, base, leader);
        dense = (uint32_t)base + __popc(nm & lanemask_lt());
      }
      if (ins < 0) { h.part[pbase + i] = make_uint4(0xFFFFFFFFu, 0u, 0u, 0u); continue; }
      if (ins == 1) {
        T.leaf_aux[slot] = dense;
        h.leaf_slot_of[dense] = (uint32_t)slot;
        table_publish(T.leaf_slot, slot, T.epoch);
      } else {
        dense = *(volatile uint32_t *)&T.leaf_aux[slot];
      }
      atomicAdd(&h.leaf_npart[dense], 1u);
      const unsigned long long m = w.lmap[s];
      h.part[pbase + i] = make_uint4(dense, item, (uint32_t)m, (uint32_t)(m >> 32));
    }
    __syncwarp();
  }
}

// H2: exclusive scan of leaf_npart[0 .. n_leaves) -> leaf_off (3 kernels; the
// grids are persistent and loop over the device-side count)
__global__ void __launch_bounds__(1024) heavy_scan_blocks(HeavyParams h) {
  __shared__ uint32_t buf[1024];
  __shared__ uint32_t wt[32];
  const unsigned long long n = *h.n_leaves;
  for (unsigned long long blk = blockIdx.x; blk * 1024 < n; blk += gridDim.x) {
    const unsigned long long i = blk * 1024 + threadIdx.x;
    buf[threadIdx.x] = i < n ? h.leaf_npart[i] : 0u;
    __syncthreads();
    const uint32_t tot = block_exclusive_scan(buf, 1024, wt);
    if (i < n) h.leaf_off[i] = buf[threadIdx.x];
    if (threadIdx.x == 0) h.scan_tmp[blk] = tot;
    __syncthreads();
  }
}
__global__ void __launch_bounds__(1024) heavy_scan_sums(HeavyParams h) {
  __shared__ uint32_t buf[1024];
  __shared__ uint32_t wt[32];
  const uint32_t nblk = (uint32_t)((*h.n_leaves + 1023) / 1024);
  uint32_t carry = 0;
  for (uint32_t o = 0; o < nblk; o += 1024) {
    const uint32_t i = o + threadIdx.x;
    buf[threadIdx.x] = i < nblk ? h.scan_tmp[i] : 0u;
    __syncthreads();
    const uint32_t tot = block_exclusive_scan(buf, 1024, wt);
    if (i < nblk) h.scan_tmp[i] = buf[threadIdx.x] + carry;
    carry += tot;
    __syncthreads();
  }
}
__global__ void __launch_bounds__(1024) heavy_scan_add(HeavyParams h) {
  const unsigned long long n = *h.n_leaves;
  for (unsigned long long i = (unsigned long long)blockIdx.x * 1024 + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * 1024)
    h.leaf_off[i] += h.scan_tmp[i / 1024];
}

// H3: partials grouped by leaf (order inside a group restored in H4)
__global__ void heavy_group_kernel(HeavyParams h) {
  const unsigned long long n = *h.n_part;
  for (unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (unsigned long long)gridDim.x * blockDim.x) {
    const uint4 r = h.part[p];
    if (r.x == 0xFFFFFFFFu) continue;
    const uint32_t pos = h.leaf_off[r.x] + atomicAdd(&h.leaf_fill[r.x], 1u);
    h.lists[pos] = make_uint4(r.y, r.z, r.w, 0u);
  }
}

// leaf verdict + its depth-(K-1) parent's child histogram (or the depth-1 counts)
template <int K>
__device__ void heavy_leaf_done(const HeavyParams &h, uint32_t dense, int q, int *acc) {
  const DevProg *prog = h.prog;
  const DevTables &T = h.tab;
  const int nf = prog->nf;
  unsigned long long nslot = 0;
  bool ok = true;
  if (K > 1) {
    const uint4 ks = T.leaf_slot[h.leaf_slot_of[dense]];
    const uint32_t k[3] = {ks.y, ks.z, ks.w};
    int ins;
    nslot = table_find_insert(T.node_slot[K - 1], T.node_cap[K - 1], T.epoch, k, K - 1, &ins, &h.acc->table_overflow);
    if (ins == 1) {
      for (int x = 0; x < kMaxFormulas * 6; ++x) T.node_hist[K - 1][nslot * kMaxFormulas * 6 + x] = 0;
      const uint32_t d = (uint32_t)atomicAdd(&h.n_nodes[K - 1], 1ull);
      T.node_aux[K - 1][nslot] = d;
      h.node_list[K - 1][d] = (uint32_t)nslot;
      table_publish(T.node_slot[K - 1], nslot, T.epoch);
    }
    ok = ins >= 0;
  }
  for (int f = 0; f < nf; ++f) {
    const int v = prog->lab[f][q];
    atomicAdd(&acc[acc_idx(f, K, v)], 1);
    if (K > 1 && ok) atomicAdd(&T.node_hist[K - 1][nslot * kMaxFormulas * 6 + f * 6 + v], 1u);
  }
}

// warp-cooperative variant (all 32 lanes call it; `act` lanes carry a leaf):
// increments of the same node-histogram counter are aggregated across the warp
template <int K>
__device__ void heavy_leaf_done_warp(const HeavyParams &h, bool act, uint32_t dense, int q, int *acc) {
  const DevProg *prog = h.prog;
  const DevTables &T = h.tab;
  const int nf = prog->nf;
  const int lane = threadIdx.x & 31;
  unsigned long long nslot = 0;
  bool ok = act;
  if (K > 1 && act) {
    const uint4 ks = T.leaf_slot[h.leaf_slot_of[dense]];
    const uint32_t k[3] = {ks.y, ks.z, ks.w};
    int ins;
    nslot = table_find_insert(T.node_slot[K - 1], T.node_cap[K - 1], T.epoch, k, K - 1, &ins, &h.acc->table_overflow);
    if (ins == 1) {
      for (int x = 0; x < kMaxFormulas * 6; ++x) T.node_hist[K - 1][nslot * kMaxFormulas * 6 + x] = 0;
      const uint32_t d = (uint32_t)atomicAdd(&h.n_nodes[K - 1], 1ull);
      T.node_aux[K - 1][nslot] = d;
      h.node_list[K - 1][d] = (uint32_t)nslot;
      table_publish(T.node_slot[K - 1], nslot, T.epoch);
    }
    ok = ins >= 0;
  }
  for (int f = 0; f < nf; ++f) {
    const int v = act ? prog->lab[f][q] : 0;
    if (act) atomicAdd(&acc[acc_idx(f, K, v)], 1);
    if (K > 1) {
      const unsigned long long key = ok ? (nslot * 8ull + (unsigned long long)v) : ~0ull;
      const uint32_t peers = __match_any_sync(0xffffffffu, key);
      if (ok && (peers & lanemask_lt()) == 0)
        atomicAdd(&T.node_hist[K - 1][nslot * kMaxFormulas * 6 + f * 6 + v], (uint32_t)__popc(peers));
    }
  }
  (void)lane;
}

// H4: leaves with <= 32 partials (thread per leaf); longer ones are listed
template <int K>
__global__ void __launch_bounds__(256) heavy_short_kernel(HeavyParams h) {
  __shared__ int acc[kMaxFormulas * (kMaxLevels + 1) * 6];
  for (int i = threadIdx.x; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  const DevProg *prog = h.prog;
  const int nq = prog->nq;
  const unsigned long long n = *h.n_leaves;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long d0 = (unsigned long long)blockIdx.x * blockDim.x; d0 < n; d0 += stride) {
    const unsigned long long d = d0 + threadIdx.x;  // warp-uniform trip count
    bool act = d < n;
    int q = prog->q0;
    if (act) {
      const uint32_t off = h.leaf_off[d], len = h.leaf_npart[d];
      if (len > 32) {
        h.long_list[atomicAdd(&h.ctr[2], 1u)] = (uint32_t)d;
        act = false;
      } else {
        // insertion sort of the leaf's partials by segment item, then ordered composition
        uint4 *l = h.lists + off;
        for (uint32_t a = 1; a < len; ++a) {
          const uint4 x = l[a];
          int bb = (int)a - 1;
          while (bb >= 0 && l[bb].x > x.x) { l[bb + 1] = l[bb]; --bb; }
          l[bb + 1] = x;
        }
        for (uint32_t a = 0; a < len; ++a) {
          const unsigned long long m = (unsigned long long)l[a].y | ((unsigned long long)l[a].z << 32);
          q = (int)((m >> (4 * q)) & 15ull);
        }
      }
    }
    (void)nq;
    heavy_leaf_done_warp<K>(h, act, (uint32_t)(act ? d : 0), q, acc);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) {
    const int v = acc[i];
    const int f = i / ((kMaxLevels + 1) * 6), l = (i / 6) % (kMaxLevels + 1), b = i % 6;
    if (v) atomicAdd(&h.acc->hist[f][l][b], (unsigned long long)(long long)v);
  }
}

// H4b: long leaves, one CTA each: the segment items of a leaf lie in one
// bucket's contiguous item range, so partial maps are placed by item and
// composed with an ordered tree reduction in shared memory.
constexpr int kLongWin = 4096;
template <int K, int NQB>
__global__ void __launch_bounds__(1024) heavy_long_kernel(HeavyParams h) {
  __shared__ unsigned long long M[kLongWin];
  __shared__ int acc[kMaxFormulas * (kMaxLevels + 1) * 6];
  __shared__ uint32_t red[32];
  __shared__ uint32_t leaf_i, span_all;
  const DevProg *prog = h.prog;
  const int nq = prog->nq, tid = threadIdx.x;
  unsigned long long ident = 0;
  for (int q = 0; q < nq; ++q) ident |= (unsigned long long)q << (4 * q);
  for (int i = tid; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) acc[i] = 0;
  while (true) {
    __syncthreads();
    if (tid == 0) leaf_i = atomicAdd(&h.ctr[3], 1u);
    __syncthreads();
    if (leaf_i >= h.ctr[2]) break;
    const uint32_t d = h.long_list[leaf_i];
    const uint32_t off = h.leaf_off[d], len = h.leaf_npart[d];
    // minimum item of the leaf
    uint32_t mn = 0xFFFFFFFFu;
    for (uint32_t a = tid; a < len; a += blockDim.x) mn = min(mn, h.lists[off + a].x);
    for (int o = 16; o; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if ((tid & 31) == 0) red[tid >> 5] = mn;
    __syncthreads();
    if (tid < 32) {
      uint32_t v = tid < (int)(blockDim.x >> 5) ? red[tid] : 0xFFFFFFFFu;
      for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (tid == 0) red[0] = v;
    }
    __syncthreads();
    const uint32_t base = red[0];
    unsigned long long total = ident;  // valid in thread 0
    // items span at most the bucket's segment count; windows of kLongWin items
    uint32_t span = 0;
    for (uint32_t a = tid; a < len; a += blockDim.x) span = max(span, h.lists[off + a].x - base + 1);
    for (int o = 16; o; o >>= 1) span = max(span, __shfl_xor_sync(0xffffffffu, span, o));
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = span;
    __syncthreads();
    if (tid < 32) {
      uint32_t v = tid < (int)(blockDim.x >> 5) ? red[tid] : 0u;
      for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (tid == 0) span_all = v;  // not red[1]: lane 1 reads that slot above
    }
    __syncthreads();
    const uint32_t nspan = span_all;
    for (uint32_t w0 = 0; w0 < nspan; w0 += kLongWin) {
      for (int x = tid; x < kLongWin; x += blockDim.x) M[x] = ident;
      __syncthreads();
      for (uint32_t a = tid; a < len; a += blockDim.x) {
        const uint4 r = h.lists[off + a];
        const uint32_t pos = r.x - base;
        if (pos >= w0 && pos < w0 + kLongWin)
          M[pos - w0] = (unsigned long long)r.y | ((unsigned long long)r.z << 32);
      }
      __syncthreads();
      for (int stride = 1; stride < kLongWin; stride <<= 1) {  // ordered tree: M[i] = M[i+s] o M[i]
        for (int x = tid * 2 * stride; x + stride < kLongWin; x += blockDim.x * 2 * stride)
          M[x] = map_apply_t<NQB>(M[x + stride], M[x]);
        __syncthreads();
      }
      if (tid == 0) total = map_apply_t<NQB>(M[0], total);
      __syncthreads();
    }
    if (tid == 0) heavy_leaf_done<K>(h, d, (int)((total >> (4 * prog->q0)) & 15ull), acc);
  }
  __syncthreads();
  for (int i = tid; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) {
    const int v = acc[i];
    const int f = i / ((kMaxLevels + 1) * 6), l = (i / 6) % (kMaxLevels + 1), b = i % 6;
    if (v) atomicAdd(&h.acc->hist[f][l][b], (unsigned long long)(long long)v);
  }
}

// H5: node verdicts of depth l (Def. 6) and their parents' child histograms
template <int K>
__global__ void __launch_bounds__(256) heavy_nodes_kernel(HeavyParams h, int l) {
  __shared__ int acc[kMaxFormulas * (kMaxLevels + 1) * 6];
  for (int i = threadIdx.x; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  const DevProg *prog = h.prog;
  const DevTables &T = h.tab;
  const int nf = prog->nf;
  const unsigned long long n = h.n_nodes[l];
  for (unsigned long long d = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; d < n;
       d += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t slot = h.node_list[l][d];
    unsigned long long pslot = 0;
    bool ok = true;
    if (l > 1) {
      const uint4 ks = T.node_slot[l][slot];
      const uint32_t k[3] = {ks.y, ks.z, ks.w};
      int ins;
      pslot = table_find_insert(T.node_slot[l - 1], T.node_cap[l - 1], T.epoch, k, l - 1, &ins, &h.acc->table_overflow);
      if (ins == 1) {
        for (int x = 0; x < kMaxFormulas * 6; ++x) T.node_hist[l - 1][pslot * kMaxFormulas * 6 + x] = 0;
        const uint32_t dd = (uint32_t)atomicAdd(&h.n_nodes[l - 1], 1ull);
        T.node_aux[l - 1][pslot] = dd;
        h.node_list[l - 1][dd] = (uint32_t)pslot;
        table_publish(T.node_slot[l - 1], pslot, T.epoch);
      }
      ok = ins >= 0;
    }
    for (int f = 0; f < nf; ++f) {
      const uint32_t *hh = T.node_hist[l] + (size_t)slot * kMaxFormulas * 6 + f * 6;
      const int v = node_verdict(prog->qkind[f][l], prog->qcmp[f][l], prog->qnum[f][l], prog->qden[f][l], hh);
      atomicAdd(&acc[acc_idx(f, l, v)], 1);
      if (l > 1 && ok) atomicAdd(&T.node_hist[l - 1][pslot * kMaxFormulas * 6 + f * 6 + v], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxFormulas * (kMaxLevels + 1) * 6; i += blockDim.x) {
    const int v = acc[i];
    const int f = i / ((kMaxLevels + 1) * 6), ll = (i / 6) % (kMaxLevels + 1), b = i % 6;
    if (v) atomicAdd(&h.acc->hist[f][ll][b], (unsigned long long)(long long)v);
  }
}

// ----------------------------------------------- per-verify reset
// the accumulators (offline), the bound-event counter and the partition totals
// zeroed in one launch (three memset nodes of the graph otherwise)
__global__ void __launch_bounds__(1024) reset_kernel(DevAcc *acc, unsigned long long *nvalid, uint32_t *totals, int ntot) {
  if (acc) {
    unsigned long long *a = reinterpret_cast<unsigned long long *>(acc);
    for (int i = threadIdx.x; i < (int)(sizeof(DevAcc) / 8); i += blockDim.x) a[i] = 0;
  }
  if (threadIdx.x == 0) *nvalid = 0;
  if (totals)
    for (int i = threadIdx.x; i < ntot; i += blockDim.x) totals[i] = 0;
}

// ----------------------------------------------- finalize
__global__ void finalize_kernel(const DevProg *prog, const DevAcc *acc, DevOut *out) {
  const int f = threadIdx.x;
  if (f < (int)prog->nf) {
    const int nl = prog->nl;
    DevResult &r = out->res[f];
    unsigned long long h1[6];
    for (int v = 0; v < 6; ++v) h1[v] = acc->hist[f][1][v];
    const int root = node_verdict(prog->qkind[f][0], prog->qcmp[f][0], prog->qnum[f][0],
                                  prog->qden[f][0], h1);
    r.verdict = root;
    r.n_levels = nl;
    for (int l = 0; l <= kMaxLevels; ++l)
      for (int v = 0; v < 6; ++v)
        r.hist[l][v] = l == 0 ? (v == root ? 1ull : 0ull) : (l <= nl ? acc->hist[f][l][v] : 0ull);
    r.events_seen = acc->events_seen;
    r.events_bound = acc->events_bound;
  }
  if (f == 0) {
    out->oversize_buckets = acc->oversize_buckets;
    out->oversize_events = acc->oversize_events;
    out->table_overflow = acc->table_overflow;
    out->leaves = acc->leaves;
    for (int l = 0; l <= kMaxLevels; ++l) out->nodes[l] = acc->nodes[l];
    out->onepass = acc->onepass;
  }
}

}  // namespace

// ------------------------------------------------------------------ launchers
#define LTL4C_LAUNCH(ID, ...)                         \
  do {                                                 \
    if (L.before) L.before(L.ctx, ID);                 \
    __VA_ARGS__;                                       \
    cudaError_t e_ = cudaGetLastError();               \
    if (L.after) L.after(L.ctx, ID);                   \
    return e_;                                         \
  } while (0)

template <int K>
static cudaError_t fast_launch(const BucketParams &p, int nf, int n_sms, const Launcher &L) {
  const size_t sm = smem_bytes(K, nf, 0);
  cudaFuncSetAttribute(bucket_fast_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int per_sm = 2;  // every resident slot: the CTA per bucket is latency-bound
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bucket_fast_kernel<K>, kBucketThreads, sm) != cudaSuccess ||
      per_sm < 1)
    per_sm = 2;
  LTL4C_LAUNCH(kKBucketFast, bucket_fast_kernel<K><<<n_sms * per_sm, kBucketThreads, sm, L.stream>>>(p));
}

cudaError_t launch_bucket_fast(const BucketParams &p, int K, int nf, int n_sms, const Launcher &L) {
  switch (K) {
    case 1: return fast_launch<1>(p, nf, n_sms, L);
    case 2: return fast_launch<2>(p, nf, n_sms, L);
    default: return fast_launch<3>(p, nf, n_sms, L);
  }
}

cudaError_t launch_unit_start(const uint32_t *off, uint32_t nb, uint32_t *ustart, uint32_t n_units, const Launcher &L,
                              uint32_t target, const uint32_t *gate, int want) {
  LTL4C_LAUNCH(kKUnitStart,
               unit_start_kernel<<<(nb + 1 + 255) / 256, 256, 0, L.stream>>>(off, nb, ustart, n_units, target, gate, want));
}

template <int K, int NF, int CAP>
static size_t warp_smem(int warps, uint32_t hdr) { return hdr + (size_t)warps * sizeof(WarpTab<K, NF, CAP>); }

template <int K, int NF>
static cudaError_t warp_launch(const BucketParams &p, uint32_t grid, const Launcher &L) {
  if (p.list) {  // medium buckets: the same kernel with 4x the capacity
    const size_t sm = warp_smem<K, NF, kWarpCapBig>(p.warps_per_cta, p.warp_hdr);
    cudaFuncSetAttribute(bucket_warp_kernel<K, NF, kWarpCapBig>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    LTL4C_LAUNCH(kKBucketWarpBig, bucket_warp_kernel<K, NF, kWarpCapBig><<<grid, 32 * p.warps_per_cta, sm, L.stream>>>(p));
  }
  const size_t sm = warp_smem<K, NF, kWarpCap>(p.warps_per_cta, p.warp_hdr);
  cudaFuncSetAttribute(bucket_warp_kernel<K, NF, kWarpCap>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  LTL4C_LAUNCH(kKBucketWarp, bucket_warp_kernel<K, NF, kWarpCap><<<grid, 32 * p.warps_per_cta, sm, L.stream>>>(p));
}

// (warps per CTA, resident CTAs per SM) with the most resident warps (registers
// and shared memory both counted by the occupancy calculator)
template <int K, int NF, int CAP>
static cudaError_t warp_config_cap(uint32_t hdr, int *warps, int *ctas) {
  int best = 0;
  for (int w = 1; w <= 8; ++w) {
    const size_t sm = warp_smem<K, NF, CAP>(w, hdr);
    if (sm > 227 * 1024) break;
    cudaError_t e = cudaFuncSetAttribute(bucket_warp_kernel<K, NF, CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    int n = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, bucket_warp_kernel<K, NF, CAP>, 32 * w, sm);
    if (e != cudaSuccess) return e;
    if (n * w >= best && n > 0) { best = n * w; *warps = w; *ctas = n; }
  }
  return best ? cudaSuccess : cudaErrorInvalidConfiguration;
}

template <int K, int NF>
static cudaError_t warp_config(uint32_t hdr, int *cfg) {
  cudaError_t e = warp_config_cap<K, NF, kWarpCap>(hdr, &cfg[0], &cfg[1]);
  return e != cudaSuccess ? e : warp_config_cap<K, NF, kWarpCapBig>(hdr, &cfg[2], &cfg[3]);
}

#define LTL4C_KNF(K, NF, FN, ...)                                        \
  switch ((K) * 10 + (NF)) {                                               \
    case 11: return FN<1, 1>(__VA_ARGS__); case 12: return FN<1, 2>(__VA_ARGS__); \
    case 13: return FN<1, 3>(__VA_ARGS__); case 14: return FN<1, 4>(__VA_ARGS__); \
    case 21: return FN<2, 1>(__VA_ARGS__); case 22: return FN<2, 2>(__VA_ARGS__); \
    case 23: return FN<2, 3>(__VA_ARGS__); case 24: return FN<2, 4>(__VA_ARGS__); \
    case 31: return FN<3, 1>(__VA_ARGS__); case 32: return FN<3, 2>(__VA_ARGS__); \
    case 33: return FN<3, 3>(__VA_ARGS__); default: return FN<3, 4>(__VA_ARGS__); \
  }

cudaError_t launch_bucket_warp(const BucketParams &p, int K, int nf, uint32_t grid, const Launcher &L) {
  LTL4C_KNF(K, nf, warp_launch, p, grid, L);
}

cudaError_t bucket_warp_config(int K, int nf, int nq, int na, int *cfg) {
  LTL4C_KNF(K, nf, warp_config, warp_hdr_bytes((uint32_t)nq, (uint32_t)na), cfg);
}

uint32_t bucket_warp_hdr(int nq, int na) { return warp_hdr_bytes((uint32_t)nq, (uint32_t)na); }

template <int K, int NF>
static cudaError_t online_leaf_launch(const OnlineParams &p, uint32_t grid, const Launcher &L) {
  const size_t sm = p.b.warp_hdr + (size_t)p.b.warps_per_cta * sizeof(OnlineTab<K>);
  cudaFuncSetAttribute(online_leaf_kernel<K, NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  LTL4C_LAUNCH(kKOnlineLeaf, online_leaf_kernel<K, NF><<<grid, 32 * p.b.warps_per_cta, sm, L.stream>>>(p));
}

cudaError_t launch_online_leaf(const OnlineParams &p, int K, int nf, uint32_t grid, const Launcher &L) {
  LTL4C_KNF(K, nf, online_leaf_launch, p, grid, L);
}

template <int K, int NF>
static cudaError_t online_config_t(uint32_t hdr, int *cfg) {
  int best = 0;
  for (int w = 1; w <= 8; ++w) {
    const size_t sm = hdr + (size_t)w * sizeof(OnlineTab<K>);
    cudaError_t e = cudaFuncSetAttribute(online_leaf_kernel<K, NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    int n = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, online_leaf_kernel<K, NF>, 32 * w, sm);
    if (e != cudaSuccess) return e;
    if (n * w >= best && n > 0) { best = n * w; cfg[0] = w; cfg[1] = n; }
  }
  return best ? cudaSuccess : cudaErrorInvalidConfiguration;
}

cudaError_t online_leaf_config(int K, int nf, int nq, int na, int *cfg) {
  LTL4C_KNF(K, nf, online_config_t, warp_hdr_bytes((uint32_t)nq, (uint32_t)na), cfg);
}

cudaError_t launch_online_nodes(const OnlineParams &p, int nf, int l, uint32_t grid, const Launcher &L) {
  switch (nf) {
    case 1: LTL4C_LAUNCH(kKOnlineNodes, online_nodes_kernel<1><<<grid, 256, 0, L.stream>>>(p, l));
    case 2: LTL4C_LAUNCH(kKOnlineNodes, online_nodes_kernel<2><<<grid, 256, 0, L.stream>>>(p, l));
    case 3: LTL4C_LAUNCH(kKOnlineNodes, online_nodes_kernel<3><<<grid, 256, 0, L.stream>>>(p, l));
    default: LTL4C_LAUNCH(kKOnlineNodes, online_nodes_kernel<4><<<grid, 256, 0, L.stream>>>(p, l));
  }
}

cudaError_t launch_rehash(const DevTables &from, const DevTables &to, int n_levels, int nf,
                          unsigned long long *overflow, const Launcher &L) {
  unsigned long long mx = from.leaf_cap;
  for (int l = 1; l < n_levels; ++l) mx = mx > from.node_cap[l] ? mx : from.node_cap[l];
  dim3 grid((unsigned)((mx + 255) / 256), (unsigned)n_levels);
  LTL4C_LAUNCH(kKRehash, rehash_kernel<<<grid, 256, 0, L.stream>>>(from, to, n_levels, nf, overflow));
}


template <int K, int NQB>
static cudaError_t heavy_all(const HeavyParams &h, int nf, int n_sms, const Launcher &L) {
  if (L.before) L.before(L.ctx, kKHeavy);
  heavy_plan_kernel<<<1, 1024, 0, L.stream>>>(h);
  {
    const size_t sm = 8 * kMaxLetters + 8 * sizeof(SegTab<K>);
    cudaFuncSetAttribute(heavy_segw_kernel<K, NQB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, heavy_segw_kernel<K, NQB>, 256, sm);
    heavy_segw_kernel<K, NQB><<<n_sms * (per_sm > 0 ? per_sm : 1), 256, sm, L.stream>>>(h);
  }
  heavy_scan_blocks<<<2 * n_sms, 1024, 0, L.stream>>>(h);
  heavy_scan_sums<<<1, 1024, 0, L.stream>>>(h);
  heavy_scan_add<<<2 * n_sms, 1024, 0, L.stream>>>(h);
  heavy_group_kernel<<<4 * n_sms, 256, 0, L.stream>>>(h);
  heavy_short_kernel<K><<<4 * n_sms, 256, 0, L.stream>>>(h);
  heavy_long_kernel<K, NQB><<<n_sms, 1024, 0, L.stream>>>(h);
  for (int l = K - 1; l >= 1; --l) heavy_nodes_kernel<K><<<4 * n_sms, 256, 0, L.stream>>>(h, l);
  cudaError_t e = cudaGetLastError();
  if (L.after) L.after(L.ctx, kKHeavy);
  return e;
}

template <int K>
static cudaError_t heavy_nq(const HeavyParams &h, int nf, int nq, int n_sms, const Launcher &L) {
  if (nq <= 2) return heavy_all<K, 2>(h, nf, n_sms, L);
  if (nq <= 4) return heavy_all<K, 4>(h, nf, n_sms, L);
  if (nq <= 8) return heavy_all<K, 8>(h, nf, n_sms, L);
  return heavy_all<K, 16>(h, nf, n_sms, L);
}

cudaError_t launch_heavy(const HeavyParams &h, int K, int nf, int nq, int n_sms, const Launcher &L) {
  switch (K) {
    case 1: return heavy_nq<1>(h, nf, nq, n_sms, L);
    case 2: return heavy_nq<2>(h, nf, nq, n_sms, L);
    default: return heavy_nq<3>(h, nf, nq, n_sms, L);
  }
}

__global__ void set_u32_kernel(uint32_t *p, uint32_t v) { *p = v; }

cudaError_t launch_set_u32(uint32_t *p, uint32_t v, const Launcher &L) {
  LTL4C_LAUNCH(kKFinalize, set_u32_kernel<<<1, 1, 0, L.stream>>>(p, v));
}

cudaError_t launch_reset(DevAcc *acc, unsigned long long *nvalid, uint32_t *totals, int ntot, const Launcher &L) {
  LTL4C_LAUNCH(kKFinalize, reset_kernel<<<1, 1024, 0, L.stream>>>(acc, nvalid, totals, ntot));
}

cudaError_t launch_finalize(const DevProg *prog, const DevAcc *acc, DevOut *out, const Launcher &L) {
  LTL4C_LAUNCH(kKFinalize, finalize_kernel<<<1, 32, 0, L.stream>>>(prog, acc, out));
}

}  // namespace ltl4c
