// hot.cu -- heavy hitters of single-level properties (K = 1, offline): the
// Zipf head of a skewed trace (C3; the paper's case study 1 socket property,
// P:1113-1126, where "few objects" carry most events).
//
// A leaf of a K = 1 property is one key value; its verdict is lambda(delta*(q0,
// u^D)) (Def. 5) and delta* over a slice is the ordered composition
// of the letters' transition maps (associative).  Instead of partitioning the
// events of the most frequent keys (most of the trace under Zipf skew), they are
// composed where they lie, and only the rest of the trace is partitioned:
//
//   hot_sample    S evenly spaced events -> sample counts per key (L2 table)
//   hot_insert    the most sampled keys take a slot of the hot table: one of
//                 two 2-way buckets picked by bits of the partition hash (a key
//                 whose buckets are full stays cold: hotness only moves work);
//                 the slot index is the key's dense id
//   hot_compose   warp per contiguous chunk of the trace, 32 events per round in
//                 trace order: a hot event's letter is applied to the warp's
//                 transition map of its key (lanes sharing a key in a round are
//                 grouped by __match_any_sync and their letters applied by the
//                 lowest lane in lane order); cold events are compacted, in trace
//                 order, into the chunk's own range of a scratch buffer; each
//                 warp finally writes its chunk's map of every slot
//   hot_gather    the chunks' cold runs concatenated in chunk order: a dense
//                 cold stream, which the ordinary partition then takes as input
//   hot_finish    per slot: the chunk maps composed in chunk order, q =
//                 map(q0), lambda_f(q) -> the leaf histogram hist[f][1]
//
// Maps (the image of every start state):
//   MAPK 0 (nq <= 4 states, <= 16 letters): 2 bits per state in one byte; a
//          letter is applied through a [256][A] shared-memory table;
//   MAPK 1 (nq <= 8 states): byte q of a u64 is the image of q; (g o f) is a
//          byte permutation of g selected by f (PRMT).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"
#include "util.cuh"

namespace ltl4c {
namespace {

constexpr uint32_t kCntSalt = 0x165667b1u;   // sample-count table hash
#ifndef LTL4C_HOT_BATCH
#define LTL4C_HOT_BATCH 16
#endif
#ifndef LTL4C_HOT_MINB
#define LTL4C_HOT_MINB 4
#endif
constexpr int kHotBatch = LTL4C_HOT_BATCH;   // rounds of 32 events whose loads are issued together

__device__ __forceinline__ uint32_t sel_of(uint32_t f) {  // bytes b0..b3 (< 8) -> nibbles b0 | b1 << 4 | ...
  const uint32_t x = f | (f >> 4);
  return __byte_perm(x, 0u, 0x4420u);
}
// (g o f) on byte-form maps: (g o f)[q] = g[f[q]]
__device__ __forceinline__ uint32_t byte_apply(uint32_t g, uint32_t f) { return __byte_perm(g, 0u, sel_of(f)); }
__device__ __forceinline__ unsigned long long byte_apply(unsigned long long g, unsigned long long f) {
  const uint32_t glo = (uint32_t)g, ghi = (uint32_t)(g >> 32);
  const uint32_t lo = __byte_perm(glo, ghi, sel_of((uint32_t)f));
  const uint32_t hi = __byte_perm(glo, ghi, sel_of((uint32_t)(f >> 32)));
  return (unsigned long long)hi << 32 | lo;
}

// a key's two candidate 2-way buckets of the hot table (two choices keep the
// table nearly collision-free at load 3/4): the LOW bits of the partition hash
// (a partition bucket is its HIGH bits) and bits 12.. of it
__device__ __forceinline__ uint32_t hot_bucket1(uint32_t h, int slots) { return (h & (uint32_t)(slots / 2 - 1)) * 2; }
__device__ __forceinline__ uint32_t hot_bucket2(uint32_t h, int slots) {
  return ((h >> 12) & (uint32_t)(slots / 2 - 1)) * 2;
}

template <int MAPK> struct HotMap;
template <> struct HotMap<0> {
  using T = uint8_t;                              // packed: bits 2q..2q+1 = image of q
  using B = uint32_t;                             // byte form used by hot_finish
  static constexpr int kSlots = kHotSlotsMax;
  __device__ static T ident() { return 0xE4; }    // 3 2 1 0
};
template <> struct HotMap<1> {
  using T = unsigned long long;                   // byte form
  using B = unsigned long long;
  static constexpr int kSlots = kHotSlotsMax / 4;
  __device__ static T ident() { return 0x0706050403020100ull; }
};

// a CTA aggregates its kSampleBlock samples in a shared-memory table first, so a
// hot key costs one global atomic per CTA (not one per sample); a thread's
// samples are loaded together
#ifndef LTL4C_SAMPLE_PER
#define LTL4C_SAMPLE_PER 2
#endif
constexpr int kSampleThreads = 256, kSamplePer = LTL4C_SAMPLE_PER;
constexpr int kSampleBlock = kSampleThreads * kSamplePer, kSampleTab = 2 * kSampleBlock;
__global__ void __launch_bounds__(kSampleThreads) hot_sample_kernel(HotParams hp) {
  __shared__ uint32_t tk[kSampleTab], tc[kSampleTab];
  for (int i = threadIdx.x; i < kSampleTab; i += blockDim.x) { tk[i] = kAbsent; tc[i] = 0; }
  const unsigned long long n = hp.n;
  uint32_t kv[kSamplePer];
#pragma unroll
  for (int q = 0; q < kSamplePer; ++q) {
    const uint32_t i = blockIdx.x * kSampleBlock + q * kSampleThreads + threadIdx.x;
    kv[q] = i < hp.n_samples ? hp.k0[(unsigned long long)i * n / (unsigned long long)hp.n_samples] : kAbsent;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kSamplePer; ++q) {
    const uint32_t k = kv[q];
    if (k == kAbsent) continue;
    uint32_t h = fmix32(k ^ kCntSalt) & (kSampleTab - 1);
    while (true) {  // (at most kSampleBlock < kSampleTab keys)
      uint32_t t = tk[h];
      if (t == kAbsent) {
        const uint32_t o = atomicCAS(&tk[h], kAbsent, k);
        t = o == kAbsent ? k : o;
      }
      if (t == k) { atomicAdd(&tc[h], 1u); break; }
      h = (h + 1) & (kSampleTab - 1);
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < kSampleTab; x += blockDim.x) {
    const uint32_t k = tk[x];
    if (k == kAbsent) continue;
    uint32_t h = fmix32(k ^ kCntSalt) & (hp.cnt_cap - 1);
    for (uint32_t probes = 0; probes < hp.cnt_cap; ++probes) {
      uint32_t t = hp.cnt_key[h];
      if (t == kAbsent) {
        const uint32_t o = atomicCAS(&hp.cnt_key[h], kAbsent, k);
        t = o == kAbsent ? k : o;
      }
      if (t == k) { atomicAdd(&hp.cnt_val[h], tc[x]); break; }
      h = (h + 1) & (hp.cnt_cap - 1);
    }
  }
}

// histogram of the sample counts (bin 63 = 63 or more; bins 1, 2: the sample's
// singletons / doubletons), per CTA in shared memory first
__global__ void __launch_bounds__(256) hot_count_hist_kernel(HotParams hp) {
  __shared__ uint32_t bin[64];
  if (threadIdx.x < 64) bin[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < hp.cnt_cap; s += gridDim.x * blockDim.x) {
    const uint32_t c = hp.cnt_val[s];
    if (c >= 1) atomicAdd(&bin[min(c, 63u)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 64 && bin[threadIdx.x]) atomicAdd(&hp.nhot[8 + threadIdx.x], bin[threadIdx.x]);
}

// keys sampled >= t times, t the smallest threshold >= kHotMinCount leaving at
// most 3/4 of the slots wanted, take a slot of their bucket; the most sampled
// first (pass 0: counts >= 4t, pass 1: the rest).  nhot[0] = keys inserted,
// nhot[1] = their sampled events.
__global__ void hot_insert_kernel(HotParams hp, int pass) {
  __shared__ uint32_t thr, bins[64];
  if (threadIdx.x < 64) bins[threadIdx.x] = hp.nhot[8 + threadIdx.x];  // (one load each, not 64 in a chain)
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t want = (uint32_t)hp.slots * 3 / 4;
    uint32_t t = 64, tot = 0;
    while (t > (uint32_t)kHotMinCount && tot + bins[t - 1] <= want) tot += bins[--t];
    thr = t;  // keys with count >= t (bin t - 1 and below did not fit)
  }
  __syncthreads();
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= hp.cnt_cap || thr >= 64) return;
  const uint32_t c = hp.cnt_val[s];
  if (pass == 0 ? c < 4 * thr : (c < thr || c >= 4 * thr)) return;
  const uint32_t k = hp.cnt_key[s];
  const uint32_t h = fmix32(k ^ kBucketSalt);
  const uint32_t b1 = hot_bucket1(h, hp.slots), b2 = hot_bucket2(h, hp.slots);
  for (int i = 0; i < 4; ++i)
    if (atomicCAS(&hp.slot_key[(i < 2 ? b1 : b2) + (i & 1)], kAbsent, k) == kAbsent) {
      atomicAdd(hp.nhot, 1u);
      atomicAdd(hp.nhot + 1, c);
      return;
    }
}

// The batch's mode, from the sample (one thread):
//   nhot[2] (dense) = the hot keys carry >= 1/4 of the sampled events: they are
//     composed where they lie and the rest is compacted into the cold stream;
//     otherwise nothing is hot and the partition reads the batch itself;
//   nhot[3] (one pass) = the cold keys are few enough for 512 coarse buckets of
//     <= ~1500 keys each: Chao1 over the sample's cold keys (D + f1^2 / 2 f2,
//     f1 / f2 = keys sampled once / twice) <= kOnePassKeys.  A coarse bucket that
//     still overflows its CTA table goes to the heavy path (same result).
__global__ void hot_decide_kernel(HotParams hp) {
  if (threadIdx.x || blockIdx.x) return;
  const uint32_t *bin = hp.nhot + 8;
  const bool dense = 4ull * hp.nhot[1] >= (unsigned long long)hp.n_samples && hp.nhot[0] > 0;
  unsigned long long d = 0;
  for (int c = 1; c < 64; ++c) d += bin[c];
  if (dense) d -= min(d, (unsigned long long)hp.nhot[0]);
  const double f1 = bin[1], f2 = bin[2] > 0 ? bin[2] : 1;
  const double chao1 = (double)d + f1 * f1 / (2.0 * f2);
  hp.nhot[2] = dense ? 1u : 0u;
  hp.nhot[3] = hp.force_onepass || chao1 <= (double)kOnePassKeys ? 1u : 0u;
}

template <int MAPK>
struct HotSmem {
  using M = typename HotMap<MAPK>::T;
  static constexpr int S = HotMap<MAPK>::kSlots;
  uint32_t key[S];                          // slot -> hot key (ABSENT: empty)
  M wmap[kHotCtaWarps][S];                  // each warp's map of every slot over its chunk so far
  uint8_t stage[kHotCtaWarps][32];          // the round's letters
  // MAPK 0: [256][A] letter table; MAPK 1: [A] letter maps
  alignas(16) uint8_t tab[MAPK == 0 ? 256 * 16 : 8 * kMaxLetters];
};

// One warp per contiguous chunk [e0, e1) of the batch (multiple of 512 events).
template <int MAPK>
__global__ void __launch_bounds__(32 * kHotCtaWarps, LTL4C_HOT_MINB) hot_compose_kernel(HotParams hp) {
  using HM = HotMap<MAPK>;
  using M = typename HM::T;
  constexpr int S = HM::kSlots;
  extern __shared__ __align__(16) uint8_t raw[];
  // not dense (no key carries enough of the sample): nothing is composed here and the
  // partition reads the batch itself -- leave before staging any table
  if (hp.nhot[2] == 0) return;
  HotSmem<MAPK> &s = *reinterpret_cast<HotSmem<MAPK> *>(raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const DevProg *prog = hp.prog;
  const int A = 1 << prog->na, nq = prog->nq;
  for (int i = tid; i < S; i += blockDim.x) s.key[i] = hp.slot_key[i];
  if (MAPK == 0) {
    for (int i = tid; i < 256 * A; i += blockDim.x) {
      const uint32_t m = (uint32_t)i / A, a = (uint32_t)i % A;
      uint32_t o = 0;
      for (int q = 0; q < 4; ++q) {
        const uint32_t img = (m >> (2 * q)) & 3u;
        o |= (img < (uint32_t)nq ? (uint32_t)prog->delta[img][a] & 3u : img) << (2 * q);
      }
      s.tab[i] = (uint8_t)o;
    }
  } else {
    unsigned long long *smap = reinterpret_cast<unsigned long long *>(s.tab);
    for (int a = tid; a < A; a += blockDim.x) {
      unsigned long long m = HotMap<1>::ident();
      for (int q = 0; q < nq; ++q) m = (m & ~(0xFFull << (8 * q))) | ((unsigned long long)prog->delta[q][a] << (8 * q));
      smap[a] = m;
    }
  }
  for (int i = lane; i < S; i += 32) s.wmap[wid][i] = HM::ident();
  __syncthreads();
  const bool dense = hp.nhot[2] != 0;  // not dense: nothing composed, the partition reads the batch itself
  const uint32_t chunk = blockIdx.x * kHotCtaWarps + wid;
  const unsigned long long n = hp.n;
  const unsigned long long e0 = (unsigned long long)chunk * hp.chunk_ev;
  const unsigned long long e1 = min(n, e0 + hp.chunk_ev);
  M *wmap = s.wmap[wid];
  uint8_t *stage = s.stage[wid];
  const uint8_t *tab = s.tab;
  const unsigned long long *smap = reinterpret_cast<const unsigned long long *>(s.tab);
  const uint32_t let_mask = hp.let_mask;
  uint32_t ncold = 0, nhot = 0;  // warp-uniform
  if (dense && chunk < (uint32_t)hp.n_chunks) {
    for (unsigned long long r0 = e0; r0 < e1; r0 += 32 * kHotBatch) {
      uint32_t kk[kHotBatch];
      uint8_t ll[kHotBatch];
#pragma unroll
      for (int r = 0; r < kHotBatch; ++r) {  // every load of the batch first (memory-level parallelism)
        const unsigned long long j = r0 + r * 32 + lane;
        const bool in = j < e1;
        kk[r] = in ? __ldcs(&hp.k0[j]) : kAbsent;
        ll[r] = in ? (uint8_t)(__ldcs(&hp.let[j]) & let_mask) : (uint8_t)0;
      }
#pragma unroll
      for (int r = 0; r < kHotBatch; ++r) {
        const uint32_t k = kk[r];
        const bool valid = k != kAbsent;
        const uint32_t h = fmix32(k ^ kBucketSalt);
        const uint32_t b1 = hot_bucket1(h, S), b2 = hot_bucket2(h, S);
        const uint2 t1 = *reinterpret_cast<const uint2 *>(&s.key[b1]);
        const uint2 t2 = *reinterpret_cast<const uint2 *>(&s.key[b2]);
        const int slot = !valid       ? -1
                         : t1.x == k ? (int)b1
                         : t1.y == k ? (int)b1 + 1
                         : t2.x == k ? (int)b2
                         : t2.y == k ? (int)b2 + 1
                                     : -1;
        const bool cold = valid && slot < 0;
        const uint32_t cm = __ballot_sync(0xffffffffu, cold);
        if (cold) {
          const unsigned long long p = e0 + ncold + __popc(cm & lanemask_lt());
          hp.cold_key[p] = k;
          hp.cold_let[p] = ll[r];
        }
        ncold += __popc(cm);
        const uint32_t hm = __ballot_sync(0xffffffffu, slot >= 0);
        nhot += __popc(hm);
        if (hm) {
          stage[lane] = ll[r];
          __syncwarp();
          if (slot >= 0) {
            const uint32_t peers = __match_any_sync(hm, (uint32_t)slot);
            if ((peers & lanemask_lt()) == 0) {  // lowest lane of its group: the letters in lane order
              M m = wmap[slot];
              uint32_t pm = peers;
              do {
                const int i = __ffs(pm) - 1;
                pm &= pm - 1;
                if (MAPK == 0) m = (M)tab[(uint32_t)m * A + stage[i]];
                else m = (M)byte_apply(smap[stage[i]], (unsigned long long)m);
              } while (pm);
              wmap[slot] = m;
            }
          }
          __syncwarp();
        }
      }
    }
  }
  __syncwarp();
  if (chunk < (uint32_t)hp.n_chunks) {
    if (dense) {
      M *out = reinterpret_cast<M *>(hp.partial) + (size_t)chunk * S;
      if (MAPK == 0) {
        const uint32_t *w4 = reinterpret_cast<const uint32_t *>(wmap);
        uint32_t *o4 = reinterpret_cast<uint32_t *>(out);
        for (int i = lane; i < S / 4; i += 32) o4[i] = w4[i];
      } else {
        for (int i = lane; i < S; i += 32) out[i] = wmap[i];
      }
    }
    if (lane == 0) {
      hp.chunk_cold[chunk] = ncold;
      if (ncold) atomicAdd(hp.n_cold, (unsigned long long)ncold);
      if (nhot) atomicAdd(&hp.acc->events_bound, (unsigned long long)nhot);
    }
  }
}

// exclusive prefix of the chunks' cold counts (one CTA) -> chunk_pre
__global__ void __launch_bounds__(1024) hot_prefix_kernel(HotParams hp) {
  __shared__ uint32_t wsum[32];
  if (hp.nhot[2] == 0) return;  // (not dense: no cold runs)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nc = hp.n_chunks, per = (nc + 1023) / 1024;
  const int c0 = min(nc, tid * per), c1 = min(nc, c0 + per);
  uint32_t sum = 0;
  for (int c = c0; c < c1; ++c) sum += hp.chunk_cold[c];
  uint32_t inc = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = wsum[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  uint32_t run = inc - sum + (wid ? wsum[wid - 1] : 0u);
  for (int c = c0; c < c1; ++c) {
    hp.chunk_pre[c] = run;
    run += hp.chunk_cold[c];
  }
}

// kGatherParts CTAs per chunk move its cold run to the dense stream (4 elements
// per thread in flight)
constexpr int kGatherParts = 4;
__global__ void __launch_bounds__(256) hot_gather_kernel(HotParams hp) {
  const uint32_t chunk = blockIdx.x / kGatherParts, part = blockIdx.x % kGatherParts;
  if (chunk >= (uint32_t)hp.n_chunks || hp.nhot[2] == 0) return;
  const uint32_t cnt = hp.chunk_cold[chunk];
  const uint32_t per = (cnt + kGatherParts - 1) / kGatherParts;
  const uint32_t lo = min(cnt, part * per), hi = min(cnt, lo + per);
  const unsigned long long src = (unsigned long long)chunk * hp.chunk_ev;
  const uint32_t *sk = hp.cold_key + src;
  const uint8_t *sl = hp.cold_let + src;
  uint32_t *dk = hp.dense_key + hp.chunk_pre[chunk];
  uint8_t *dl = hp.dense_let + hp.chunk_pre[chunk];
  for (uint32_t i = lo + threadIdx.x; i < hi; i += 4 * blockDim.x) {
    uint32_t k[4];
    uint8_t l[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t x = i + u * blockDim.x;
      k[u] = x < hi ? __ldcs(&sk[x]) : 0u;
      l[u] = x < hi ? __ldcs(&sl[x]) : (uint8_t)0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t x = i + u * blockDim.x;
      if (x < hi) { dk[x] = k[u]; dl[x] = l[u]; }
    }
  }
}

// per slot (x: 32 consecutive slots, y: 32 ranges of chunks): the chunk maps in
// chunk order, then the leaf's verdicts (Def. 5) into the leaf histogram
template <int MAPK>
__global__ void __launch_bounds__(1024) hot_finish_kernel(HotParams hp) {
  using HM = HotMap<MAPK>;
  using M = typename HM::T;
  using Bm = typename HM::B;
  constexpr int S = HM::kSlots;
  constexpr int kU = 4;
  __shared__ Bm part[32][33];
  __shared__ uint32_t unpack[256];
  __shared__ uint32_t sacc[kMaxFormulas * 6];
  if (hp.nhot[2] == 0) return;  // (not dense: no hot key was composed)
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kMaxFormulas * 6; i += blockDim.x) sacc[i] = 0;
  if (MAPK == 0)
    for (int m = threadIdx.x; m < 256; m += blockDim.x) {
      uint32_t o = 0;
      for (int q = 0; q < 4; ++q) o |= ((m >> (2 * q)) & 3u) << (8 * q);
      unpack[m] = o;
    }
  __syncthreads();
  const DevProg *prog = hp.prog;
  const int slot = blockIdx.x * 32 + tx;
  const int nc = hp.n_chunks, per = (nc + 31) / 32;
  const int c0 = min(nc, ty * per), c1 = min(nc, c0 + per);
  const M *partial = reinterpret_cast<const M *>(hp.partial);
  Bm m = (Bm)HotMap<1>::ident();
  for (int c = c0; c < c1; c += kU) {
    M x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) x[u] = c + u < c1 ? partial[(size_t)(c + u) * S + slot] : HM::ident();
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      Bm f;
      if (MAPK == 0) f = (Bm)unpack[(uint32_t)x[u]];
      else f = (Bm)x[u];
      m = byte_apply(f, m);
    }
  }
  part[ty][tx] = m;
  __syncthreads();
  if (ty == 0 && hp.slot_key[slot] != kAbsent) {
    Bm t = part[0][tx];
    for (int g = 1; g < 32; ++g) t = byte_apply(part[g][tx], t);
    const uint32_t q = (uint32_t)(t >> (8 * prog->q0)) & 0xFFu;
    for (uint32_t f = 0; f < prog->nf; ++f) atomicAdd(&sacc[f * 6 + prog->lab[f][q]], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxFormulas * 6; i += blockDim.x)
    if (sacc[i]) atomicAdd(&hp.acc->hist[i / 6][1][i % 6], (unsigned long long)sacc[i]);
}

}  // namespace

#define LTL4C_LAUNCH(ID, ...)           \
  do {                                   \
    if (L.before) L.before(L.ctx, ID);   \
    __VA_ARGS__;                         \
    cudaError_t e_ = cudaGetLastError(); \
    if (L.after) L.after(L.ctx, ID);     \
    return e_;                           \
  } while (0)

int hot_slots(int mapk) { return mapk == 0 ? HotMap<0>::kSlots : HotMap<1>::kSlots; }
int hot_map_bytes(int mapk) { return mapk == 0 ? 1 : 8; }

cudaError_t launch_hot_select(const HotParams &hp, const Launcher &L) {
  if (L.before) L.before(L.ctx, kKHot);
  hot_sample_kernel<<<(hp.n_samples + kSampleBlock - 1) / kSampleBlock, 256, 0, L.stream>>>(hp);
  hot_count_hist_kernel<<<std::min<uint32_t>((hp.cnt_cap + 255) / 256, 148 * 4), 256, 0, L.stream>>>(hp);
  hot_insert_kernel<<<(hp.cnt_cap + 255) / 256, 256, 0, L.stream>>>(hp, 0);
  hot_insert_kernel<<<(hp.cnt_cap + 255) / 256, 256, 0, L.stream>>>(hp, 1);
  hot_decide_kernel<<<1, 32, 0, L.stream>>>(hp);
  cudaError_t e = cudaGetLastError();
  if (L.after) L.after(L.ctx, kKHot);
  return e;
}

template <int MAPK>
static cudaError_t compose_t(const HotParams &hp, const Launcher &L) {
  const size_t sm = sizeof(HotSmem<MAPK>);
  cudaFuncSetAttribute(hot_compose_kernel<MAPK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int grid = (hp.n_chunks + kHotCtaWarps - 1) / kHotCtaWarps;
  LTL4C_LAUNCH(kKHotCompose, hot_compose_kernel<MAPK><<<grid, 32 * kHotCtaWarps, sm, L.stream>>>(hp));
}

cudaError_t launch_hot_compose(const HotParams &hp, const Launcher &L) {
  cudaError_t e = hp.mapk == 0 ? compose_t<0>(hp, L) : compose_t<1>(hp, L);
  if (e != cudaSuccess) return e;
  if (L.before) L.before(L.ctx, kKHot);
  hot_prefix_kernel<<<1, 1024, 0, L.stream>>>(hp);
  hot_gather_kernel<<<hp.n_chunks * kGatherParts, 256, 0, L.stream>>>(hp);
  e = cudaGetLastError();
  if (L.after) L.after(L.ctx, kKHot);
  return e;
}

cudaError_t launch_hot_finish(const HotParams &hp, const Launcher &L) {
  if (hp.mapk == 0) LTL4C_LAUNCH(kKHot, hot_finish_kernel<0><<<HotMap<0>::kSlots / 32, 1024, 0, L.stream>>>(hp));
  LTL4C_LAUNCH(kKHot, hot_finish_kernel<1><<<HotMap<1>::kSlots / 32, 1024, 0, L.stream>>>(hp));
}

int hot_ctas_per_sm(int mapk) {
  int n = 1;
  if (mapk == 0) {
    cudaFuncSetAttribute(hot_compose_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HotSmem<0>));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, hot_compose_kernel<0>, 32 * kHotCtaWarps, sizeof(HotSmem<0>));
  } else {
    cudaFuncSetAttribute(hot_compose_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HotSmem<1>));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, hot_compose_kernel<1>, 32 * kHotCtaWarps, sizeof(HotSmem<1>));
  }
  return n > 0 ? n : 1;
}

}  // namespace ltl4c
