// hot.cu -- heavy hitters of single-level properties (K = 1, offline): the
// Zipf head of a skewed trace (C3; the paper's case study 1 socket property,
// P:1113-1126, where "few objects" carry most events).
//
// A leaf of a K = 1 property is one key value; its verdict is lambda(delta*(q0,
// u^D)) (Def. 5) and delta* over a slice is the ordered composition
// of the letters' transition maps (associative).  Instead of partitioning the
// events of the most frequent keys (most of the trace under Zipf skew), they are
// composed where they lie:
//
//   hot_sample   S evenly spaced events -> sample counts per key (L2 table)
//   hot_select   keys with >= kHotMinCount samples -> hot table (<= kHotKeys)
//   part_count_hot  the first partition pass's counting kernel as persistent
//                CTAs over contiguous tile ranges: cold events are counted by
//                digit as usual; a hot event's letter map is composed, in trace
//                order, onto its warp's map of that key (lanes sharing a key in
//                a round are grouped by __match_any_sync and their maps composed
//                in lane order); at the end of a tile the warps' maps are
//                composed onto the CTA's map in warp order; each CTA writes its
//                chunk's map per hot key
//   (the first scatter pass drops hot events: they never enter the partition)
//   hot_finish   per hot key: the CTA chunk maps composed in chunk order (an
//                ordered shuffle tree), q = map(q0), lambda_f(q) -> the leaf
//                histogram hist[f][1]
// Which keys are hot does not change the result (each key is wholly hot or
// wholly cold); the sample only decides where the work goes.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "util.cuh"

namespace ltl4c {
namespace {

constexpr uint32_t kCntSalt = 0x165667b1u;   // sample-count table hash

// Transition maps of monitors with at most NQB (<= 8) states in byte form: byte q
// is the image of state q (u32 for NQB <= 4, u64 for NQB <= 8).  (g o f)[q] =
// g[f[q]] is a byte permutation of g selected by f: PRMT with f's bytes packed
// into selector nibbles.
template <int NQB> struct HotMap { using T = uint32_t; };
template <> struct HotMap<8> { using T = unsigned long long; };

__device__ __forceinline__ uint32_t sel_of(uint32_t f) {  // bytes b0..b3 (< 8) -> nibbles b0 | b1 << 4 | ...
  const uint32_t x = f | (f >> 4);
  return __byte_perm(x, 0u, 0x4420u);
}
__device__ __forceinline__ uint32_t hot_apply(uint32_t g, uint32_t f) { return __byte_perm(g, 0u, sel_of(f)); }
__device__ __forceinline__ unsigned long long hot_apply(unsigned long long g, unsigned long long f) {
  const uint32_t glo = (uint32_t)g, ghi = (uint32_t)(g >> 32);
  const uint32_t lo = __byte_perm(glo, ghi, sel_of((uint32_t)f));
  const uint32_t hi = __byte_perm(glo, ghi, sel_of((uint32_t)(f >> 32)));
  return (unsigned long long)hi << 32 | lo;
}
template <int NQB>
__device__ __forceinline__ typename HotMap<NQB>::T hot_ident() {
  return (typename HotMap<NQB>::T)0x0706050403020100ull;
}
template <int NQB>
__device__ __forceinline__ uint32_t hot_image(typename HotMap<NQB>::T m, uint32_t q) {
  return (uint32_t)(m >> (8 * q)) & 0xFFu;
}

__global__ void hot_sample_kernel(HotParams hp) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long n = hp.n;
  if (i >= (uint32_t)kHotSamples || n == 0) return;
  const unsigned long long j = (unsigned long long)i * n / (unsigned long long)kHotSamples;
  const uint32_t k = hp.k0[j];
  if (k == kAbsent) return;
  uint32_t h = fmix32(k ^ kCntSalt) & (kHotCountCap - 1);
  for (int probes = 0; probes < kHotCountCap; ++probes) {
    uint32_t t = hp.cnt_key[h];
    if (t == kAbsent) {
      const uint32_t o = atomicCAS(&hp.cnt_key[h], kAbsent, k);
      t = o == kAbsent ? k : o;
    }
    if (t == k) {
      atomicAdd(&hp.cnt_val[h], 1u);
      return;
    }
    h = (h + 1) & (kHotCountCap - 1);
  }
}

// the most sampled keys are hot: a histogram of the sample counts (bin 63 = 63 or
// more) gives the smallest threshold t >= kHotMinCount with at most kHotKeys keys
// counted >= t
__global__ void hot_count_hist_kernel(HotParams hp) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= (uint32_t)kHotCountCap) return;
  const uint32_t c = hp.cnt_val[s];
  if (c >= (uint32_t)kHotMinCount) atomicAdd(&hp.nhot[1 + min(c, 63u)], 1u);
}

// keys counted >= t get a dense id and a slot of their table bucket (a key whose
// bucket is full stays cold: hotness only moves work)
__global__ void hot_select_kernel(HotParams hp) {
  __shared__ uint32_t thr;
  if (threadIdx.x == 0) {
    uint32_t t = 64, tot = 0;
    while (t > (uint32_t)kHotMinCount && tot + hp.nhot[1 + t - 1] <= (uint32_t)kHotKeys) tot += hp.nhot[1 + --t];
    thr = t;  // keys with count >= t (bin t - 1 and below did not fit)
  }
  __syncthreads();
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= (uint32_t)kHotCountCap || hp.cnt_val[s] < thr || thr >= 64) return;
  const uint32_t k = hp.cnt_key[s];
  const uint32_t id = atomicAdd(hp.nhot, 1u);
  if (id >= (uint32_t)kHotKeys) return;
  const uint32_t b = hot_bucket(k);
  for (int i = 0; i < 4; ++i) {
    if (atomicCAS(&hp.hot[4 * b + i], kAbsent, k) == kAbsent) {
      hp.hid[4 * b + i] = (uint16_t)id;
      hp.key_of[id] = k;
      return;
    }
  }
}

constexpr int kHotCtaWarps = 8;
template <int NQB>
struct HotSmem {
  using M = typename HotMap<NQB>::T;
  uint4 hot[kHotBuckets];                  // the hot table (4 keys per bucket)
  uint16_t hid[kHotBuckets * 4];
  M smap[kMaxLetters];                     // letter maps
  M wmap[kHotCtaWarps][kHotKeys];          // each warp's map of every hot key over its chunk so far
  uint32_t hist[kHotCtaWarps][kMaxDigits]; // each warp's digit counts of its current tile
  M stage[kHotCtaWarps][32];
};

// dense hot id of key k (partition hash h), or -1 (one 16-byte shared-memory probe)
__device__ __forceinline__ int hot_id(const uint4 *tab, const uint16_t *hid, uint32_t k, uint32_t h) {
  const uint32_t b = hot_bucket_of_hash(h);
  const uint4 v = tab[b];
  const int i = v.x == k ? 0 : v.y == k ? 1 : v.z == k ? 2 : v.w == k ? 3 : -1;
  return i < 0 ? -1 : (int)hid[4 * b + i];
}

// The first partition pass's count kernel with the hot keys composed on the fly
// (K = 1).  Every WARP owns a contiguous range of tiles (a chunk) and walks it in
// trace order, 32 events per round: cold events are counted by digit into the
// warp's histogram of the tile (written to counts[d][tile] at the tile's end);
// lanes holding a hot key are grouped by __match_any_sync, the group's letter
// maps composed in lane (= trace) order by its lowest lane and that onto the
// warp's map of the key.  Each round's hot ballot goes to hp.mask (the first
// scatter pass drops those events); each warp finally writes its chunk's maps.
template <int NQB>
__global__ void __launch_bounds__(256, 3) part_count_hot_kernel(PartPlan pl, HotParams hp) {
  using M = typename HotMap<NQB>::T;
  constexpr int kBatch = 16;  // rounds whose loads are issued together
  extern __shared__ __align__(16) uint8_t raw[];
  HotSmem<NQB> &s = *reinterpret_cast<HotSmem<NQB> *>(raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const M ident = hot_ident<NQB>();
  const DevProg *prog = hp.prog;
  const int A = 1 << prog->na, nq = prog->nq;
  for (int i = tid; i < kHotBuckets; i += blockDim.x) s.hot[i] = reinterpret_cast<const uint4 *>(hp.hot)[i];
  for (int i = tid; i < kHotBuckets * 4; i += blockDim.x) s.hid[i] = hp.hid[i];
  for (int a = tid; a < A; a += blockDim.x) {
    M m = ident;
    for (int q = 0; q < nq; ++q) m = (m & ~((M)0xFF << (8 * q))) | ((M)prog->delta[q][a] << (8 * q));
    s.smap[a] = m;
  }
  for (int i = lane; i < kHotKeys; i += 32) s.wmap[wid][i] = ident;
  __syncthreads();
  const bool any_hot = *hp.nhot > 0;
  const uint32_t *in_k0 = pl.in_key[0];
  const uint8_t *in_let = pl.in_let;
  const unsigned long long n = pl.n;
  const uint32_t dmask = (1u << pl.width[0]) - 1u;
  const int lo = pl.lo[0];
  const uint32_t chunk = blockIdx.x * kHotCtaWarps + wid;
  const uint32_t per = (pl.n_tiles + hp.n_chunks - 1) / hp.n_chunks;
  const uint32_t t0 = chunk * per;
  uint32_t *hist = s.hist[wid];
  M *wmap = s.wmap[wid];
  M *stage = s.stage[wid];
  const uint32_t shift = 32 - pl.bits;  // (K = 1 batches have bits >= 1)
  uint32_t my_cold = 0, my_bound = 0;     // warp-uniform
  // trip counts are the same in every warp (collectives stay provably convergent):
  // a warp's tiles past the batch just see no events
  for (uint32_t i = 0; i < per; ++i) {
    const uint32_t tile = t0 + i;
    for (int d = lane; d < kMaxDigits; d += 32) hist[d] = 0;
    __syncwarp();
    const unsigned long long tbase = (unsigned long long)tile * kTileEv;
    const uint32_t tn = tbase < n ? (uint32_t)min((unsigned long long)kTileEv, n - tbase) : 0u;  // events of the tile
    const uint32_t *tk = in_k0 + tbase;
    const uint8_t *tl = in_let + tbase;
    for (uint32_t r0 = 0; r0 < (uint32_t)kTileEv; r0 += 32 * kBatch) {
      uint32_t kk[kBatch];
      uint8_t ll[kBatch];
#pragma unroll
      for (int r = 0; r < kBatch; ++r) {  // every load of the batch first (memory-level parallelism)
        const uint32_t j = r0 + r * 32 + lane;
        const bool in = j < tn;
        kk[r] = in ? __ldcs(&tk[j]) : kAbsent;
        ll[r] = in ? (uint8_t)(__ldcs(&tl[j]) & pl.let_mask) : (uint8_t)0;
      }
      uint32_t hmask = 0;  // lane r: the hot ballot of round r
#pragma unroll
      for (int r = 0; r < kBatch; ++r) {
        const uint32_t k = kk[r];
        const bool valid = k != kAbsent;
        const uint32_t h = fmix32(k ^ pl.salt);
        const int id = valid && any_hot ? hot_id(s.hot, s.hid, k, h) : -1;
        const bool cold = valid && id < 0;
        if (cold) atomicAdd(&hist[(h >> shift >> lo) & dmask], 1u);
        my_bound += __popc(__ballot_sync(0xffffffffu, valid));
        my_cold += __popc(__ballot_sync(0xffffffffu, cold));
        const uint32_t hm = __ballot_sync(0xffffffffu, id >= 0);
        if (lane == r) hmask = hm;
        if (hm) {
          stage[lane] = s.smap[ll[r]];
          const uint32_t peers = __match_any_sync(0xffffffffu, id);
          __syncwarp();
          if (id >= 0 && (peers & lanemask_lt()) == 0) {
            M m = stage[lane];
            uint32_t pm = peers & (peers - 1);
            while (pm) {
              const int i = __ffs(pm) - 1;
              pm &= pm - 1;
              m = hot_apply(stage[i], m);
            }
            wmap[id] = hot_apply(m, wmap[id]);
          }
          __syncwarp();
        }
      }
      if (lane < kBatch && r0 + 32 * lane < tn) hp.mask[((tbase + r0) >> 5) + lane] = hmask;
    }
    __syncwarp();
    if (tile < pl.n_tiles)
      for (uint32_t d = lane; d <= dmask; d += 32) pl.counts[(size_t)d * pl.n_tiles + tile] = hist[d];
    __syncwarp();
  }
  if (chunk < (uint32_t)hp.n_chunks)
    for (int i = lane; i < kHotKeys; i += 32) reinterpret_cast<M *>(hp.partial)[(size_t)chunk * kHotKeys + i] = wmap[i];
  if (lane == 0) {
    if (my_cold) atomicAdd(pl.nvalid, (unsigned long long)my_cold);
    if (my_bound) atomicAdd(&pl.acc->events_bound, (unsigned long long)my_bound);
  }
}

// per hot key (a warp each): the chunk maps composed in chunk order, the leaf's
// verdicts (Def. 5) into the leaf histogram
template <int NQB>
__global__ void __launch_bounds__(256) hot_finish_kernel(HotParams hp, int n_chunks) {
  using M = typename HotMap<NQB>::T;
  __shared__ uint32_t sacc[kMaxFormulas * 6];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kMaxFormulas * 6; i += blockDim.x) sacc[i] = 0;
  __syncthreads();
  const DevProg *prog = hp.prog;
  const M ident = hot_ident<NQB>();
  const M *partial = reinterpret_cast<const M *>(hp.partial);
  const int id = blockIdx.x * (blockDim.x >> 5) + wid;
  if (id < kHotKeys && hp.key_of[id] != kAbsent) {
    const int per = (n_chunks + 31) / 32;
    const int c0 = min(n_chunks, lane * per), c1 = min(n_chunks, c0 + per);
    M m = ident;
    for (int c = c0; c < c1; ++c) m = hot_apply(partial[(size_t)c * kHotKeys + id], m);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {  // ordered tree: lane l's range precedes lane l + d's
      const M o = __shfl_down_sync(0xffffffffu, m, d);
      if ((lane & (2 * d - 1)) == 0) m = hot_apply(o, m);
    }
    if (lane == 0) {
      const uint32_t q = hot_image<NQB>(m, prog->q0);
      for (uint32_t f = 0; f < prog->nf; ++f) atomicAdd(&sacc[f * 6 + prog->lab[f][q]], 1u);
    }
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

cudaError_t launch_hot_select(const HotParams &hp, const Launcher &L) {
  if (L.before) L.before(L.ctx, kKHot);
  hot_sample_kernel<<<kHotSamples / 256, 256, 0, L.stream>>>(hp);
  hot_count_hist_kernel<<<kHotCountCap / 256, 256, 0, L.stream>>>(hp);
  hot_select_kernel<<<kHotCountCap / 256, 256, 0, L.stream>>>(hp);
  cudaError_t e = cudaGetLastError();
  if (L.after) L.after(L.ctx, kKHot);
  return e;
}

template <int NQB>
static cudaError_t count_hot_t(const PartPlan &p, const HotParams &hp, const Launcher &L) {
  const size_t sm = sizeof(HotSmem<NQB>);
  cudaFuncSetAttribute(part_count_hot_kernel<NQB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int grid = (hp.n_chunks + kHotCtaWarps - 1) / kHotCtaWarps;
  LTL4C_LAUNCH(kKPartCount, part_count_hot_kernel<NQB><<<grid, 32 * kHotCtaWarps, sm, L.stream>>>(p, hp));
}

cudaError_t launch_part_count_hot(const PartPlan &p, const HotParams &hp, int nq, const Launcher &L) {
  if (nq <= 4) return count_hot_t<4>(p, hp, L);
  return count_hot_t<8>(p, hp, L);
}

template <int NQB>
static cudaError_t finish_t(const HotParams &hp, const Launcher &L) {
  LTL4C_LAUNCH(kKHot, hot_finish_kernel<NQB><<<kHotKeys / 8, 256, 0, L.stream>>>(hp, hp.n_chunks));
}

cudaError_t launch_hot_finish(const HotParams &hp, int nq, const Launcher &L) {
  if (nq <= 4) return finish_t<4>(hp, L);
  return finish_t<8>(hp, L);
}

int hot_ctas_per_sm(int nq) {
  int n = 1;
  if (nq <= 4) {
    cudaFuncSetAttribute(part_count_hot_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HotSmem<4>));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, part_count_hot_kernel<4>, 256, sizeof(HotSmem<4>));
  } else {
    cudaFuncSetAttribute(part_count_hot_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HotSmem<8>));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, part_count_hot_kernel<8>, 256, sizeof(HotSmem<8>));
  }
  return n > 0 ? n : 1;
}

}  // namespace ltl4c
