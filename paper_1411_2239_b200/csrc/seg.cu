// seg.cu -- the bucket kernel of single-level properties (K = 1, offline):
// a3 SpawnMonitors + a4 Distribute/UpdateMonitor + a5 (leaf level) of arXiv:
// 1411.2239 Alg. 1 on the partitioned trace.
//
// For K = 1 a leaf is one key value and its verdict is lambda(delta*(q0, u^D))
// (Def. 5).  A warp takes a work unit (a run of consecutive buckets,
// which hold whole slices in trace order) and streams it 32 events per round:
//   - every lane finds or inserts its key in the warp's table (one 64-bit CAS
//     on {epoch, key}; a new leaf starts at q0);
//   - the round's letters become transition maps, and a SEGMENTED inclusive scan
//     over the lanes (a segment = a run of consecutive lanes with the same key;
//     5 shuffle steps, maps composed by byte permutation) leaves every run's
//     ordered composition in its last lane;
//   - run ends apply their map to the leaf's state (run ends of one key in a
//     round are grouped by __match_any_sync and applied in lane order).
// A unit's table holds its distinct keys only, so a bucket of any length streams
// through one warp (slices of skewed keys are long, their keys few); buckets
// above kSegMax events go to the heavy path, units with too many distinct keys
// to the CTA kernel.  At the end of a unit every leaf's verdict is counted.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "util.cuh"

namespace ltl4c {
namespace {

constexpr int kSegWarps = 8;
constexpr int kSegSlots = 512;          // table slots per warp (claims <= kSegSlots / 2)
constexpr uint32_t kSegMax = 1u << 14;  // buckets above this many events: heavy path (parallel segments)
constexpr int kSegRounds = 8;           // rounds of 32 events whose loads are issued together
constexpr uint32_t kSegSalt = 0x27d4eb2fu;

__device__ __forceinline__ uint32_t sel_of(uint32_t f) {  // bytes b0..b3 (< 8) -> nibbles
  const uint32_t x = f | (f >> 4);
  return __byte_perm(x, 0u, 0x4420u);
}
// transition maps: byte q = image of state q (NQB <= 8), composed by PRMT; nibble
// q (NQB = 16) composed nibble by nibble.  apply(g, f) = g o f (f first).
template <int NQB> struct SegMap {
  using T = unsigned long long;
  __device__ static T ident() { return 0xFEDCBA9876543210ull; }
  __device__ static T apply(T g, T f) {
    T r = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) r |= ((g >> (4 * ((f >> (4 * q)) & 15u))) & 15u) << (4 * q);
    return r;
  }
  __device__ static uint32_t image(T m, uint32_t q) { return (uint32_t)(m >> (4 * q)) & 15u; }
  __device__ static T of_row(const uint8_t *d, int nq) {
    T m = ident();
    for (int q = 0; q < nq; ++q) m = (m & ~(15ull << (4 * q))) | ((T)d[q] << (4 * q));
    return m;
  }
};
template <> struct SegMap<4> {
  using T = uint32_t;
  __device__ static T ident() { return 0x03020100u; }
  __device__ static T apply(T g, T f) { return __byte_perm(g, 0u, sel_of(f)); }
  __device__ static uint32_t image(T m, uint32_t q) { return (m >> (8 * q)) & 0xFFu; }
  __device__ static T of_row(const uint8_t *d, int nq) {
    T m = ident();
    for (int q = 0; q < nq; ++q) m = (m & ~(0xFFu << (8 * q))) | ((T)d[q] << (8 * q));
    return m;
  }
};
template <> struct SegMap<8> {
  using T = unsigned long long;
  __device__ static T ident() { return 0x0706050403020100ull; }
  __device__ static T apply(T g, T f) {
    const uint32_t glo = (uint32_t)g, ghi = (uint32_t)(g >> 32);
    const uint32_t lo = __byte_perm(glo, ghi, sel_of((uint32_t)f));
    const uint32_t hi = __byte_perm(glo, ghi, sel_of((uint32_t)(f >> 32)));
    return (T)hi << 32 | lo;
  }
  __device__ static uint32_t image(T m, uint32_t q) { return (uint32_t)(m >> (8 * q)) & 0xFFu; }
  __device__ static T of_row(const uint8_t *d, int nq) {
    T m = ident();
    for (int q = 0; q < nq; ++q) m = (m & ~(0xFFull << (8 * q))) | ((T)d[q] << (8 * q));
    return m;
  }
};

template <class T>
__device__ __forceinline__ T shfl_up(T v, int d) {
  if constexpr (sizeof(T) == 8) {
    const uint32_t lo = __shfl_up_sync(0xffffffffu, (uint32_t)v, d);
    const uint32_t hi = __shfl_up_sync(0xffffffffu, (uint32_t)(v >> 32), d);
    return (T)hi << 32 | lo;
  } else {
    return __shfl_up_sync(0xffffffffu, v, d);
  }
}

struct SegTab {
  unsigned long long slot[kSegSlots];   // epoch << 32 | key (other epochs = empty)
  uint8_t state[kSegSlots];
  uint16_t list[kSegSlots / 2];         // claimed slots of the unit
  uint32_t ncl;
};

template <int NQB, int NF>
__global__ void __launch_bounds__(32 * kSegWarps, 4) bucket_seg_kernel(BucketParams p) {
  using SM = SegMap<NQB>;
  using M = typename SM::T;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const DevProg *prog = p.prog;
  const int nq = prog->nq, A = 1 << prog->na;
  M *smap = reinterpret_cast<M *>(smem_raw);                                   // [A] letter maps
  uint32_t *sacc = reinterpret_cast<uint32_t *>(smem_raw + sizeof(M) * kMaxLetters);  // [NF][6]
  uint8_t *slab = reinterpret_cast<uint8_t *>(sacc + kMaxFormulas * 6);        // [NF][kMaxStates]
  M *stage_all = reinterpret_cast<M *>(smem_raw + sizeof(M) * kMaxLetters + 4 * kMaxFormulas * 6 +
                                       kMaxFormulas * kMaxStates);
  SegTab *tabs = reinterpret_cast<SegTab *>(stage_all + 32 * kSegWarps);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  SegTab &w = tabs[wid];
  M *stage = stage_all + 32 * wid;
  for (int a = threadIdx.x; a < A; a += blockDim.x) {
    uint8_t d[kMaxStates];
    for (int q = 0; q < nq; ++q) d[q] = prog->delta[q][a];
    smap[a] = SM::of_row(d, nq);
  }
  for (int i = threadIdx.x; i < kMaxFormulas * 6; i += blockDim.x) sacc[i] = 0;
  for (int i = threadIdx.x; i < kMaxFormulas * kMaxStates; i += blockDim.x)
    slab[i] = prog->lab[i / kMaxStates][i % kMaxStates];
  for (int i = lane; i < kSegSlots; i += 32) w.slot[i] = 0;
  __syncthreads();
  const uint32_t q0 = prog->q0;
  // per-lane leaf verdict counts, 16-bit fields j = 0..3 for v = 0, 2, 3, 5
  unsigned long long lc[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) lc[f] = 0;
  uint32_t since = 0;
  auto flush = [&]() {
#pragma unroll
    for (int f = 0; f < NF; ++f) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t c = __reduce_add_sync(0xffffffffu, (uint32_t)(lc[f] >> (16 * j)) & 0xFFFFu);
        if (lane == 0 && c) atomicAdd(&sacc[f * 6 + (j == 0 ? 0 : j + 1 + (j == 3))], c);
      }
      lc[f] = 0;
    }
  };
  const uint32_t n_items = min(p.n_units, (uint32_t)(*p.nvalid / kUnitTarget) + 2u);
  uint32_t ep = 0;
  auto take = [&]() { uint32_t u = 0; if (lane == 0) u = atomicAdd(p.bucket_counter, 1u); return __shfl_sync(0xffffffffu, u, 0); };
  // stream events [start, end) of buckets [bl, bh) through the table; false: overflow
  auto run = [&](uint32_t start, uint32_t end) -> bool {
    ++ep;
    if (lane == 0) w.ncl = 0;
    __syncwarp();
    for (uint32_t base = start; base < end; base += 32 * kSegRounds) {
      uint32_t kk[kSegRounds];
      uint8_t ll[kSegRounds];
#pragma unroll
      for (int r = 0; r < kSegRounds; ++r) {
        const uint32_t e = base + 32 * r + lane;
        kk[r] = e < end ? __ldcs(&p.key[0][e]) : kAbsent;
        ll[r] = e < end ? __ldcs(&p.let[e]) : (uint8_t)0;
      }
#pragma unroll
      for (int r = 0; r < kSegRounds; ++r) {
        if (base + 32 * r >= end) break;  // (warp-uniform)
        const bool valid = base + 32 * r + lane < end;
        const uint32_t k = kk[r];
        int slot = -1;
        bool ovf = false;
        if (valid) {
          uint32_t h = fmix32(k ^ kSegSalt) & (kSegSlots - 1);
          const unsigned long long mine = (unsigned long long)ep << 32 | k;
          while (true) {
            unsigned long long s = w.slot[h];
            if ((uint32_t)(s >> 32) != ep) {
              if (*(volatile uint32_t *)&w.ncl >= (uint32_t)(kSegSlots / 2)) { ovf = true; break; }
              const unsigned long long o = atomicCAS(&w.slot[h], s, mine);
              if (o == s) {
                w.state[h] = (uint8_t)q0;
                w.list[atomicAdd(&w.ncl, 1u)] = (uint16_t)h;
                slot = (int)h;
                break;
              }
              s = o;
            }
            if (s == mine) { slot = (int)h; break; }
            h = (h + 1) & (kSegSlots - 1);
          }
        }
        if (__any_sync(0xffffffffu, ovf)) return false;
        // segmented inclusive scan of the letter maps over runs of equal slots
        M m = slot >= 0 ? smap[ll[r]] : SM::ident();
        const int prev = __shfl_up_sync(0xffffffffu, slot, 1);
        bool f = lane == 0 || prev != slot;
        // (a lane whose window (lane - 2d, lane] holds its run's head is done; lane 0
        // is a head, so the scan stops after log2 of the longest run)
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          if (__all_sync(0xffffffffu, f)) break;
          const M y = shfl_up(m, d);
          const bool yf = __shfl_up_sync(0xffffffffu, f, d);
          if (lane >= d) {
            if (!f) m = SM::apply(m, y);
            f = f || yf;
          }
        }
        const int next = __shfl_down_sync(0xffffffffu, slot, 1);
        const bool tail = slot >= 0 && (lane == 31 || next != slot);
        const uint32_t tm = __ballot_sync(0xffffffffu, tail);
        if (tail) stage[lane] = m;
        __syncwarp();
        if (tail) {
          const uint32_t peers = __match_any_sync(tm, (uint32_t)slot);
          if ((peers & lanemask_lt()) == 0) {
            uint32_t q = w.state[slot];
            uint32_t pm = peers;
            do {
              const int i = __ffs(pm) - 1;
              pm &= pm - 1;
              q = SM::image(stage[i], q);
            } while (pm);
            w.state[slot] = (uint8_t)q;
          }
        }
        __syncwarp();
      }
    }
    // every leaf of the unit: its verdict (Def. 5) into the per-lane counts
    const uint32_t nl = w.ncl;
    for (uint32_t i = lane; i < nl; i += 32) {
      const uint32_t q = w.state[w.list[i]];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int v = slab[f * kMaxStates + q];
        lc[f] += 1ull << (16 * ((v + 1) >> 1));
      }
    }
    since += (nl + 31) / 32;
    if (since > 60000u) { flush(); since = 0; }
    __syncwarp();
    return true;
  };
  auto spill = [&](uint32_t bl, uint32_t bh) {
    for (uint32_t x = bl + lane; x < bh; x += 32)
      if (p.bucket_off[x + 1] > p.bucket_off[x]) p.spill_list[atomicAdd(p.spill_len, 1ull)] = x;
  };
  for (uint32_t u = take(); u < n_items; u = take()) {
    const uint32_t bl = p.unit_start[u], bh = p.unit_start[u + 1];
    if (bh <= bl) continue;
    const uint32_t s0 = p.bucket_off[bl], s1 = p.bucket_off[bh];
    if (s1 == s0) continue;
    if (s1 - s0 <= kSegMax) {
      if (!run(s0, s1)) spill(bl, bh);
      continue;
    }
    for (uint32_t b = bl; b < bh; ++b) {  // a unit above kSegMax: bucket by bucket
      const uint32_t b0 = p.bucket_off[b], b1 = p.bucket_off[b + 1];
      if (b1 == b0) continue;
      if (b1 - b0 > kSegMax) {
        if (lane == 0) {
          p.oversize_list[atomicAdd(&p.acc->oversize_buckets, 1ull)] = b;
          atomicAdd(&p.acc->oversize_events, (unsigned long long)(b1 - b0));
        }
      } else if (!run(b0, b1)) {
        spill(b, b + 1);
      }
    }
  }
  flush();
  __syncthreads();
  for (int i = threadIdx.x; i < NF * 6; i += blockDim.x)
    if (sacc[i]) atomicAdd(&p.acc->hist[i / 6][1][i % 6], (unsigned long long)sacc[i]);
}

template <int NQB, int NF>
size_t seg_smem() {
  using M = typename SegMap<NQB>::T;
  return sizeof(M) * kMaxLetters + 4 * kMaxFormulas * 6 + kMaxFormulas * kMaxStates + sizeof(M) * 32 * kSegWarps +
         sizeof(SegTab) * kSegWarps;
}

}  // namespace

template <int NQB, int NF>
static cudaError_t seg_launch(const BucketParams &p, uint32_t grid, const Launcher &L) {
  const size_t sm = seg_smem<NQB, NF>();
  cudaFuncSetAttribute(bucket_seg_kernel<NQB, NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (L.before) L.before(L.ctx, kKBucketWarp);
  bucket_seg_kernel<NQB, NF><<<grid, 32 * kSegWarps, sm, L.stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (L.after) L.after(L.ctx, kKBucketWarp);
  return e;
}

template <int NQB>
static cudaError_t seg_nf(const BucketParams &p, int nf, uint32_t grid, const Launcher &L) {
  switch (nf) {
    case 1: return seg_launch<NQB, 1>(p, grid, L);
    case 2: return seg_launch<NQB, 2>(p, grid, L);
    case 3: return seg_launch<NQB, 3>(p, grid, L);
    default: return seg_launch<NQB, 4>(p, grid, L);
  }
}

cudaError_t launch_bucket_seg(const BucketParams &p, int nq, int nf, uint32_t grid, const Launcher &L) {
  if (nq <= 4) return seg_nf<4>(p, nf, grid, L);
  if (nq <= 8) return seg_nf<8>(p, nf, grid, L);
  return seg_nf<16>(p, nf, grid, L);
}

int bucket_seg_ctas_per_sm(int nq) {
  int n = 1;
  const auto q = [&](auto kern, size_t sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 32 * kSegWarps, sm);
  };
  if (nq <= 4) q(bucket_seg_kernel<4, 4>, seg_smem<4, 4>());
  else if (nq <= 8) q(bucket_seg_kernel<8, 4>, seg_smem<8, 4>());
  else q(bucket_seg_kernel<16, 4>, seg_smem<16, 4>());
  return n > 0 ? n : 1;
}

}  // namespace ltl4c
