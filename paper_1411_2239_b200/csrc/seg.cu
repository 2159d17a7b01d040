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
#ifndef LTL4C_SEG_ROUNDS
#define LTL4C_SEG_ROUNDS 8
#endif
constexpr int kSegRounds = LTL4C_SEG_ROUNDS;  // rounds of 32 events whose loads are issued together
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
  if (p.gate && ((*p.gate != 0) != (p.gate_want != 0))) return;  // (the other mode of a K = 1 hot batch)
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
  const uint32_t n_items = min(p.n_units, (uint32_t)(*p.nvalid / p.unit_target) + 2u);
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
                const uint32_t c = atomicAdd(&w.ncl, 1u);  // (lanes of one round may pass the check together)
                if (c < (uint32_t)(kSegSlots / 2)) w.list[c] = (uint16_t)h;
                else ovf = true;
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
        // the round regrouped stably by key (a group = the lanes of one key, in lane
        // order = trace order): __match_any_sync, then group offsets by a scan of
        // the group sizes over the group leaders (lowest lanes); lane -> position
        // offset + rank
        const uint32_t vm = __ballot_sync(0xffffffffu, slot >= 0);
        const int nv = __popc(vm);  // valid lanes are a prefix of the warp
        uint32_t peers = 0;
        if (slot >= 0) peers = __match_any_sync(vm, (uint32_t)slot);
        const uint32_t rank = __popc(peers & lanemask_lt());
        const bool lead = slot >= 0 && rank == 0;
        const uint32_t gsz = lead ? (uint32_t)__popc(peers) : 0u;
        uint32_t incl = gsz;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += y;
        }
        const int leader = slot >= 0 ? __ffs(peers) - 1 : lane;
        const uint32_t off = __shfl_sync(0xffffffffu, incl - gsz, leader);
        const uint32_t heads = __reduce_or_sync(0xffffffffu, lead ? 1u << off : 0u);
        if (slot >= 0) stage[off + rank] = smap[ll[r]];
        __syncwarp();
        // segmented inclusive scan of the regrouped letter maps (a segment = a group;
        // a lane whose window holds its segment's head is done, so the scan stops
        // after log2 of the largest group)
        M m = lane < nv ? stage[lane] : SM::ident();
        bool f = ((heads >> lane) & 1u) || lane >= nv;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          if (__all_sync(0xffffffffu, f || lane < d)) break;
          const M y = shfl_up(m, d);
          const bool yf = __shfl_up_sync(0xffffffffu, f, d);
          if (lane >= d) {
            if (!f) m = SM::apply(m, y);
            f = f || yf;
          }
        }
        __syncwarp();
        stage[lane] = m;
        __syncwarp();
        // each group's leader applies the group's composition (at its last position)
        if (lead) w.state[slot] = (uint8_t)SM::image(stage[off + gsz - 1], w.state[slot]);
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



// ---------------------------------------------------------------- bucket_coarse
// One-pass mode of a K = 1 hot batch (monitors of <= 4 states, <= 16 letters):
// the cold stream is partitioned ONCE (512 coarse buckets, whole slices each, in
// trace order, keys interleaved as in the trace).  A CTA takes a coarse bucket
// and cuts it into 16 contiguous warp ranges; keys are found or inserted in the
// CTA's table (64-bit CAS on {epoch, key}), and every warp composes, in trace
// order, its own transition map of each key it meets (2-bit packed maps, a
// letter applied through a [256][A] table; lanes sharing a key in a round are
// grouped by __match_any_sync and their letters applied by the lowest lane in
// lane order).  A leaf's state is q0 taken through the warps' maps in warp
// order.  A bucket with more than kCoarseClaims keys goes to the heavy path.
#ifndef LTL4C_COARSE_WARPS
#define LTL4C_COARSE_WARPS 16
#endif
constexpr int kCoarseWarps = LTL4C_COARSE_WARPS;
constexpr int kCoarseSlots = 4096;
constexpr int kCoarseClaims = 3072;
struct CoarseSmem {
  unsigned long long slot[kCoarseSlots];   // epoch << 32 | key
  uint8_t wmap[kCoarseWarps][kCoarseSlots];   // per-warp maps (identity outside the bucket's keys)
  uint8_t tab[256 * 16];                   // [map][letter] -> map
  uint16_t list[kCoarseClaims];            // claimed slots
  uint8_t stage[kCoarseWarps][32];
  uint32_t sacc[kMaxFormulas * 6];
  uint8_t slab[kMaxFormulas * kMaxStates];
  uint32_t ncl, ovf, item;
};

template <int NF>
__global__ void __launch_bounds__(32 * kCoarseWarps, 32 / kCoarseWarps) bucket_coarse_kernel(BucketParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  if (p.gate && ((*p.gate != 0) != (p.gate_want != 0))) return;  // (the other mode)
  CoarseSmem &s = *reinterpret_cast<CoarseSmem *>(smem_raw);
  const DevProg *prog = p.prog;
  const int nq = prog->nq, A = 1 << prog->na;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (blockIdx.x == 0 && tid == 0) p.acc->onepass = 1;
  for (int i = tid; i < 256 * A; i += blockDim.x) {
    const uint32_t m = (uint32_t)i / A, a = (uint32_t)i % A;
    uint32_t o = 0;
    for (int q = 0; q < 4; ++q) {
      const uint32_t img = (m >> (2 * q)) & 3u;
      o |= (img < (uint32_t)nq ? (uint32_t)prog->delta[img][a] & 3u : img) << (2 * q);
    }
    s.tab[i] = (uint8_t)o;
  }
  for (int i = tid; i < kCoarseSlots; i += blockDim.x) s.slot[i] = 0;
  for (int i = tid; i < kCoarseWarps * kCoarseSlots / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(&s.wmap[0][0])[i] = 0xE4E4E4E4u;
  for (int i = tid; i < kMaxFormulas * 6; i += blockDim.x) s.sacc[i] = 0;
  for (int i = tid; i < kMaxFormulas * kMaxStates; i += blockDim.x) s.slab[i] = prog->lab[i / kMaxStates][i % kMaxStates];
  const uint32_t q0 = prog->q0;
  unsigned long long lc[NF];  // per-thread leaf verdict counts, 16-bit fields for v = 0, 2, 3, 5
#pragma unroll
  for (int f = 0; f < NF; ++f) lc[f] = 0;
  uint32_t ep = 0;
  uint8_t *wm = s.wmap[wid];
  uint8_t *stage = s.stage[wid];
  while (true) {
    __syncthreads();  // every thread is done with the previous bucket's shared state
    if (tid == 0) {
      s.item = atomicAdd(p.bucket_counter, 1u);
      s.ncl = 0;
      s.ovf = 0;
    }
    __syncthreads();
    if (s.item >= p.n_buckets) break;
    const uint32_t c = p.list ? p.list[s.item] : s.item;  // (largest buckets first)
    const uint32_t s0 = p.bucket_off[c], s1 = p.bucket_off[c + 1];
    if (s1 == s0) continue;
    ++ep;
    const unsigned long long epk = (unsigned long long)ep << 32;
    const uint32_t per = ((s1 - s0 + kCoarseWarps - 1) / kCoarseWarps + 31) & ~31u;
    const uint32_t w0 = min(s1, s0 + wid * per), w1 = min(s1, w0 + per);
    for (uint32_t base = w0; base < w1; base += 32 * kSegRounds) {
      if (__any_sync(0xffffffffu, *(volatile uint32_t *)&s.ovf != 0)) break;
      uint32_t kk[kSegRounds];
      uint8_t ll[kSegRounds];
#pragma unroll
      for (int r = 0; r < kSegRounds; ++r) {
        const uint32_t e = base + 32 * r + lane;
        kk[r] = e < w1 ? __ldcs(&p.key[0][e]) : kAbsent;
        ll[r] = e < w1 ? __ldcs(&p.let[e]) : (uint8_t)0;
      }
#pragma unroll
      for (int r = 0; r < kSegRounds; ++r) {
        if (base + 32 * r >= w1) break;  // (warp-uniform)
        const uint32_t k = kk[r];
        int slot = -1;
        bool bad = false;
        if (base + 32 * r + lane < w1) {
          uint32_t h = fmix32(k ^ kSegSalt) & (kCoarseSlots - 1);
          const unsigned long long mine = epk | k;
          bad = true;  // (unless found or claimed within one sweep of the table)
          for (int it = 0; it < kCoarseSlots; ++it) {
            unsigned long long v = s.slot[h];
            if ((v >> 32) != ep) {
              const unsigned long long o = atomicCAS(&s.slot[h], v, mine);
              if (o == v) {
                const uint32_t x = atomicAdd(&s.ncl, 1u);
                bad = x >= (uint32_t)kCoarseClaims;
                if (!bad) s.list[x] = (uint16_t)h;
                slot = (int)h;
                break;
              }
              v = o;
            }
            if (v == mine) { slot = (int)h; bad = false; break; }
            h = (h + 1) & (kCoarseSlots - 1);
          }
        }
        // too many keys: the bucket goes to the heavy path.  Every warp reads the flag
        // each round, so no warp keeps claiming slots after the table is over its bound
        // (and a probe gives up after one sweep of the table)
        if (bad) s.ovf = 1;
        if (__any_sync(0xffffffffu, *(volatile uint32_t *)&s.ovf != 0)) break;
        const uint32_t hm = __ballot_sync(0xffffffffu, slot >= 0);
        stage[lane] = ll[r];
        __syncwarp();
        if (slot >= 0) {
          const uint32_t peers = __match_any_sync(hm, (uint32_t)slot);
          if ((peers & lanemask_lt()) == 0) {
            uint32_t m = wm[slot];
            uint32_t pm = peers;
            do {
              const int i = __ffs(pm) - 1;
              pm &= pm - 1;
              m = s.tab[m * A + stage[i]];
            } while (pm);
            wm[slot] = (uint8_t)m;
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    const bool ovf = s.ovf != 0;
    if (ovf) {
      // too many keys for the table: the bucket goes to the heavy path (every map is
      // reset: warps may have met keys that were never listed)
      for (int i = tid; i < kCoarseWarps * kCoarseSlots / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(&s.wmap[0][0])[i] = 0xE4E4E4E4u;
      if (tid == 0) {
        p.oversize_list[atomicAdd(&p.acc->oversize_buckets, 1ull)] = c;
        atomicAdd(&p.acc->oversize_events, (unsigned long long)(s1 - s0));
      }
      continue;
    }
    // every leaf of the bucket: q0 through the warps' maps in warp order; the maps
    // are reset to the identity for the next bucket
    const uint32_t ncl = s.ncl;
    for (uint32_t i = tid; i < ncl; i += blockDim.x) {
      const uint32_t h = s.list[i];
      uint32_t q = q0;
#pragma unroll
      for (int w = 0; w < kCoarseWarps; ++w) {
        q = (s.wmap[w][h] >> (2 * q)) & 3u;
        s.wmap[w][h] = 0xE4;
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) lc[f] += 1ull << (16 * ((s.slab[f * kMaxStates + q] + 1) >> 1));
    }
    // (a thread counts at most kCoarseClaims / 512 = 6 leaves per bucket: the 16-bit
    // fields are flushed every 8192 buckets)
    if ((ep & 8191u) == 0) {
#pragma unroll
      for (int f = 0; f < NF; ++f) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t x = __reduce_add_sync(0xffffffffu, (uint32_t)(lc[f] >> (16 * j)) & 0xFFFFu);
          if (lane == 0 && x) atomicAdd(&s.sacc[f * 6 + (j == 0 ? 0 : j + 1 + (j == 3))], x);
        }
        lc[f] = 0;
      }
    }
  }
#pragma unroll
  for (int f = 0; f < NF; ++f) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t x = __reduce_add_sync(0xffffffffu, (uint32_t)(lc[f] >> (16 * j)) & 0xFFFFu);
      if (lane == 0 && x) atomicAdd(&s.sacc[f * 6 + (j == 0 ? 0 : j + 1 + (j == 3))], x);
    }
  }
  __syncthreads();
  for (int i = tid; i < NF * 6; i += blockDim.x)
    if (s.sacc[i]) atomicAdd(&p.acc->hist[i / 6][1][i % 6], (unsigned long long)s.sacc[i]);
}

// the coarse buckets' offsets and their order by decreasing size (one CTA).  A
// coarse bucket is a digit of the first partition pass, so its size is that
// digit's total (hist, from part_scan) and the offsets are their exclusive scan
// (no pass over the events); then a bitonic sort of (size, id): CTAs take the
// largest first, so the last wave holds the small ones
__global__ void __launch_bounds__(1024) coarse_order_kernel(const uint32_t *hist, uint32_t *off, uint32_t nb,
                                                            uint32_t *order, const uint32_t *gate) {
  __shared__ unsigned long long v[1024];
  __shared__ uint32_t wt[32];
  if (gate && *gate == 0) return;
  const uint32_t t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint32_t c = t < nb ? hist[t] : 0u;
  uint32_t inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) wt[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = wt[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    wt[lane] = w;
  }
  __syncthreads();
  const uint32_t ex = inc - c + (wid ? wt[wid - 1] : 0u);
  if (t < nb) off[t] = ex;
  if (t == nb - 1) off[nb] = ex + c;
  // key: larger size first, then smaller id (ascending sort of ~size << 32 | id)
  v[t] = t < nb ? ((unsigned long long)(~c) << 32 | t) : ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= 1024; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const uint32_t x = t ^ j;
      if (x > t) {
        const bool up = (t & k) == 0;
        const unsigned long long a = v[t], b = v[x];
        if ((a > b) == up) { v[t] = b; v[x] = a; }
      }
      __syncthreads();
    }
  if (t < nb) order[t] = (uint32_t)v[t];
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



template <int NF>
static cudaError_t coarse_launch(const BucketParams &p, uint32_t grid, const Launcher &L) {
  const size_t sm = sizeof(CoarseSmem);
  cudaFuncSetAttribute(bucket_coarse_kernel<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (L.before) L.before(L.ctx, kKBucketWarp);
  bucket_coarse_kernel<NF><<<grid, 32 * kCoarseWarps, sm, L.stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (L.after) L.after(L.ctx, kKBucketWarp);
  return e;
}

cudaError_t launch_bucket_coarse(const BucketParams &p, int nf, uint32_t grid, const Launcher &L) {
  if (p.list) {
    if (L.before) L.before(L.ctx, kKBucketWarp);
    coarse_order_kernel<<<1, 1024, 0, L.stream>>>(p.coarse_hist, const_cast<uint32_t *>(p.bucket_off), p.n_buckets,
                                                  const_cast<uint32_t *>(p.list), p.gate);
    if (L.after) L.after(L.ctx, kKBucketWarp);
  }
  switch (nf) {
    case 1: return coarse_launch<1>(p, grid, L);
    case 2: return coarse_launch<2>(p, grid, L);
    case 3: return coarse_launch<3>(p, grid, L);
    default: return coarse_launch<4>(p, grid, L);
  }
}

int bucket_coarse_ctas_per_sm() {
  int n = 1;
  cudaFuncSetAttribute(bucket_coarse_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CoarseSmem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, bucket_coarse_kernel<4>, 32 * kCoarseWarps, sizeof(CoarseSmem));
  return n > 0 ? n : 1;
}

}  // namespace ltl4c
