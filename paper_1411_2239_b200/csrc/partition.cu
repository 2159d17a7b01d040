// partition.cu -- a1 (epsilon) + a2 (SortTrace) of arXiv:1411.2239 Alg. 1
// on sm_100a: a STABLE LSD partition of the bound events of a
// batch by bucket = top `bits` bits of hash(k0).
//
//   part_count     per 4096-event tile: digit counts (pass 0 reads every key:
//                  epsilon filter, Eq. D P:530 -- an event binds a value vector
//                  only if every guard key is present; later passes read k0).
//   part_scan      exclusive scan of each digit's row of tile counts.
//   part_scatter   the tile is staged in shared memory, ranked stably by digit
//                  (warp __match_any_sync rounds in trace order + per-warp digit
//                  counters) and written back digit run by digit run (coalesced).
//   bucket_bounds  bucket offsets mu from the final order.
//
// Stability keeps every slice u^D in trace order (reading A15); a bucket holds
// whole level-0 subtrees because every tree node's key starts with k0.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "util.cuh"

namespace ltl4c {
namespace {

constexpr int kPWarps = kPartThreads / 32;
constexpr int kRounds = kTileEv / kPartThreads;  // rounds of 32 events per warp

// Digit counts of one tile (counts[d][tile]).  Pass 0 reads the batch and
// applies the epsilon filter; later passes read k0 of the previous pass.
// (persistent: CTA b takes tiles b, b + grid, ... below the events of this pass)
template <int K, bool kFirst, bool kDeep>
__global__ void __launch_bounds__(kPartThreads) part_count_kernel(PartPlan pl, int pass) {
  __shared__ uint32_t h[kMaxDigits];
  __shared__ uint32_t nv;
  if (pass_skipped(pl, pass)) return;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < kMaxDigits; i += kPartThreads) h[i] = 0;
  if (tid == 0) nv = 0;
  __syncthreads();
  const bool dense = kFirst && first_dense(pl);
  const uint32_t *const *in_key = kFirst ? pl.in_key : (const uint32_t *const *)pl.buf_key[(pass - 1) & 1];
  const unsigned long long n = kFirst ? first_n(pl) : *pl.nvalid;
  for (uint32_t tile = blockIdx.x; (unsigned long long)tile * kTileEv < n; tile += gridDim.x) {
    const unsigned long long base = (unsigned long long)tile * kTileEv;
    const uint32_t dmask = (1u << pl.width[pass]) - 1u;
    const int lo = pl.lo[pass];
    uint32_t k0[kRounds];  // the hash key (column 0, or K-1 if kDeep; pass 0 also checks every guard key)
    bool ok[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {  // all loads first (memory-level parallelism)
      const unsigned long long j = base + (unsigned long long)r * kPartThreads + tid;
      ok[r] = j < n;
      if (kFirst && kDeep) {
        uint32_t kv[K];
#pragma unroll
        for (int i = 0; i < K; ++i) kv[i] = ok[r] ? in_key[i][j] : 0u;
#pragma unroll
        for (int i = 1; i < K; ++i) ok[r] &= kv[i] != kAbsent;
        k0[r] = kv[0] == kAbsent ? kAbsent : kv[K - 1];  // (kv[0] absent: unbound, never counted)
      } else if (kFirst) {
        k0[r] = ok[r] ? (dense ? pl.dense_key[j] : in_key[0][j]) : 0u;
#pragma unroll
        for (int i = 1; i < K; ++i) ok[r] &= !(ok[r] && in_key[i][j] == kAbsent);
      } else {
        k0[r] = ok[r] ? pl.hcol[(pass - 1) & 1][j] : 0u;
      }
    }
    uint32_t myvalid = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const bool v = ok[r] && (!kFirst || k0[r] != kAbsent);
      if (v) atomicAdd(&h[(salted_bucket(k0[r], pl.bits, pl.salt) >> lo) & dmask], 1u);
      myvalid += v;
    }
    if (kFirst) {
      for (int d = 16; d; d >>= 1) myvalid += __shfl_down_sync(0xffffffffu, myvalid, d);
      if (lane == 0 && myvalid) atomicAdd(&nv, myvalid);
    }
    __syncthreads();
    for (int d = tid; d < (1 << pl.width[pass]); d += kPartThreads) {
      pl.counts[(size_t)d * pl.n_tiles + tile] = h[d];
      h[d] = 0;
    }
    __syncthreads();
  }
  if (kFirst && tid == 0 && nv) {
    atomicAdd(pl.nvalid, (unsigned long long)nv);
    atomicAdd(&pl.acc->events_bound, (unsigned long long)nv);
  }
}

// A tiny batch (<= kTinyBatch events, one CTA): the epsilon filter (Eq. D: an
// event binds a value vector only if every guard key is present), the bound events
// compacted in trace order into the final partition buffers as ONE bucket (bucket 0;
// every later bucket starts at the end), the bound count.  The bucket kernels then
// see a single unit holding the whole batch in trace order.
template <int K>
__global__ void __launch_bounds__(kTinyBatch) tiny_stage_kernel(PartPlan pl, uint32_t *off, uint32_t nb) {
  __shared__ uint32_t wt[kTinyBatch / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t n = (uint32_t)pl.n;
  uint32_t kv[K];
  uint8_t let = 0;
  bool v = (uint32_t)tid < n;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    kv[i] = v ? pl.in_key[i][tid] : kAbsent;
    v &= kv[i] != kAbsent;
  }
  if (v) let = (uint8_t)(pl.in_let[tid] & pl.let_mask);
  const uint32_t bal = __ballot_sync(0xffffffffu, v);
  if (lane == 0) wt[wid] = __popc(bal);
  __syncthreads();
  uint32_t before = 0, total = 0;
  for (int w = 0; w < kTinyBatch / 32; ++w) {
    before += w < wid ? wt[w] : 0u;
    total += wt[w];
  }
  const int fin = (pl.passes - 1) & 1;
  if (v) {
    const uint32_t pos = before + __popc(bal & lanemask_lt());
#pragma unroll
    for (int i = 0; i < K; ++i) pl.buf_key[fin][i][pos] = kv[i];
    pl.buf_let[fin][pos] = let;
  }
  for (uint32_t c = tid; c <= nb; c += blockDim.x) off[c] = c == 0 ? 0u : total;
  if (tid == 0) {
    *pl.nvalid = total;
    if (total) atomicAdd(&pl.acc->events_bound, (unsigned long long)total);
  }
}

// exclusive scan of counts[d][0..n_tiles) in place (one CTA per digit), totals[d]:
// thread t owns a contiguous run of the row (all its loads issued at once), one
// block scan of the run sums
#ifndef LTL4C_SCAN_THREADS
#define LTL4C_SCAN_THREADS 256
#endif
constexpr int kScanThreads = LTL4C_SCAN_THREADS;
constexpr int kScanPer = 16;  // rows up to 16 x kScanThreads tiles in one sweep (256: 4096 tiles, 16.7M events)
__global__ void __launch_bounds__(kScanThreads) part_scan_kernel(PartPlan pl, int pass) {
  __shared__ uint32_t wt[kScanThreads / 32];
  if (pass_skipped(pl, pass)) return;
  uint32_t *row = pl.counts + (size_t)blockIdx.x * pl.n_tiles;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // tiles holding events of this pass (later passes read only the bound events)
  const uint32_t nt = (uint32_t)(((pass == 0 ? first_n(pl) : *pl.nvalid) + kTileEv - 1) / kTileEv);
  uint32_t carry = 0;
  for (uint32_t off = 0; off < nt; off += kScanThreads * kScanPer) {
    const uint32_t per = min((uint32_t)kScanPer, (nt - off + kScanThreads - 1) / kScanThreads);
    const uint32_t lo = off + tid * per;
    uint32_t v[kScanPer];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
      v[i] = ((uint32_t)i < per && lo + i < nt) ? row[lo + i] : 0u;
      sum += v[i];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    if (lane == 31) wt[wid] = inc;
    __syncthreads();
    uint32_t t = lane < kScanThreads / 32 ? wt[lane] : 0u;
#pragma unroll
    for (int d = 1; d < kScanThreads / 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, t, kScanThreads / 32 - 1);
    uint32_t run = carry + inc - sum + (wid ? __shfl_sync(0xffffffffu, t, wid - 1) : 0u);
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
      if ((uint32_t)i < per && lo + i < nt) row[lo + i] = run;
      run += v[i];
    }
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) pl.digit_hist[pass * kMaxDigits + blockIdx.x] = carry;
}

static_assert(kPartThreads >= kMaxDigits / 2 && kPartThreads <= 1024, "two digits per thread of the first half");

template <int K>
struct SweepSmem {
  uint32_t kout[K][kTileEv];        // the tile in digit order
  uint32_t gout[kTileEv];           // global position of each of them
  uint8_t lout[kTileEv];
  uint16_t wcnt[kPWarps][kMaxDigits];  // per-warp digit counts -> tile-local run starts
  uint32_t gdelta[kMaxDigits];      // global run start - tile-local run start
  uint32_t wt[kPWarps];
};

// exclusive scan over the block, one value per thread (kPartThreads = 16 warps):
// warp scans by shuffles, then the 16 warp totals are scanned by shuffles in
// every warp (one broadcast load each)
__device__ __forceinline__ uint32_t block_scan_512(uint32_t x, uint32_t *wt) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) wt[wid] = inc;
  __syncthreads();
  uint32_t t = wt[lane & (kPWarps - 1)];
#pragma unroll
  for (int d = 1; d < kPWarps; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, t, d);
    if ((lane & (kPWarps - 1)) >= d) t += y;
  }
  const uint32_t add = wid ? __shfl_sync(0xffffffffu, t, wid - 1) : 0u;
  __syncthreads();
  return inc - x + add;
}

// One tile of 4096 events: warp w loads its contiguous 256 events into
// registers (8 coalesced rounds of 32), ranks them stably by digit in trace
// order (match masks of all rounds first, then the per-warp digit counters),
// scatters them into shared memory in digit order together with their global
// position, and the tile is written out digit run by digit run (coalesced).
//
// kFirst: pass 0 (events may lack guard keys: the epsilon filter); kFull: a
// tile without a ragged end (no range checks).  A later pass's input holds only
// bound events, so a full tile of a later pass needs no validity test at all.
template <int K, bool kDeep, bool kFirst, bool kFull>
__device__ __forceinline__ void scatter_tile(const PartPlan &pl, int pass, SweepSmem<K> &s, const uint32_t tile) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr bool first = kFirst;
  const bool dense = first && first_dense(pl);  // K = 1 hot path: the dense cold stream
  const uint32_t *const *in_key = first ? pl.in_key : (const uint32_t *const *)pl.buf_key[(pass - 1) & 1];
  const uint8_t *in_let = first ? (dense ? pl.dense_let : pl.in_let) : pl.buf_let[(pass - 1) & 1];
  uint32_t *const *out_key = pl.buf_key[pass & 1];
  uint8_t *out_let = pl.buf_let[pass & 1];
  const unsigned long long n = first ? first_n(pl) : *pl.nvalid;
  if ((unsigned long long)tile * kTileEv >= n) return;  // (uniform per CTA) no events in this tile
  const int width = pl.width[pass];
  const uint32_t dmask = (1u << width) - 1u;
  const int lo = pl.lo[pass];
  const unsigned long long wbase = (unsigned long long)tile * kTileEv + (unsigned long long)wid * (kTileEv / kPWarps);
  // loads first (memory-level parallelism)
  uint32_t rk[kRounds][K];
  uint32_t rl[(kRounds + 3) / 4] = {};  // letters, four per register
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const unsigned long long j = wbase + r * 32 + lane;
    const bool in = kFull || j < n;
#pragma unroll
    for (int k = 0; k < K; ++k) rk[r][k] = in ? __ldcs(k == 0 && dense ? &pl.dense_key[j] : &in_key[k][j]) : kAbsent;
    rl[r >> 2] |= (in ? (uint32_t)(__ldcs(&in_let[j]) & (kFirst ? pl.let_mask : 0xFFu)) : 0u) << (8 * (r & 3));
  }
  // digits 2t, 2t+1 belong to thread t < kMaxDigits / 2: global run start =
  // pass base (scan of the digit totals) + the tile's offset within the digit
  const bool dth = tid < kMaxDigits / 2;
  const int d0 = 2 * tid, d1 = 2 * tid + 1;
  uint32_t tot0 = 0, tot1 = 0, til0 = 0, til1 = 0;
  if (dth) {
    tot0 = pl.digit_hist[pass * kMaxDigits + d0];
    tot1 = pl.digit_hist[pass * kMaxDigits + d1];
    if (d0 <= (int)dmask) til0 = pl.counts[(size_t)d0 * pl.n_tiles + tile];
    if (d1 <= (int)dmask) til1 = pl.counts[(size_t)d1 * pl.n_tiles + tile];
  }
  static_assert(sizeof(s.wcnt) % (16 * kPartThreads) == 0, "wcnt zeroing by 16-byte stores");
#pragma unroll
  for (int i = tid; i < (int)(sizeof(s.wcnt) / 16); i += kPartThreads) reinterpret_cast<uint4 *>(&s.wcnt[0][0])[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // stable rank within the warp's range
  uint32_t dg[kRounds], pm[kRounds];
  bool vd[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    bool valid = true;
    if (kFirst || !kFull) {
#pragma unroll
      for (int k = 0; k < (kFirst ? K : 1); ++k) valid &= rk[r][k] != kAbsent;
    }
    vd[r] = valid;
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r)
    dg[r] = vd[r] ? (salted_bucket(rk[r][kDeep ? K - 1 : 0], pl.bits, pl.salt) >> lo) & dmask : 0u;
  if (pl.rank_ballot) {
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      uint32_t m = __ballot_sync(0xffffffffu, vd[r]);
#pragma unroll
      for (int b = 0; b < kMaxDigitBits; ++b) {
        if (b < width) {
          const bool bit = (dg[r] >> b) & 1u;
          const uint32_t bal = __ballot_sync(0xffffffffu, bit);
          m &= bit ? bal : ~bal;
        }
      }
      pm[r] = vd[r] ? m : 0u;
    }
  } else {
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const uint32_t vm = __ballot_sync(0xffffffffu, vd[r]);
      pm[r] = vd[r] ? __match_any_sync(vm, dg[r]) : 0u;
    }
  }
  // dr[r] = digit | rank << 16 (the rank within the tile is < 4096)
  uint32_t dr[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    uint32_t old = 0;
    if (vd[r]) old = s.wcnt[wid][dg[r]];
    dr[r] = dg[r] | (old + __popc(pm[r] & lanemask_lt())) << 16;
    __syncwarp();
    if (vd[r] && (pm[r] & lanemask_lt()) == 0) s.wcnt[wid][dg[r]] = (uint16_t)(old + __popc(pm[r]));
    __syncwarp();
  }
  __syncthreads();
  // digits 2t, 2t+1: exclusive over warps (two u16 halves per word, < 4096 each),
  // tile totals, tile-local run starts
  uint32_t *wc32 = reinterpret_cast<uint32_t *>(&s.wcnt[0][0]);
  // (the per-warp prefix is recomputed in the write-back loop below instead of kept
  // in 16 registers: the kernel no longer spills at 64 registers)
  uint32_t run = 0;
  if (dth) {
#pragma unroll
    for (int w = 0; w < kPWarps; ++w) run += wc32[w * (kMaxDigits / 2) + tid];
  }
  const uint32_t c0 = run & 0xFFFFu, c1 = run >> 16;
  const uint32_t loc0 = block_scan_512(c0 + c1, s.wt), loc1 = loc0 + c0;
  const uint32_t pb0 = block_scan_512(tot0 + tot1, s.wt), pb1 = pb0 + tot0;
  if (dth) {
    uint32_t pre = loc0 | loc1 << 16;
#pragma unroll
    for (int w = 0; w < kPWarps; ++w) {
      const uint32_t v = wc32[w * (kMaxDigits / 2) + tid];
      wc32[w * (kMaxDigits / 2) + tid] = pre;
      pre += v;
    }
    s.gdelta[d0] = pb0 + til0 - loc0;
    s.gdelta[d1] = pb1 + til1 - loc1;
  }
  __syncthreads();
  // local scatter into digit order (from registers)
  uint32_t ntile = 0;
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    ntile += __popc(__ballot_sync(0xffffffffu, vd[r]));
    if (!vd[r]) continue;
    const uint32_t d = dr[r] & 0xFFFFu;
    const uint32_t lp = s.wcnt[wid][d] + (dr[r] >> 16);
#pragma unroll
    for (int k = 0; k < K; ++k) s.kout[k][lp] = rk[r][k];
    s.lout[lp] = (uint8_t)(rl[r >> 2] >> (8 * (r & 3)));
    s.gout[lp] = lp + s.gdelta[d];
  }
  if (lane == 0) s.wt[wid] = ntile;
  __syncthreads();
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < kPWarps; ++w) total += s.wt[w];
  // coalesced write-out, digit run by digit run
  for (uint32_t i = tid; i < total; i += kPartThreads) {
    const uint32_t g = s.gout[i];
#pragma unroll
    for (int k = 0; k < K; ++k) out_key[k][g] = s.kout[k][i];
    out_let[g] = s.lout[i];
  }
}

template <int K, bool kDeep, bool kFirst>
__global__ void __launch_bounds__(kPartThreads, 1024 / kPartThreads) part_scatter_kernel(PartPlan pl, int pass) {
  extern __shared__ __align__(16) uint8_t raw[];
  SweepSmem<K> &s = *reinterpret_cast<SweepSmem<K> *>(raw);
  if (pass_skipped(pl, pass)) return;
  const unsigned long long n = kFirst ? first_n(pl) : *pl.nvalid;
  // one CTA per tile (measured faster than a persistent tile loop on full batches:
  // C2 0.476 vs 0.533 ms); the first pass of a K = 1 hot batch, whose dense input is
  // known only on the device, launches a quarter of the tiles and strides (fewer
  // CTAs that find no tile)
  for (uint32_t tile = blockIdx.x; (unsigned long long)tile * kTileEv < n; tile += gridDim.x) {
    if ((unsigned long long)(tile + 1) * kTileEv <= n) scatter_tile<K, kDeep, kFirst, true>(pl, pass, s, tile);
    else scatter_tile<K, kDeep, kFirst, false>(pl, pass, s, tile);
    if (gridDim.x >= pl.n_tiles) break;
    __syncthreads();
  }
}

// off[c] = first position of bucket c in the final order, off[NB] = n.  Each
// thread covers 16 consecutive positions (four 16-byte loads issued together).
constexpr int kBoundsPer = 16;
__global__ void bucket_bounds_kernel(const uint32_t *k0, const unsigned long long *nvalid, uint32_t salt, int shift,
                                     uint32_t mask, uint32_t *off, uint32_t nb, const uint32_t *gate, int want) {
  // (n < 2^32 - 2^20: 32-bit positions; bucket ids are < 2^27, so b + 1 never wraps)
  if (gate && ((*gate != 0) != (want != 0))) return;  // (the other mode of a K = 1 hot batch)
  const uint32_t n = (uint32_t)*nvalid;
  auto bucket = [&](uint32_t k) { return (fmix32(k ^ salt) >> shift) & mask; };
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= n / kBoundsPer; t += gridDim.x * blockDim.x) {
    const uint32_t i0 = kBoundsPer * t;
    uint32_t prev = 0;  // bucket of event i0 - 1, plus one (0 before the first event)
    if (i0 > 0) prev = bucket(k0[i0 - 1]) + 1;
    if (i0 + kBoundsPer <= n) {
      uint32_t kv[kBoundsPer];
#pragma unroll
      for (int q = 0; q < kBoundsPer / 4; ++q) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(k0 + i0) + q);
        kv[4 * q] = v.x; kv[4 * q + 1] = v.y; kv[4 * q + 2] = v.z; kv[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < kBoundsPer; ++j) {
        const uint32_t b = bucket(kv[j]);
        for (uint32_t c = prev; c <= b; ++c) off[c] = i0 + j;  // buckets (previous, b] start here
        prev = max(prev, b + 1);
      }
    } else {  // the ragged end (t = n / 16) also writes the offsets after the last bucket
      for (uint32_t j = 0; i0 + j <= n; ++j) {
        const uint32_t b = i0 + j < n ? bucket(k0[i0 + j]) : nb;
        for (uint32_t c = prev; c <= b; ++c) off[c] = i0 + j;
        prev = max(prev, b + 1);
      }
    }
  }
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

static unsigned part_grid(const PartPlan &p, int per_sm) {
  const unsigned g = (unsigned)(p.n_sms > 0 ? p.n_sms * per_sm : 148 * per_sm);
  return p.n_tiles < g ? (p.n_tiles ? p.n_tiles : 1) : g;
}

template <int K, bool kDeep>
static cudaError_t count_first(const PartPlan &p, int pass, const Launcher &L) {
  LTL4C_LAUNCH(kKPartCount, part_count_kernel<K, true, kDeep><<<part_grid(p, 4), kPartThreads, 0, L.stream>>>(p, pass));
}

cudaError_t launch_part_count(const PartPlan &p, int pass, const Launcher &L) {
  if (pass == 0) {
    const bool deep = p.hk != 0;
    switch (p.K) {
      case 1: return count_first<1, false>(p, pass, L);
      case 2: return deep ? count_first<2, true>(p, pass, L) : count_first<2, false>(p, pass, L);
      default: return deep ? count_first<3, true>(p, pass, L) : count_first<3, false>(p, pass, L);
    }
  }
  LTL4C_LAUNCH(kKPartCount, part_count_kernel<1, false, false><<<part_grid(p, 4), kPartThreads, 0, L.stream>>>(p, pass));
}

cudaError_t launch_tiny_stage(const PartPlan &p, uint32_t *off, uint32_t n_buckets, const Launcher &L) {
  switch (p.K) {
    case 1: LTL4C_LAUNCH(kKPartCount, tiny_stage_kernel<1><<<1, kTinyBatch, 0, L.stream>>>(p, off, n_buckets));
    case 2: LTL4C_LAUNCH(kKPartCount, tiny_stage_kernel<2><<<1, kTinyBatch, 0, L.stream>>>(p, off, n_buckets));
    default: LTL4C_LAUNCH(kKPartCount, tiny_stage_kernel<3><<<1, kTinyBatch, 0, L.stream>>>(p, off, n_buckets));
  }
}

cudaError_t launch_part_scan(const PartPlan &p, int pass, const Launcher &L) {
  LTL4C_LAUNCH(kKPartScan, part_scan_kernel<<<1u << p.width[pass], kScanThreads, 0, L.stream>>>(p, pass));
}

template <int K, bool kDeep>
static cudaError_t scatter(const PartPlan &p, int pass, const Launcher &L) {
  const size_t sm = sizeof(SweepSmem<K>);
  if (pass == 0) {
    cudaFuncSetAttribute(part_scatter_kernel<K, kDeep, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const unsigned grid = p.dense_flag ? (p.n_tiles + 3) / 4 : p.n_tiles;
    LTL4C_LAUNCH(kKPartScatter, part_scatter_kernel<K, kDeep, true><<<grid, kPartThreads, sm, L.stream>>>(p, pass));
  }
  cudaFuncSetAttribute(part_scatter_kernel<K, kDeep, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const unsigned grid = p.skip_flag ? (p.n_tiles + 3) / 4 : p.n_tiles;  // (usually skipped: see above)
  LTL4C_LAUNCH(kKPartScatter, part_scatter_kernel<K, kDeep, false><<<grid, kPartThreads, sm, L.stream>>>(p, pass));
}

cudaError_t launch_part_scatter(const PartPlan &p, int pass, const Launcher &L) {
  const bool deep = p.hk != 0;
  switch (p.K) {
    case 1: return scatter<1, false>(p, pass, L);
    case 2: return deep ? scatter<2, true>(p, pass, L) : scatter<2, false>(p, pass, L);
    default: return deep ? scatter<3, true>(p, pass, L) : scatter<3, false>(p, pass, L);
  }
}

// gate: the launch runs iff (*gate != 0) == want (a K = 1 hot batch: the one-pass
// mode's coarse offsets are the first pass's digit totals, coarse_order_kernel)
cudaError_t launch_bucket_bounds(const PartPlan &p, uint32_t *off, uint32_t n_buckets, const Launcher &L,
                                 const uint32_t *gate, int want) {
  const uint32_t *k0 = p.hcol[(p.passes - 1) & 1];
  int shift = 0;
  uint32_t mask = 0;
  if (p.bits > 0) {
    shift = 32 - p.bits;
    mask = p.bits >= 32 ? 0xFFFFFFFFu : (1u << p.bits) - 1u;
  }
  const unsigned long long want_t = (p.n / kBoundsPer + 1 + 255) / 256;
  const unsigned grid = (unsigned)(want_t > 148 * 16 ? 148 * 16 : want_t);
  LTL4C_LAUNCH(kKBucketBounds, bucket_bounds_kernel<<<grid ? grid : 1, 256, 0, L.stream>>>(
                                   k0, p.nvalid, p.salt, shift, mask, off, n_buckets, gate, want));
}

}  // namespace ltl4c
