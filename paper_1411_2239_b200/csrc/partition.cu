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
template <int K, bool kFirst>
__global__ void __launch_bounds__(kPartThreads) part_count_kernel(PartPlan pl, int pass) {
  __shared__ uint32_t h[256];
  __shared__ uint32_t nv;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 256; i += kPartThreads) h[i] = 0;
  if (tid == 0) nv = 0;
  __syncthreads();
  const uint32_t *const *in_key = kFirst ? pl.in_key : (const uint32_t *const *)pl.buf_key[(pass - 1) & 1];
  const unsigned long long n = kFirst ? pl.n : *pl.nvalid;
  const unsigned long long base = (unsigned long long)blockIdx.x * kTileEv;
  const uint32_t dmask = (1u << pl.width[pass]) - 1u;
  const int lo = pl.lo[pass];
  uint32_t k0[kRounds];
  bool ok[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {  // all loads first (memory-level parallelism)
    const unsigned long long j = base + (unsigned long long)r * kPartThreads + tid;
    ok[r] = j < n;
    k0[r] = ok[r] ? in_key[0][j] : 0u;
    if (kFirst) {
#pragma unroll
      for (int i = 1; i < K; ++i) ok[r] &= !(ok[r] && in_key[i][j] == kAbsent);
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
  for (int d = tid; d < (1 << pl.width[pass]); d += kPartThreads) pl.counts[(size_t)d * pl.n_tiles + blockIdx.x] = h[d];
  if (kFirst && tid == 0 && nv) {
    atomicAdd(pl.nvalid, (unsigned long long)nv);
    atomicAdd(&pl.acc->events_bound, (unsigned long long)nv);
  }
}

// exclusive scan of counts[d][0..n_tiles) in place (one CTA per digit), totals[d]
__global__ void __launch_bounds__(1024) part_scan_kernel(PartPlan pl, int pass) {
  __shared__ uint32_t buf[1024];
  __shared__ uint32_t wt[32];
  uint32_t *row = pl.counts + (size_t)blockIdx.x * pl.n_tiles;
  uint32_t carry = 0;
  for (uint32_t off = 0; off < pl.n_tiles; off += 1024) {
    const uint32_t i = off + threadIdx.x;
    buf[threadIdx.x] = i < pl.n_tiles ? row[i] : 0;
    __syncthreads();
    const uint32_t tot = block_exclusive_scan(buf, 1024, wt);
    if (i < pl.n_tiles) row[i] = buf[threadIdx.x] + carry;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) pl.digit_hist[pass * 256 + blockIdx.x] = carry;
}

template <int K>
struct SweepSmem {
  uint32_t kout[K][kTileEv];
  uint8_t lout[kTileEv];
  uint8_t dout[kTileEv];
  uint16_t wcnt[kPWarps][256];
  uint32_t loc[256];     // tile-local exclusive offset of each digit
  uint32_t tcnt[256];    // tile count of each digit
  uint32_t gbase[256];   // global position of the tile's digit run
  uint32_t pbase[256];   // exclusive scan of the pass's digit totals
  uint32_t wt[32];
  uint32_t ntile;        // bound events in this tile
};

// One tile of 4096 events: warp w loads its contiguous 256 events into
// registers (8 coalesced rounds of 32), ranks them stably by digit in trace
// order (match masks of all rounds first, then the per-warp digit counters),
// scatters them into shared memory in digit order and the tile is written out
// digit run by digit run (coalesced).
template <int K>
__global__ void __launch_bounds__(kPartThreads, 2) part_scatter_kernel(PartPlan pl, int pass) {
  extern __shared__ __align__(16) uint8_t raw[];
  SweepSmem<K> &s = *reinterpret_cast<SweepSmem<K> *>(raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool first = pass == 0;
  const uint32_t *const *in_key = first ? pl.in_key : (const uint32_t *const *)pl.buf_key[(pass - 1) & 1];
  const uint8_t *in_let = first ? pl.in_let : pl.buf_let[(pass - 1) & 1];
  uint32_t *const *out_key = pl.buf_key[pass & 1];
  uint8_t *out_let = pl.buf_let[pass & 1];
  const unsigned long long n = first ? pl.n : *pl.nvalid;
  const uint32_t dmask = (1u << pl.width[pass]) - 1u;
  const int lo = pl.lo[pass];
  const uint32_t tile = blockIdx.x;
  const unsigned long long wbase = (unsigned long long)tile * kTileEv + (unsigned long long)wid * (kTileEv / kPWarps);
  // loads first (memory-level parallelism)
  uint32_t rk[kRounds][K];
  uint8_t rl[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const unsigned long long j = wbase + r * 32 + lane;
    const bool in = j < n;
#pragma unroll
    for (int k = 0; k < K; ++k) rk[r][k] = in ? __ldcs(&in_key[k][j]) : kAbsent;
    rl[r] = in ? __ldcs(&in_let[j]) : (uint8_t)0;
  }
  if (tid < 256) {
    s.pbase[tid] = pl.digit_hist[pass * 256 + tid];
    s.loc[tid] = 0;
  }
  for (int i = tid; i < kPWarps * 256; i += kPartThreads) (&s.wcnt[0][0])[i] = 0;
  __syncthreads();
  // pass base offsets: exclusive scan of the digit totals (first 256 threads)
  if (tid < 256) {
    uint32_t x = s.pbase[tid];
    uint32_t inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    if (lane == 31) s.wt[wid] = inc;
    s.pbase[tid] = inc - x;
  }
  __syncthreads();
  if (tid < 256) {
    uint32_t add = 0;
    for (int w = 0; w < wid; ++w) add += s.wt[w];
    s.pbase[tid] += add;
  }
  // stable rank within the warp's range
  uint32_t dg[kRounds], pm[kRounds], rank[kRounds];
  bool vd[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    bool valid = true;
#pragma unroll
    for (int k = 0; k < K; ++k) valid &= rk[r][k] != kAbsent;
    vd[r] = valid;
    dg[r] = valid ? (salted_bucket(rk[r][0], pl.bits, pl.salt) >> lo) & dmask : 0u;
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint32_t vm = __ballot_sync(0xffffffffu, vd[r]);
    pm[r] = vd[r] ? __match_any_sync(vm, dg[r]) : 0u;
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    uint32_t old = 0;
    if (vd[r]) old = s.wcnt[wid][dg[r]];
    rank[r] = old + __popc(pm[r] & lanemask_lt());
    __syncwarp();
    if (vd[r] && (pm[r] & lanemask_lt()) == 0) s.wcnt[wid][dg[r]] = (uint16_t)(old + __popc(pm[r]));
    __syncwarp();
  }
  __syncthreads();
  if (tid < 256) {  // per digit: exclusive over warps, tile total
    uint32_t run = 0;
    for (int w = 0; w < kPWarps; ++w) {
      const uint32_t c = s.wcnt[w][tid];
      s.wcnt[w][tid] = (uint16_t)run;
      run += c;
    }
    s.tcnt[tid] = run;
    s.loc[tid] = run;
  }
  __syncthreads();
  if (tid < 256) {  // tile-local exclusive digit offsets
    uint32_t x = s.loc[tid], inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    if (lane == 31) s.wt[wid] = inc;
    s.loc[tid] = inc - x;
  }
  __syncthreads();
  if (tid < 256) {
    uint32_t add = 0;
    for (int w = 0; w < wid; ++w) add += s.wt[w];
    s.loc[tid] += add;
    if (tid == 255) s.ntile = s.loc[255] + s.tcnt[255];
    s.gbase[tid] = s.pbase[tid] + (tid < (1 << pl.width[pass]) ? pl.counts[(size_t)tid * pl.n_tiles + tile] : 0u);
  }
  __syncthreads();
  // local scatter into digit order (from registers)
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    if (!vd[r]) continue;
    const uint32_t d = dg[r];
    const uint32_t lp = s.loc[d] + s.wcnt[wid][d] + rank[r];
#pragma unroll
    for (int k = 0; k < K; ++k) s.kout[k][lp] = rk[r][k];
    s.lout[lp] = rl[r];
    s.dout[lp] = (uint8_t)d;
  }
  __syncthreads();
  // coalesced write-out, digit run by digit run
  const uint32_t nt = s.ntile;
  for (uint32_t i = tid; i < nt; i += kPartThreads) {
    const uint32_t d = s.dout[i];
    const uint32_t g = s.gbase[d] + (i - s.loc[d]);
#pragma unroll
    for (int k = 0; k < K; ++k) out_key[k][g] = s.kout[k][i];
    out_let[g] = s.lout[i];
  }
}

// off[c] = first position of bucket c in the final order, off[NB] = n.
__global__ void bucket_bounds_kernel(const uint32_t *k0, const unsigned long long *nvalid, int bits,
                                     uint32_t *off, uint32_t nb) {
  const unsigned long long n = *nvalid;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const long long prev = i == 0 ? -1 : (long long)bucket_of(k0[i - 1], bits);
    const long long cur = i == n ? (long long)nb : (long long)bucket_of(k0[i], bits);
    for (long long c = prev + 1; c <= cur; ++c) off[c] = (uint32_t)i;
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

cudaError_t launch_part_count(const PartPlan &p, int pass, const Launcher &L) {
  if (pass == 0) {
    switch (p.K) {
      case 1: LTL4C_LAUNCH(kKPartCount, part_count_kernel<1, true><<<p.n_tiles, kPartThreads, 0, L.stream>>>(p, pass));
      case 2: LTL4C_LAUNCH(kKPartCount, part_count_kernel<2, true><<<p.n_tiles, kPartThreads, 0, L.stream>>>(p, pass));
      default: LTL4C_LAUNCH(kKPartCount, part_count_kernel<3, true><<<p.n_tiles, kPartThreads, 0, L.stream>>>(p, pass));
    }
  }
  LTL4C_LAUNCH(kKPartCount, part_count_kernel<1, false><<<p.n_tiles, kPartThreads, 0, L.stream>>>(p, pass));
}

cudaError_t launch_part_scan(const PartPlan &p, int pass, const Launcher &L) {
  LTL4C_LAUNCH(kKPartScan, part_scan_kernel<<<1u << p.width[pass], 1024, 0, L.stream>>>(p, pass));
}

template <int K>
static cudaError_t scatter(const PartPlan &p, int pass, const Launcher &L) {
  const size_t sm = sizeof(SweepSmem<K>);
  cudaFuncSetAttribute(part_scatter_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  LTL4C_LAUNCH(kKPartScatter, part_scatter_kernel<K><<<p.n_tiles, kPartThreads, sm, L.stream>>>(p, pass));
}

cudaError_t launch_part_scatter(const PartPlan &p, int pass, const Launcher &L) {
  switch (p.K) {
    case 1: return scatter<1>(p, pass, L);
    case 2: return scatter<2>(p, pass, L);
    default: return scatter<3>(p, pass, L);
  }
}

cudaError_t launch_bucket_bounds(const PartPlan &p, uint32_t *off, uint32_t n_buckets, const Launcher &L) {
  const uint32_t *k0 = p.buf_key[(p.passes - 1) & 1][0];
  const unsigned grid = (unsigned)((p.n + 1 + 255) / 256 > 148 * 16 ? 148 * 16 : (p.n + 1 + 255) / 256);
  LTL4C_LAUNCH(kKBucketBounds, bucket_bounds_kernel<<<grid ? grid : 1, 256, 0, L.stream>>>(k0, p.nvalid, p.bits, off, n_buckets));
}

}  // namespace ltl4c
