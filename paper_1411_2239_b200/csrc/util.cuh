// util.cuh -- small warp/block primitives shared by the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ltl4c {
namespace {

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan of n (<= blockDim * per) values held in smem `a` (u32), in place.
// Returns the total.  All threads of the block must call it.
__device__ uint32_t block_exclusive_scan(uint32_t *a, int n, uint32_t *warp_tot) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int per = (n + nt - 1) / nt;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  uint32_t s = 0;
  for (int i = lo; i < hi; ++i) s += a[i];
  uint32_t x = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int nw = nt >> 5;
    uint32_t w = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < nw) warp_tot[lane] = w;  // inclusive
  }
  __syncthreads();
  uint32_t base = (x - s) + (wid ? warp_tot[wid - 1] : 0);
  for (int i = lo; i < hi; ++i) {
    uint32_t v = a[i];
    a[i] = base;
    base += v;
  }
  uint32_t total = warp_tot[(nt >> 5) - 1];
  __syncthreads();
  return total;
}


__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

}  // namespace
}  // namespace ltl4c
