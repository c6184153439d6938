// Single-CTA exclusive scan shared by the mask and assignment kernels.
#pragma once
#include "common.cuh"

namespace bam {

// single-CTA exclusive scan of n int32 -> off[n+1]
static __global__ void scan_kernel(const int32_t* __restrict__ cnt, int64_t n, int32_t* __restrict__ off) {
  __shared__ int32_t carry;
  __shared__ int32_t warp_sums[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    int32_t v = i < n ? cnt[i] : 0, x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane_id() >= (uint32_t)o) x += y;
    }
    if (lane_id() == 31) warp_sums[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int32_t w = threadIdx.x < (blockDim.x >> 5) ? warp_sums[threadIdx.x] : 0, z = w;
      for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane_id() >= (uint32_t)o) z += y;
      }
      warp_sums[threadIdx.x] = z - w;
    }
    __syncthreads();
    const int32_t excl = carry + warp_sums[threadIdx.x >> 5] + x - v;
    if (i < n) off[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[n] = carry;
}

}  // namespace bam
