// Development aid: checks the SWIZZLE_NONE K-major shared-memory descriptor for
// a K = 16 tcgen05.mma (the backward's bias MMA): D[128 x 64] = A[128 x 16] B[64 x 16]^T
// with A / B in the canonical core-matrix layout [k chunk][row group][8 rows][16 B].
// Prints the max error for each (LBO, SBO) interpretation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/umma_k16_test.cu -o /tmp/umma_k16_test -lcuda
#include <cstdio>
#include <vector>

#include "../paper_2503_11367_b200/csrc/common.cuh"

using namespace bam;

__device__ __forceinline__ uint64_t sdesc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// a: [128][16] bf16 row-major values, b: [64][16]
__global__ void __launch_bounds__(128, 1) k16_kernel(const __nv_bfloat16* a, const __nv_bfloat16* b,
                                                     int variant, float* out) {
  __shared__ __align__(1024) __nv_bfloat16 sa[128 * 16];
  __shared__ __align__(1024) __nv_bfloat16 sb[64 * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const uint32_t warp = warp_id(), lane = lane_id();
  // canonical layout: element (r, k) at ((k / 8) * R/8 + r / 8) * 64 + (r % 8) * 8 + k % 8
  for (int i = threadIdx.x; i < 128 * 16; i += 128) {
    const int r = i / 16, k = i % 16;
    sa[((k / 8) * 16 + r / 8) * 64 + (r % 8) * 8 + k % 8] = a[i];
  }
  for (int i = threadIdx.x; i < 64 * 16; i += 128) {
    const int r = i / 16, k = i % 16;
    sb[((k / 8) * 8 + r / 8) * 64 + (r % 8) * 8 + k % 8] = b[i];
  }
  fence_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&tmem_base, 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    // A: k-chunk stride 16 row groups x 128 B = 2048, row-group stride 128
    // B: k-chunk stride 8 x 128 = 1024, row-group stride 128
    uint32_t lbo_a = 2048, sbo_a = 128, lbo_b = 1024, sbo_b = 128;
    if (variant == 1) {
      lbo_a = 128; sbo_a = 2048; lbo_b = 128; sbo_b = 1024;
    }
    const uint64_t da = sdesc_none(smem_u32(sa), lbo_a, sbo_a);
    const uint64_t db = sdesc_none(smem_u32(sb), lbo_b, sbo_b);
    mma_ss(tmem, da, db, idesc_bf16(128, 64, 0, 0), 0);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t row = warp * 32 + lane;
  for (int c = 0; c < 64; c += 32) {
    uint32_t r[32];
    BAM_TMEM_LD32(tmem + ((warp * 32) << 16) + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out[row * 64 + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
}

int main() {
  std::vector<__nv_bfloat16> a(128 * 16), b(64 * 16);
  std::vector<float> af(128 * 16), bf(64 * 16);
  for (int i = 0; i < 128 * 16; ++i) {
    af[i] = float((i * 37) % 17 - 8) / 8.f;
    a[i] = __float2bfloat16(af[i]);
    af[i] = __bfloat162float(a[i]);
  }
  for (int i = 0; i < 64 * 16; ++i) {
    bf[i] = float((i * 53) % 13 - 6) / 4.f;
    b[i] = __float2bfloat16(bf[i]);
    bf[i] = __bfloat162float(b[i]);
  }
  __nv_bfloat16 *da, *db;
  float* dout;
  cudaMalloc(&da, a.size() * 2);
  cudaMalloc(&db, b.size() * 2);
  cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 2; ++variant) {
    k16_kernel<<<1, 128>>>(da, db, variant, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("variant %d: %s\n", variant, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> out(128 * 64);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 64; ++c) {
        double ref = 0;
        for (int k = 0; k < 16; ++k) ref += double(af[r * 16 + k]) * bf[c * 16 + k];
        const double d = fabs(ref - out[r * 64 + c]);
        mx = d > mx ? d : mx;
      }
    printf("{\"variant\": %d, \"lbo_is_k_stride\": %s, \"max_err\": %.3g}\n", variant,
           variant == 0 ? "true" : "false", mx);
  }
  return 0;
}
