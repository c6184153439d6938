// tcgen05 / TMA self test: validates every operand mode the attention kernels
// use (SS with K-major A/B, TS with A in TMEM and an MN-major B, SS with an
// MN-major A) on one 128x128x128 bf16 problem per mode.
#include "../../include/bam.h"
#include "common.cuh"
#include "tma.h"

namespace bam {

struct SelftestSmem {
  alignas(1024) uint8_t a[32768];
  alignas(1024) uint8_t b[32768];
  alignas(1024) uint8_t v[32768];
  alignas(1024) uint8_t x[32768];
  uint64_t bar_load;
  uint64_t bar_mma;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(128, 1)
    selftest_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_x,
                    const __nv_bfloat16* __restrict__ a_glob, float* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SelftestSmem& sm = *reinterpret_cast<SelftestSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(&sm.bar_load, 1);
    mbar_init(&sm.bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (threadIdx.x == 0) {
    mbar_expect_tx(&sm.bar_load, 4 * 32768);
    const CUtensorMap* maps[4] = {&tm_a, &tm_b, &tm_v, &tm_x};
    uint8_t* dst[4] = {sm.a, sm.b, sm.v, sm.x};
    for (int t = 0; t < 4; ++t)
      for (int h = 0; h < 2; ++h) tma_load_3d(maps[t], &sm.bar_load, dst[t] + h * 16384, h * 64, 0, 0);
  }
  mbar_wait(&sm.bar_load, 0);

  // ---- test 1: D0 = A * B^T, both K-major (the S = Q K^T shape)
  if (threadIdx.x == 0) {
    tc_fence_after();
    const uint32_t idesc = idesc_bf16(128, 128, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
      mma_ss(tmem + 0, sdesc_sw128(smem_u32(sm.a) + off, 16, 1024),
             sdesc_sw128(smem_u32(sm.b) + off, 16, 1024), idesc, kk > 0);
    }
    tc_commit(&sm.bar_mma);
  }
  mbar_wait(&sm.bar_mma, 0);
  tc_fence_after();

  // ---- test 2: A (bf16) into TMEM cols 256..319, D1 = A[tmem] * V (V MN-major)
  {
    const uint32_t row = warp * 32 + lane;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a_glob + row * 128);
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = src[i];
    BAM_TMEM_ST32(tmem + ((warp * 32) << 16) + 256, r);
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = src[32 + i];
    BAM_TMEM_ST32(tmem + ((warp * 32) << 16) + 256 + 32, r);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc_fence_after();
    const uint32_t idesc = idesc_bf16(128, 128, 0, 1);
    for (int kk = 0; kk < 8; ++kk)
      mma_ts(tmem + 128, tmem + 256 + kk * 8, sdesc_sw128(smem_u32(sm.v) + kk * 2048, 16384, 1024),
             idesc, kk > 0);
    // ---- test 3: D2 = X^T * V, A MN-major (X stored [k][m]) and B MN-major
    const uint32_t idesc3 = idesc_bf16(128, 128, 1, 1);
    for (int kk = 0; kk < 8; ++kk)
      mma_ss(tmem + 384, sdesc_sw128(smem_u32(sm.x) + kk * 2048, 16384, 1024),
             sdesc_sw128(smem_u32(sm.v) + kk * 2048, 16384, 1024), idesc3, kk > 0);
    tc_commit(&sm.bar_mma);
  }
  mbar_wait(&sm.bar_mma, 1);
  tc_fence_after();

  const uint32_t row = warp * 32 + lane;
  const int cols[3] = {0, 128, 384};
  for (int t = 0; t < 3; ++t) {
    for (int c = 0; c < 128; c += 32) {
      uint32_t r[32];
      BAM_TMEM_LD32(tmem + ((warp * 32) << 16) + cols[t] + c, r);
      tmem_wait_ld();
      for (int i = 0; i < 32; ++i) out[(t * 128 + row) * 128 + c + i] = __uint_as_float(r[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace bam

using namespace bam;

extern "C" int bam_selftest_umma(const void* a, const void* b, const void* v, const void* x,
                                 float* out, void* stream) {
  CUtensorMap ma, mb, mv, mx;
  int rc;
  if ((rc = make_tmap_rows_heads_d128(&ma, a, 128, 1, 128))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mb, b, 128, 1, 128))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mv, v, 128, 1, 128))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mx, x, 128, 1, 128))) return rc;
  const int smem = sizeof(SelftestSmem) + 1024;
  BAM_CUDA_TRY(cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  selftest_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(ma, mb, mv, mx,
                                                          (const __nv_bfloat16*)a, out);
  BAM_LAUNCH_CHECK();
  return kOk;
}
