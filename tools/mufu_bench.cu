// Microbenchmark (development aid): MUFU.EX2 and FFMA2 issue throughput per
// SM sub-partition.  One CTA per SM with W warps (W/4 per SMSP); each warp
// runs 8 independent chains.  Prints clk per warp-instruction per SMSP.
#include <cstdio>
#include <cstdint>
__global__ void ex2_bench(float* out, long long* clk, int iters) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = -0.001f * (threadIdx.x + k);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
__global__ void ffma2_bench(float* out, long long* clk, int iters) {
  uint64_t a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  const uint64_t b = 0x3f8000003f800000ull;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a[k]) : "l"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  uint64_t s = 0;
  for (int k = 0; k < 8; ++k) s ^= a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
__global__ void f2fp_bench(float* out, long long* clk, int iters) {
  uint32_t a[8];
  float x = threadIdx.x * 0.5f;
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(a[k]) : "f"(__uint_as_float(a[k])), "f"(x));
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
  for (int k = 0; k < 8; ++k) s ^= a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 4096;
  for (int w : {4, 8, 16}) {
    for (int kind = 0; kind < 3; ++kind) {
      for (int rep = 0; rep < 2; ++rep) {
        if (kind == 0) ex2_bench<<<sms, 32 * w>>>(out, clk, iters);
        else if (kind == 1) ffma2_bench<<<sms, 32 * w>>>(out, clk, iters);
        else f2fp_bench<<<sms, 32 * w>>>(out, clk, iters);
        cudaDeviceSynchronize();
      }
      long long h[148]; cudaMemcpy(h, clk, sms * 8, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
      const double instr_per_smsp = (double)iters * 8 * (w / 4);
      printf("{\"op\": \"%s\", \"warps_per_smsp\": %d, \"clk_per_warp_instr_per_smsp\": %.2f}\n",
             kind == 0 ? "MUFU.EX2" : kind == 1 ? "FFMA2" : "F2FP.BF16 (cvt.rn.bf16x2.f32)", w / 4,
             avg / instr_per_smsp);
    }
  }
  return 0;
}
