// Microbenchmark (development aid): tcgen05.ld / tcgen05.st throughput per SM
// with W warps per CTA (one CTA per SM), 32x32b shapes of 16/32/64 columns.
// Each warp reads (or writes) its own TMEM lane quadrant (warp % 4), walking
// the 512 columns; every load is waited (tcgen05.wait::ld) before the next so
// the registers are really produced.  Prints bytes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/tmem_bench.cu -o gpurun_out/tmem_bench -lcuda
#include "../paper_2503_11367_b200/csrc/common.cuh"

using namespace bam;

constexpr int kIters = 2048;

#define LD16(taddr, r)                                                                       \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10," \
               "%11,%12,%13,%14,%15}, [%16];"                                              \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),    \
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),  \
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                         \
               : "r"(taddr))

// kOp 0: ld x16, 1: ld x32, 2: two ld x32 then one wait, 3: st x32, 4: st x16
template <int kOp>
__global__ void __launch_bounds__(512, 1) tmem_bench(long long* out, uint32_t* sink) {
  __shared__ uint32_t tmem_base;
  const uint32_t warp = warp_id();
  if (warp == 0) {
    tmem_alloc(&tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base + (((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kIters; ++i) {
    const uint32_t col = (uint32_t)((i * 64 + (warp >> 2) * 32) & 511);
    if constexpr (kOp == 0) {
      uint32_t r[16];
      LD16(tmem + (col & ~15u), r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) acc ^= r[j];
    } else if constexpr (kOp == 1) {
      uint32_t r[32];
      BAM_TMEM_LD32(tmem + (col & ~31u), r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= r[j];
    } else if constexpr (kOp == 2) {
      uint32_t r[32], s[32];
      BAM_TMEM_LD32(tmem + (col & ~63u), r);
      BAM_TMEM_LD32(tmem + (col & ~63u) + 32, s);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= r[j] + s[j];
    } else if constexpr (kOp == 3) {
      uint32_t r[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) r[j] = acc + j;
      BAM_TMEM_ST32(tmem + (col & ~31u), r);
      tmem_wait_st();
      acc += 1;
    } else {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) r[j] = acc + j;
      BAM_TMEM_ST16(tmem + (col & ~15u), r);
      tmem_wait_st();
      acc += 1;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int kOp>
static void run(const char* name, int warps, int sms, long long* d_out, uint32_t* sink) {
  tmem_bench<kOp><<<sms, warps * 32>>>(d_out, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  long long h[1024];
  cudaMemcpy(h, d_out, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long sum = 0;
  for (int i = 0; i < sms; ++i) sum += h[i];
  const double cyc = double(sum) / sms;
  const int cols = kOp == 0 || kOp == 4 ? 16 : (kOp == 2 ? 64 : 32);
  const double bytes = double(warps) * kIters * 32 * cols * 4;
  printf("{\"op\": \"%s\", \"warps\": %d, \"cols_per_op\": %d, \"cycles\": %.0f, "
         "\"bytes_per_clk_per_sm\": %.1f}\n", name, warps, cols, cyc, bytes / cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d_out;
  uint32_t* sink;
  cudaMalloc(&d_out, sizeof(long long) * 1024);
  cudaMalloc(&sink, 4 * 1024);
  for (int w : {4, 8, 12, 16}) {
    run<0>("ld_x16", w, sms, d_out, sink);
    run<1>("ld_x32", w, sms, d_out, sink);
    run<2>("ld_2x32", w, sms, d_out, sink);
    run<3>("st_x32", w, sms, d_out, sink);
    run<4>("st_x16", w, sms, d_out, sink);
  }
  return 0;
}
