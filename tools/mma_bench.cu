// Microbenchmark (development aid): tcgen05.mma throughput per shape / operand
// source on one CTA per SM.  Operands are uninitialised shared memory / TMEM
// (throughput does not depend on values).  Prints cycles per MMA and the
// achieved fraction of 8192 dense bf16 flop/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/mma_bench.cu -o gpurun_out/mma_bench -lcuda
#include "../paper_2503_11367_b200/csrc/common.cuh"

using namespace bam;

constexpr int kIters = 4096;

struct alignas(1024) BenchSmem {
  uint8_t a[65536];
  uint8_t b[65536];
  uint64_t bar;
  uint32_t tmem;
};

// mode 0: SS K-major x K-major; 1: TS (A from TMEM) x K-major; 2: SS MN-major x MN-major
template <int kMode, int kN>
__global__ void __launch_bounds__(128, 1) mma_bench(long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  BenchSmem& sm = *reinterpret_cast<BenchSmem*>(raw);
  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) {
    mbar_init(&sm.bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&sm.tmem, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  if (warp == 0) {
    const uint32_t leader = elect_one();
    const uint32_t id = idesc_bf16(128, kN, kMode == 2, kMode == 2);
    const uint64_t da = sdesc_sw128(smem_u32(sm.a), kMode == 2 ? 16384 : 16, 1024);
    const uint64_t db = sdesc_sw128(smem_u32(sm.b), kMode == 2 ? 16384 : 16, 1024);
    const uint32_t tD = tmem + 256, tA = tmem;  // D: up to 256 columns; A: 64 columns
    __syncwarp();
    const long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < kIters; i += 8) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = kMode == 2 ? kk * 128 : ((kk >> 2) * 1024 + (kk & 3) * 2);
        if (kMode == 1)
          mma_ts_w(tD, tA + 8 * kk, db + off, id, kk > 0, leader);
        else
          mma_ss_w(tD, da + off, db + off, id, kk > 0, leader);
      }
    }
    tc_commit_w(&sm.bar, leader);
    mbar_wait_sleep(&sm.bar, 0);
    const long long t1 = clock64();
    if (lane_id() == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int kMode, int kN>
static void run(const char* name, int sms, long long* d_out) {
  auto k = mma_bench<kMode, kN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BenchSmem));
  k<<<sms, 128, sizeof(BenchSmem)>>>(d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  long long h[1024];
  cudaMemcpy(h, d_out, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0, sum = 0;
  for (int i = 0; i < sms; ++i) {
    sum += h[i];
    mx = h[i] > mx ? h[i] : mx;
  }
  const double cyc = double(sum) / sms / kIters;
  const double ideal = 2.0 * 128 * kN * 16 / 8192.0;
  printf("{\"shape\": \"%s\", \"N\": %d, \"cycles_per_mma\": %.2f, \"ideal\": %.1f, \"frac\": %.3f}\n",
         name, kN, cyc, ideal, ideal / cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d_out;
  cudaMalloc(&d_out, sizeof(long long) * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    run<0, 32>("SS", sms, d_out);
    run<0, 64>("SS", sms, d_out);
    run<0, 128>("SS", sms, d_out);
    run<0, 256>("SS", sms, d_out);
    run<1, 32>("TS", sms, d_out);
    run<1, 64>("TS", sms, d_out);
    run<1, 128>("TS", sms, d_out);
    run<1, 256>("TS", sms, d_out);
    run<2, 64>("SS_MN", sms, d_out);
    run<2, 128>("SS_MN", sms, d_out);
  }
  return 0;
}
