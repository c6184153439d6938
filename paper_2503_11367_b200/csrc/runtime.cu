// Host-side runtime of libbam: error reporting, the exact ILP oracle of the
// reference API (balance.py:124-192, host C++), fp32->bf16 conversion and the
// tcgen05/TMA self test.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <set>
#include <vector>

#include "../../include/bam.h"
#include "common.cuh"
#include "tma.h"

namespace bam {

static thread_local char g_last_error[1024] = "";

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

// ----------------------------------------------------------------------------- ILP (host)
// balance.py:106-121 (_feasible): can `jobs` be packed with every load <= limit?
static bool feasible(const int64_t* jobs, int n, std::vector<int64_t>& loads, int64_t limit) {
  if (n == 0) return true;
  std::set<int64_t> tried;  // identical loads are symmetric
  for (size_t g = 0; g < loads.size(); ++g) {
    if (!tried.insert(loads[g]).second) continue;
    if (loads[g] + jobs[0] <= limit) {
      loads[g] += jobs[0];
      const bool ok = feasible(jobs + 1, n - 1, loads, limit);
      loads[g] -= jobs[0];
      if (ok) return true;
    }
  }
  return false;
}

struct Search {
  std::vector<int64_t> jobs;
  int64_t best, lower;
  int G;
  void run(size_t idx, std::vector<int64_t>& loads) {  // balance.py:148-163
    if (best == lower) return;
    if (idx == jobs.size()) {
      best = std::min(best, *std::max_element(loads.begin(), loads.end()));
      return;
    }
    std::set<int64_t> tried;
    for (int g = 0; g < G; ++g) {
      if (!tried.insert(loads[g]).second) continue;
      if (loads[g] + jobs[idx] >= best) continue;
      loads[g] += jobs[idx];
      run(idx + 1, loads);
      loads[g] -= jobs[idx];
    }
  }
};

__global__ void f32_to_bf16_kernel(const float4* __restrict__ src, uint2* __restrict__ dst,
                                   int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    dst[i] = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  }
}

}  // namespace bam

using namespace bam;

extern "C" {

const char* bam_last_error(void) { return g_last_error; }

int bam_version(void) { return 2; }

int64_t bam_sizeof(const char* name) {
  if (name == nullptr) return -1;
  if (!strcmp(name, "BamBlockSummary")) return sizeof(BamBlockSummary);
  if (!strcmp(name, "BamAttnFwdParams")) return sizeof(BamAttnFwdParams);
  if (!strcmp(name, "BamAttnBwdParams")) return sizeof(BamAttnBwdParams);
  if (!strcmp(name, "BamPlan")) return sizeof(BamPlan);
  return -1;
}

int bam_ilp_optimal(const int64_t* w, int32_t n, int32_t G, int32_t* assignment,
                    int64_t* makespan) {
  if (n < 1) {
    set_last_error("workloads must be nonempty");
    return BAM_INVALID_ARGUMENT;
  }
  if (n > 14 || G > 4) {
    set_last_error("instance (%d blocks, %d GPUs) exceeds the exact-search budget (14 blocks, 4 GPUs)",
                   n, G);
    return BAM_BUDGET_EXCEEDED;
  }
  if (G < 1) {
    set_last_error("num_gpus must be >= 1");
    return BAM_INVALID_ARGUMENT;
  }
  Search s;
  s.G = G;
  s.jobs.assign(w, w + n);
  std::stable_sort(s.jobs.begin(), s.jobs.end(), [](int64_t a, int64_t b) { return a > b; });
  int64_t total = 0;
  for (int64_t j : s.jobs) total += j;
  s.lower = std::max(s.jobs[0], (total + G - 1) / G);
  s.best = total;
  std::vector<int64_t> loads(G, 0);
  s.run(0, loads);
  const int64_t opt = s.best;
  // lexicographic extraction (balance.py:169-189)
  std::vector<int> by_size(n);
  for (int i = 0; i < n; ++i) by_size[i] = i;
  std::stable_sort(by_size.begin(), by_size.end(), [&](int a, int b) { return w[a] > w[b]; });
  std::vector<int> asg(n, -1);
  std::fill(loads.begin(), loads.end(), 0);
  for (int b = 0; b < n; ++b) {
    bool placed = false;
    for (int g = 0; g < G && !placed; ++g) {
      if (loads[g] + w[b] > opt) continue;
      loads[g] += w[b];
      asg[b] = g;
      std::vector<int64_t> rem;
      for (int j : by_size)
        if (asg[j] == -1) rem.push_back(w[j]);
      if (feasible(rem.data(), (int)rem.size(), loads, opt)) {
        placed = true;
      } else {
        loads[g] -= w[b];
        asg[b] = -1;
      }
    }
    if (!placed) {
      set_last_error("internal error: optimal makespan not extractable");
      return BAM_INVALID_ARGUMENT;
    }
  }
  for (int b = 0; b < n; ++b) assignment[b] = asg[b];
  *makespan = opt;
  return BAM_OK;
}

int bam_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream) {
  BAM_CHECK_ARG(n % 4 == 0, "bam_f32_to_bf16: n=%lld must be a multiple of 4", (long long)n);
  const int64_t n4 = n / 4;
  if (n4 == 0) return kOk;
  int64_t grid = (n4 + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  f32_to_bf16_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(src), reinterpret_cast<uint2*>(dst), n4);
  BAM_LAUNCH_CHECK();
  return kOk;
}

}  // extern "C"

// Stream-ordered flag store (cuStreamWriteValue32 through the runtime's driver
// entry point, so libbam needs no -lcuda): no SM involved, ordered after the
// stream's previous work with a memory barrier.
extern "C" int bam_stream_write_i32(int32_t* dst, int32_t value, void* stream) {
  using Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static Fn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &ptr, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      bam::set_last_error("cuStreamWriteValue32 unavailable from the driver");
      return bam::kCudaError;
    }
    fn = reinterpret_cast<Fn>(ptr);
  }
  BAM_CHECK_ARG(dst != nullptr && (reinterpret_cast<uintptr_t>(dst) & 3) == 0,
                "bam_stream_write_i32: bad destination");
  const CUresult r = fn((CUstream)stream, (CUdeviceptr)dst, (cuuint32_t)value, 0);
  if (r != CUDA_SUCCESS) {
    bam::set_last_error("cuStreamWriteValue32 failed (%d)", (int)r);
    return bam::kCudaError;
  }
  return bam::kOk;
}

// Strided copy on the stream's copy engine (cudaMemcpy2DAsync, UVA direction:
// a peer's symmetric buffer works as the source): height rows of width bytes.
extern "C" int bam_copy_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                           int64_t width, int64_t height, void* stream) {
  BAM_CHECK_ARG(dst && src && width > 0 && height > 0 && dpitch >= width && spitch >= width,
                "bam_copy_2d: bad arguments");
  BAM_CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width,
                                 (size_t)height, cudaMemcpyDefault, (cudaStream_t)stream));
  return bam::kOk;
}

extern "C" int bam_stream_wait_i32_geq(const int32_t* src, int32_t value, void* stream) {
  using Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static Fn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &ptr, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      bam::set_last_error("cuStreamWaitValue32 unavailable from the driver");
      return bam::kCudaError;
    }
    fn = reinterpret_cast<Fn>(ptr);
  }
  BAM_CHECK_ARG(src != nullptr && (reinterpret_cast<uintptr_t>(src) & 3) == 0,
                "bam_stream_wait_i32_geq: bad source");
  const CUresult r = fn((CUstream)stream, (CUdeviceptr)src, (cuuint32_t)value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) {
    bam::set_last_error("cuStreamWaitValue32 failed (%d)", (int)r);
    return bam::kCudaError;
  }
  return bam::kOk;
}
