// Block-to-rank distribution kernels (reference src/mmplan/balance.py).
//
//   lpt_distribute     balance.py:58-76   sort (-w, id) + argmin (load, gpu)
//   zigzag_distribute  balance.py:79-102  2G chunks, GPU i gets i and 2G-1-i
//   split_block        balance.py:217-220 (pieces for intra_schedule)
//   intra_schedule     balance.py:251-259 list scheduling == LPT over pieces
//   contiguous split   (not in the reference; BASELINE.json config 5 baseline)
//
// The heap in the reference always holds one (load, g) entry per GPU, so a
// pop is argmin over (load, g): the sequential step here is one warp-wide
// min-reduction per item.  The sort key is (INT32_MAX - w) << 32 | id.
#include "../../include/bam.h"
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace bam {

__device__ __forceinline__ uint64_t lpt_key(int32_t w, int64_t i) {
  return (uint64_t(uint32_t(0x7FFFFFFF - w)) << 32) | uint64_t(uint32_t(i));
}

// One-CTA bitonic sort in shared memory (n_pad power of two <= kSortSmemMax).
__global__ void __launch_bounds__(1024) sort_smem_kernel(const int32_t* __restrict__ w,
                                                         int64_t n, int64_t n_pad,
                                                         uint64_t* __restrict__ sorted,
                                                         int32_t* __restrict__ order) {
  extern __shared__ uint64_t keys[];
  for (int64_t i = threadIdx.x; i < n_pad; i += blockDim.x)
    keys[i] = i < n ? lpt_key(w[i], i) : ~0ull;
  __syncthreads();
  for (int64_t k = 2; k <= n_pad; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < n_pad; i += blockDim.x) {
        const int64_t p = i ^ j;
        if (p > i) {
          const uint64_t a = keys[i], b = keys[p];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    if (sorted) sorted[i] = keys[i];
    if (order) order[i] = (int32_t)uint32_t(keys[i]);
  }
}

// Multi-CTA bitonic sort in global memory for large n: init + one launch per stage.
__global__ void sort_init_kernel(const int32_t* __restrict__ w, int64_t n, int64_t n_pad,
                                 uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad;
       i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = i < n ? lpt_key(w[i], i) : ~0ull;
}
__global__ void sort_stage_kernel(uint64_t* __restrict__ keys, int64_t n_pad, int64_t k,
                                  int64_t j) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i ^ j;
    if (p > i) {
      const uint64_t a = keys[i], b = keys[p];
      if ((a > b) == ((i & k) == 0)) {
        keys[i] = b;
        keys[p] = a;
      }
    }
  }
}

// Sequential greedy assignment by one warp, then per-unit CSR scatter.
// rank[] (workspace) holds each item's position within its unit's list.
__global__ void __launch_bounds__(1024) lpt_assign_kernel(
    const int32_t* __restrict__ w, const uint64_t* __restrict__ sorted, int64_t n, int32_t G,
    int32_t* __restrict__ owner, int32_t* __restrict__ rank, int32_t* __restrict__ flat,
    int32_t* __restrict__ off, int64_t* __restrict__ loads_out) {
  extern __shared__ uint64_t sh[];
  uint64_t* load = sh;                                  // [G]
  int32_t* cnt = reinterpret_cast<int32_t*>(sh + G);    // [G]
  __shared__ unsigned long long total;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    load[g] = 0;
    cnt[g] = 0;
  }
  if (threadIdx.x == 0) total = 0;
  __syncthreads();
  unsigned long long part = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) part += (unsigned long long)w[i];
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&total, part);
  __syncthreads();
  // fast path: G <= 32 and every partial load < 2^27 so (load << 5 | g) fits 32 bits
  const bool use_fast = G <= 32 && total < (1ull << 27);
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    if (use_fast) {
      // G <= 32 and total load < 2^27: key = load << 5 | g fits 32 bits.
      uint32_t my = lane < (uint32_t)G ? lane : 0xFFFFFFFFu;  // load 0, unit = lane
      int32_t my_cnt = 0;
      for (int64_t i = 0; i < n; ++i) {
        const int64_t item = int64_t(uint32_t(sorted[i]));
        const uint32_t best = __reduce_min_sync(0xffffffffu, my);
        const uint32_t g = best & 31u;
        if (lane == g) {
          owner[item] = (int32_t)g;
          rank[item] = my_cnt++;
          my += uint32_t(w[item]) << 5;
        }
      }
      if (lane < (uint32_t)G) {
        load[lane] = my >> 5;
        cnt[lane] = my_cnt;
      }
    } else {
      for (int64_t i = 0; i < n; ++i) {
        const int64_t item = int64_t(uint32_t(sorted[i]));
        uint64_t bl = ~0ull;
        int32_t bg = 0x7FFFFFFF;
        for (int g = lane; g < G; g += 32) {
          const uint64_t l = load[g];
          if (l < bl) { bl = l; bg = g; }   // g ascending: ties keep the lower g
        }
        for (int o = 16; o; o >>= 1) {
          const uint64_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
          const int32_t og = __shfl_xor_sync(0xffffffffu, bg, o);
          if (ol < bl || (ol == bl && og < bg)) { bl = ol; bg = og; }
        }
        if (lane == (uint32_t)(bg & 31)) {
          owner[item] = bg;
          rank[item] = cnt[bg]++;
          load[bg] = bl + uint64_t(w[item]);
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int g = 0; g < G; ++g) {
      off[g] = acc;
      acc += cnt[g];
      loads_out[g] = (int64_t)load[g];
    }
    off[G] = acc;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) flat[off[owner[i]] + rank[i]] = (int32_t)i;
}

// Zigzag (balance.py:79-102) and contiguous splits: closed-form chunking.
__device__ __forceinline__ int64_t chunk_start(int64_t c, int64_t base, int64_t extra) {
  return c * base + (c < extra ? c : extra);
}
__device__ __forceinline__ int64_t chunk_size(int64_t c, int64_t base, int64_t extra) {
  return base + (c < extra ? 1 : 0);
}

__global__ void __launch_bounds__(1024) chunk_assign_kernel(const int32_t* __restrict__ w,
                                                            int64_t n, int32_t G, int zigzag,
                                                            int32_t* __restrict__ owner,
                                                            int32_t* __restrict__ flat,
                                                            int32_t* __restrict__ off,
                                                            int64_t* __restrict__ loads) {
  extern __shared__ unsigned long long lsh[];  // [G] loads
  const int64_t nchunks = zigzag ? 2 * (int64_t)G : G;
  const int64_t base = n / nchunks, extra = n % nchunks;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    lsh[g] = 0;
    int64_t o = 0;
    for (int h = 0; h < g; ++h)
      o += chunk_size(h, base, extra) + (zigzag ? chunk_size(nchunks - 1 - h, base, extra) : 0);
    off[g] = (int32_t)o;
    if (g == G - 1) off[G] = (int32_t)n;
  }
  __syncthreads();
  for (int64_t b = threadIdx.x; b < n; b += blockDim.x) {
    // chunk of b: the first `extra` chunks hold base+1 blocks
    const int64_t big = extra * (base + 1);
    const int64_t c = b < big ? b / (base + 1) : extra + (b - big) / (base > 0 ? base : 1);
    int64_t g, pos;
    if (!zigzag || c < G) {
      g = c;
      pos = b - chunk_start(c, base, extra);
    } else {
      g = nchunks - 1 - c;
      pos = chunk_size(g, base, extra) + (b - chunk_start(c, base, extra));
    }
    owner[b] = (int32_t)g;
    atomicAdd(&lsh[g], (unsigned long long)w[b]);
    // offsets are needed before the flat write: recompute (off[] written above)
    int64_t o = 0;
    for (int h = 0; h < g; ++h)
      o += chunk_size(h, base, extra) + (zigzag ? chunk_size(nchunks - 1 - h, base, extra) : 0);
    flat[o + pos] = (int32_t)b;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) loads[g] = (int64_t)lsh[g];
}

__global__ void split_count_kernel(const int32_t* __restrict__ w, int64_t n, int32_t s,
                                   int32_t* __restrict__ cnt) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
       b += (int64_t)gridDim.x * blockDim.x)
    cnt[b] = (w[b] + s - 1) / s;
}
__global__ void split_fill_kernel(const int32_t* __restrict__ w, int64_t n, int32_t s,
                                  const int32_t* __restrict__ off, int32_t* __restrict__ size,
                                  int32_t* __restrict__ blk, int32_t* __restrict__ idx) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int32_t wb = w[b], full = wb / s, rem = wb % s;
    const int32_t o = off[b];
    for (int32_t i = 0; i < full; ++i) {
      size[o + i] = s;
      blk[o + i] = (int32_t)b;
      idx[o + i] = i;
    }
    if (rem) {
      size[o + full] = rem;
      blk[o + full] = (int32_t)b;
      idx[o + full] = full;
    }
  }
}


}  // namespace bam

using namespace bam;

static int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

extern "C" {

int64_t bam_lpt_workspace_bytes(int64_t n) {
  // sorted keys (n_pad u64) + rank (n i32), 256-B aligned pieces
  const int64_t np = next_pow2(n < 1 ? 1 : n);
  return ((np * 8 + 255) / 256) * 256 + ((n * 4 + 255) / 256) * 256;
}

int bam_lpt_assign(const int32_t* w, int64_t n, int32_t G, int32_t* owner, int32_t* flat,
                   int32_t* off, int64_t* loads, void* workspace, void* stream) {
  BAM_CHECK_ARG(G >= 1, "num_gpus must be >= 1");
  BAM_CHECK_ARG(n >= 1, "workloads must be nonempty");
  BAM_CHECK_ARG(n < (1ll << 31) && G <= 8192, "bam_lpt_assign: n=%lld G=%d unsupported",
                (long long)n, G);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t np = next_pow2(n);
  uint8_t* ws = (uint8_t*)workspace;
  uint64_t* keys = (uint64_t*)ws;
  int32_t* rank = (int32_t*)(ws + ((np * 8 + 255) / 256) * 256);
  if (np <= kSortSmemMax) {
    const size_t smem = np * sizeof(uint64_t);
    BAM_CUDA_TRY(cudaFuncSetAttribute(sort_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    sort_smem_kernel<<<1, 1024, smem, s>>>(w, n, np, keys, nullptr);
    BAM_LAUNCH_CHECK();
  } else {
    const int grid = 148 * 8;
    sort_init_kernel<<<grid, 256, 0, s>>>(w, n, np, keys);
    for (int64_t k = 2; k <= np; k <<= 1)
      for (int64_t j = k >> 1; j > 0; j >>= 1) sort_stage_kernel<<<grid, 256, 0, s>>>(keys, np, k, j);
    BAM_LAUNCH_CHECK();
  }
  const size_t smem = (size_t)G * (sizeof(uint64_t) + sizeof(int32_t));
  BAM_CUDA_TRY(cudaFuncSetAttribute(lpt_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  lpt_assign_kernel<<<1, 1024, smem, s>>>(w, keys, n, G, owner, rank, flat, off, loads);
  BAM_LAUNCH_CHECK();
  return kOk;
}

static int chunk_assign(const int32_t* w, int64_t n, int32_t G, int zz, int32_t* owner,
                        int32_t* flat, int32_t* off, int64_t* loads, void* stream) {
  BAM_CHECK_ARG(G >= 1, "num_gpus must be >= 1");
  BAM_CHECK_ARG(n >= 1, "workloads must be nonempty");
  BAM_CHECK_ARG(G <= 16384 && n < (1ll << 31), "chunk assign: G=%d unsupported", G);
  const size_t smem = (size_t)G * sizeof(unsigned long long);
  BAM_CUDA_TRY(cudaFuncSetAttribute(chunk_assign_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  chunk_assign_kernel<<<1, 1024, smem, (cudaStream_t)stream>>>(w, n, G, zz, owner, flat, off,
                                                               loads);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_zigzag_assign(const int32_t* w, int64_t n, int32_t G, int32_t* owner, int32_t* flat,
                      int32_t* off, int64_t* loads, void* stream) {
  return chunk_assign(w, n, G, 1, owner, flat, off, loads, stream);
}

int bam_contiguous_assign(const int32_t* w, int64_t n, int32_t G, int32_t* owner, int32_t* flat,
                          int32_t* off, int64_t* loads, void* stream) {
  return chunk_assign(w, n, G, 0, owner, flat, off, loads, stream);
}

int bam_split_count(const int32_t* w, int64_t n, int32_t s, int32_t* piece_cnt,
                    int32_t* piece_off, void* stream) {
  BAM_CHECK_ARG(s >= 1, "subblock_size must be >= 1");
  BAM_CHECK_ARG(n >= 0, "bam_split_count: n=%lld", (long long)n);
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) {
    BAM_CUDA_TRY(cudaMemsetAsync(piece_off, 0, sizeof(int32_t), st));
    return kOk;
  }
  split_count_kernel<<<148, 256, 0, st>>>(w, n, s, piece_cnt);
  scan_kernel<<<1, 1024, 0, st>>>(piece_cnt, n, piece_off);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_split_fill(const int32_t* w, int64_t n, int32_t s, const int32_t* piece_off,
                   int32_t* piece_size, int32_t* piece_block, int32_t* piece_index, void* stream) {
  BAM_CHECK_ARG(s >= 1, "subblock_size must be >= 1");
  if (n == 0) return kOk;
  split_fill_kernel<<<148, 256, 0, (cudaStream_t)stream>>>(w, n, s, piece_off, piece_size,
                                                           piece_block, piece_index);
  BAM_LAUNCH_CHECK();
  return kOk;
}

}  // extern "C"
