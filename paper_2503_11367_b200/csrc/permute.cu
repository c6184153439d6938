// Token permutation around CP attention: block-row gather /
// scatter of up to four tensors per launch.  Pure HBM streaming: every thread
// moves 16-B vectors, four in flight, over a grid of 148 x 8 CTAs.
#include "../../include/bam.h"
#include "common.cuh"

namespace bam {
namespace perm {

struct PermuteArgs {
  const uint4* src[BAM_PERMUTE_MAX];
  uint4* dst[BAM_PERMUTE_MAX];
  int64_t row_vec[BAM_PERMUTE_MAX];   // 16-B vectors per row
  int64_t total[BAM_PERMUTE_MAX];     // vectors per tensor = n_blocks * block_rows * row_vec
  int32_t n_tensors;
};

__global__ void __launch_bounds__(256) permute_kernel(const PermuteArgs a,
                                                      const int32_t* __restrict__ idx,
                                                      int32_t block_rows, int32_t scatter) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int t = 0; t < a.n_tensors; ++t) {
    const int64_t rv = a.row_vec[t], per_block = rv * block_rows, total = a.total[t];
    const uint4* __restrict__ src = a.src[t];
    uint4* __restrict__ dst = a.dst[t];
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < total;
         base += 4 * stride) {
      uint4 v[4];
      int64_t out[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = base + u * stride;
        out[u] = -1;
        if (e < total) {
          const int64_t blk = e / per_block, within = e - blk * per_block;
          const int64_t other = (int64_t)__ldg(idx + blk) * per_block + within;
          v[u] = __ldg(src + (scatter ? e : other));
          out[u] = scatter ? other : e;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (out[u] >= 0) dst[out[u]] = v[u];
    }
  }
}

// dst_c[row, h, 0:128] = bf16( sum_p src[p*part_stride + c*comp_stride +
//                                       h*head_stride + row*row_stride + 0:128] )
// One thread per 8 outputs (two float4 loads per part, one 16-B store); the
// output order is token-major so stores are fully coalesced, and every read
// is a whole 32-B sector run of 512 B per (row, head).
__global__ void __launch_bounds__(256) reduce_partials_kernel(
    const float* __restrict__ src, int32_t n_parts, int64_t part_stride, int64_t comp_stride,
    int64_t head_stride, int64_t row_stride, int32_t n_heads, int64_t n_rows,
    uint4* __restrict__ dst0, uint4* __restrict__ dst1, int32_t n_comp) {
  const int64_t per_comp = n_rows * n_heads * 16;
  const int64_t total = per_comp * n_comp;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / per_comp, r = e - c * per_comp;
    const int64_t v = r & 15, rh = r >> 4;
    const int64_t row = rh / n_heads, h = rh - row * n_heads;
    const float* p = src + c * comp_stride + h * head_stride + row * row_stride + v * 8;
    float4 a = __ldcs(reinterpret_cast<const float4*>(p));
    float4 b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
    for (int q = 1; q < n_parts; ++q) {
      const float4* pq = reinterpret_cast<const float4*>(p + q * part_stride);
      const float4 x = __ldcs(pq), y = __ldcs(pq + 1);
      a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
      b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
    }
    uint4 o;
    o.x = pack_bf16(a.x, a.y);
    o.y = pack_bf16(a.z, a.w);
    o.z = pack_bf16(b.x, b.y);
    o.w = pack_bf16(b.z, b.w);
    (c == 0 ? dst0 : dst1)[r] = o;
  }
}

// Token-major K/V [n, nkv, 128] bf16 -> head-major [nkv, rows_i, 128] at row
// offset off_i of up to two destinations (the copy-engine CP gather: this rank's
// shard into its symmetric buffer, which the peers pull, and into its own slot of
// the gathered buffer the forward reads).  One 16-B vector per thread per
// tensor: reads are contiguous, writes are 256-B runs per (token, head).
__global__ void __launch_bounds__(256) kv_head_major_kernel(
    const uint4* __restrict__ k, const uint4* __restrict__ v, int64_t n, int32_t nkv,
    uint4* __restrict__ k0, uint4* __restrict__ v0, int64_t rows0, int64_t off0,
    uint4* __restrict__ k1, uint4* __restrict__ v1, int64_t rows1, int64_t off1) {
  const int64_t per = n * nkv * 16;   // vectors per tensor
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < 2 * per; e += stride) {
    const bool is_v = e >= per;
    const int64_t i = is_v ? e - per : e;
    const uint4 x = __ldcs((is_v ? v : k) + i);
    const int64_t c = i & 15, th = i >> 4;
    const int64_t t = th / nkv, h = th - t * nkv;
    (is_v ? v0 : k0)[((h * rows0) + off0 + t) * 16 + c] = x;
    if (k1 != nullptr) (is_v ? v1 : k1)[((h * rows1) + off1 + t) * 16 + c] = x;
  }
}

}  // namespace perm
}  // namespace bam

using namespace bam;

extern "C" int bam_permute_blocks(const void* const* src, void* const* dst,
                                  const int64_t* row_bytes, int32_t n_tensors, const int32_t* idx,
                                  int32_t n_blocks, int32_t block_rows, int32_t scatter,
                                  void* stream) {
  BAM_CHECK_ARG(n_tensors >= 1 && n_tensors <= BAM_PERMUTE_MAX && src && dst && row_bytes,
                "bam_permute_blocks: n_tensors=%d (1..%d)", n_tensors, BAM_PERMUTE_MAX);
  BAM_CHECK_ARG(n_blocks >= 0 && block_rows >= 1, "bam_permute_blocks: n_blocks=%d block_rows=%d",
                n_blocks, block_rows);
  if (n_blocks == 0) return kOk;
  BAM_CHECK_ARG(idx != nullptr, "bam_permute_blocks: null idx");
  perm::PermuteArgs a = {};
  a.n_tensors = n_tensors;
  for (int t = 0; t < n_tensors; ++t) {
    BAM_CHECK_ARG(row_bytes[t] > 0 && row_bytes[t] % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(src[t]) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(dst[t]) & 15) == 0,
                  "bam_permute_blocks: tensor %d needs 16-byte aligned rows / pointers "
                  "(row_bytes=%lld)", t, (long long)row_bytes[t]);
    a.src[t] = static_cast<const uint4*>(src[t]);
    a.dst[t] = static_cast<uint4*>(dst[t]);
    a.row_vec[t] = row_bytes[t] / 16;
    a.total[t] = a.row_vec[t] * block_rows * (int64_t)n_blocks;
  }
  perm::permute_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(a, idx, block_rows, scatter);
  BAM_LAUNCH_CHECK();
  return kOk;
}

extern "C" int bam_reduce_partials_bf16(const float* src, int32_t n_parts, int64_t part_stride,
                                        int64_t comp_stride, int64_t head_stride,
                                        int64_t row_stride, int32_t n_heads, int64_t n_rows,
                                        void* dst0, void* dst1, void* stream) {
  BAM_CHECK_ARG(src && dst0 && n_parts >= 1 && n_heads >= 1 && n_rows >= 0,
                "bam_reduce_partials_bf16: n_parts=%d n_heads=%d n_rows=%lld", n_parts, n_heads,
                (long long)n_rows);
  BAM_CHECK_ARG((reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(dst0) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(dst1) & 15) == 0 &&
                    part_stride % 4 == 0 && comp_stride % 4 == 0 && head_stride % 4 == 0 &&
                    row_stride % 4 == 0,
                "bam_reduce_partials_bf16: pointers and strides must be 16-byte aligned");
  if (n_rows == 0) return kOk;
  perm::reduce_partials_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
      src, n_parts, part_stride, comp_stride, head_stride, row_stride, n_heads, n_rows,
      static_cast<uint4*>(dst0), static_cast<uint4*>(dst1), dst1 ? 2 : 1);
  BAM_LAUNCH_CHECK();
  return kOk;
}

extern "C" int bam_kv_head_major(const void* k, const void* v, int64_t n, int32_t nkv,
                                 void* k0, void* v0, int64_t rows0, int64_t off0, void* k1,
                                 void* v1, int64_t rows1, int64_t off1, void* stream) {
  BAM_CHECK_ARG(n >= 0 && nkv >= 1, "bam_kv_head_major: n=%lld nkv=%d", (long long)n, nkv);
  if (n == 0) return kOk;
  BAM_CHECK_ARG(k && v && k0 && v0 && off0 >= 0 && off0 + n <= rows0 &&
                    (k1 == nullptr || (v1 && off1 >= 0 && off1 + n <= rows1)),
                "bam_kv_head_major: n=%lld nkv=%d rows0=%lld off0=%lld rows1=%lld off1=%lld",
                (long long)n, nkv, (long long)rows0, (long long)off0, (long long)rows1,
                (long long)off1);
  BAM_CHECK_ARG(((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
                  reinterpret_cast<uintptr_t>(k0) | reinterpret_cast<uintptr_t>(v0) |
                  reinterpret_cast<uintptr_t>(k1) | reinterpret_cast<uintptr_t>(v1)) & 15) == 0,
                "bam_kv_head_major: pointers must be 16-byte aligned");
  perm::kv_head_major_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const uint4*>(k), static_cast<const uint4*>(v), n, nkv,
      static_cast<uint4*>(k0), static_cast<uint4*>(v0), rows0, off0, static_cast<uint4*>(k1),
      static_cast<uint4*>(v1), rows1, off1);
  BAM_LAUNCH_CHECK();
  return kOk;
}
