// Bitfield mask kernels: descriptor expansion, validation, block summaries,
// tile classification + per-row workloads, and the CSR/CSC tile lists the
// attention kernels consume.
//
// Semantics follow /root/reference/pkg/src/mmplan/mask.py:
//   build_bitfield    mask.py:71-103   (expand: one descriptor per token)
//   validate          mask.py:53-68    (first failing token, first failing check)
//   materialize       mask.py:106-112  (bam_allowed in common.cuh)
//   _classify_pair    mask.py:132-165  (skip / full / partial)
//   block_workloads   mask.py:168-188  (W_b = non-skip tiles in row b)
// Classification decides most tiles from per-block OR/AND summaries (rules
// proved in SURVEY.md Appendix A.1) and falls back to an exact warp-parallel
// element scan (any/all with early exit) for the rest, so the result equals
// the reference element count for every valid descriptor array.
#include <stdarg.h>
#include <stdio.h>

#include "../../include/bam.h"
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace bam {

// ----------------------------------------------------------------------------- expand
__global__ void expand_kernel(const int64_t* __restrict__ seg_desc,
                              const int64_t* __restrict__ seg_end, int32_t nseg, int64_t T,
                              int64_t* __restrict__ desc) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg - 1;  // first segment whose end > t
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (seg_end[mid] > t) hi = mid; else lo = mid + 1;
    }
    desc[t] = seg_desc[lo];
  }
}

// ----------------------------------------------------------------------------- validate
// err[0] = min over failing tokens of (t << 2 | kind); kind 1 control bits,
// 2 zero, 3 pure modality with popcount != 1.  Host pre-sets err[0] = ~0.
__global__ void validate_kernel(const int64_t* __restrict__ desc, int64_t T,
                                unsigned long long* __restrict__ err) {
  unsigned long long best = ~0ull;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = (unsigned long long)desc[t];
    int kind = 0;
    if (d & (7ull << 61)) kind = 1;
    else if (d == 0) kind = 2;
    else if (!(d & 1ull) && __popcll(d) != 1) kind = 3;
    if (kind) {
      best = min(best, ((unsigned long long)t << 2) | kind);
      break;  // later tokens of this thread are larger
    }
  }
  for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(err, best);
}

// ----------------------------------------------------------------------------- summaries
// One warp per block of `bs` tokens.
__global__ void summarize_kernel(const int64_t* __restrict__ desc, int64_t T, int64_t bs,
                                 int64_t nb, BamBlockSummary* __restrict__ out) {
  const int64_t b = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nb) return;
  const int64_t lo = b * bs, hi = min(lo + bs, T);
  unsigned long long o = 0, a = ~0ull;
  int all_text = 1, any_text = 0;
  for (int64_t t = lo + lane_id(); t < hi; t += 32) {
    const unsigned long long d = (unsigned long long)desc[t];
    o |= d;
    a &= d;
    all_text &= int(d & 1);
    any_text |= int(d & 1);
  }
  for (int s = 16; s; s >>= 1) {
    o |= __shfl_xor_sync(0xffffffffu, o, s);
    a &= __shfl_xor_sync(0xffffffffu, a, s);
    all_text &= __shfl_xor_sync(0xffffffffu, all_text, s);
    any_text |= __shfl_xor_sync(0xffffffffu, any_text, s);
  }
  if (lane_id() == 0) {
    BamBlockSummary s;
    s.or_bits = (int64_t)o;
    s.and_bits = (int64_t)a;
    s.lo = lo;
    s.hi = hi;
    s.flags = (all_text ? BAM_SUMMARY_ALL_TEXT : 0) | (any_text ? 0 : BAM_SUMMARY_NO_TEXT);
    s.pad = 0;
    out[b] = s;
  }
}

// ----------------------------------------------------------------------------- classify
enum : int { kSkip = 0, kFull = 1, kPartial = 2, kUndecided = 3 };

__device__ __forceinline__ int classify_from_summary(const BamBlockSummary& Q,
                                                     const BamBlockSummary& K) {
  const unsigned long long qo = Q.or_bits, qa = Q.and_bits, ko = K.or_bits, ka = K.and_bits;
  if ((qo & ko) == 0) return kSkip;                                  // mask.py:143-144
  const bool q_uniform = qo == qa, k_uniform = ko == ka;
  if (q_uniform && !(qa & 1) && k_uniform && qa == ka) return kFull;  // mask.py:146-153
  if (Q.flags & BAM_SUMMARY_ALL_TEXT) {
    if (K.lo > Q.hi - 1) return kSkip;                  // every key after every query
    if (K.hi - 1 <= Q.lo && (qa & ka) != 0) return kFull;  // all causal, shared bit everywhere
    return kUndecided;
  }
  if ((Q.flags & BAM_SUMMARY_NO_TEXT) && q_uniform) {  // pure-modality query block, value qa
    if (k_uniform) return ka == qa ? kFull : kSkip;
    if ((ko & qa) == 0) return kSkip;                   // no key can equal qa
    return kUndecided;
  }
  return kUndecided;
}

// Exact element scan of one tile by one warp: any / all of materialize().
__device__ int classify_scan_warp(const int64_t* __restrict__ desc, const BamBlockSummary& Q,
                                  const BamBlockSummary& K) {
  bool any = false, all = true;
  for (int64_t q = Q.lo; q < Q.hi; ++q) {
    const long long dq = desc[q];
    for (int64_t k0 = K.lo; k0 < K.hi; k0 += 32) {
      const int64_t k = k0 + lane_id();
      const bool valid = k < K.hi;
      const bool ok = valid && bam_allowed(dq, q, desc[valid ? k : K.lo], k);
      const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
      const uint32_t omask = __ballot_sync(0xffffffffu, ok);
      any |= omask != 0;
      all &= omask == vmask;
      if (any && !all) return kPartial;
    }
  }
  return any ? kFull : kSkip;
}

// One CTA per query block row; 256 threads.  Chunks of 256 key blocks: each
// thread decides its tile from summaries, undecided tiles are scanned by the
// CTA's warps.  Writes classes[row, :] (uint8) and W[row].
__global__ void __launch_bounds__(256) classify_kernel(const int64_t* __restrict__ desc,
                                                       const BamBlockSummary* __restrict__ sum,
                                                       int64_t nb, uint8_t* __restrict__ classes,
                                                       int32_t* __restrict__ W) {
  __shared__ int queue[256];
  __shared__ int qn;
  __shared__ int wcount;
  const int64_t row = blockIdx.x;
  const BamBlockSummary Q = sum[row];
  if (threadIdx.x == 0) wcount = 0;
  int my_nonskip = 0;
  for (int64_t c0 = 0; c0 < nb; c0 += 256) {
    if (threadIdx.x == 0) qn = 0;
    __syncthreads();
    const int64_t c = c0 + threadIdx.x;
    if (c < nb) {
      const int cls = classify_from_summary(Q, sum[c]);
      if (cls == kUndecided) {
        queue[atomicAdd(&qn, 1)] = (int)threadIdx.x;
      } else {
        classes[row * nb + c] = (uint8_t)cls;
        my_nonskip += cls != kSkip;
      }
    }
    __syncthreads();
    const int n = qn;
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5) {
      const int64_t cc = c0 + queue[i];
      const int cls = classify_scan_warp(desc, Q, sum[cc]);
      if (lane_id() == 0) {
        classes[row * nb + cc] = (uint8_t)cls;
        my_nonskip += cls != kSkip;
      }
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) my_nonskip += __shfl_xor_sync(0xffffffffu, my_nonskip, o);
  if (lane_id() == 0) atomicAdd(&wcount, my_nonskip);
  __syncthreads();
  if (threadIdx.x == 0) W[row] = wcount;
}

// ----------------------------------------------------------------------------- tile lists
// Row-compaction of classes restricted to the local query blocks:
//   fwd (CSR): for local q block j (gid q_gid[j]) the non-skip key blocks kb,
//              entry = kb << 2 | class, in increasing kb.
//   bwd (CSC): for key block kb the local q blocks j with a non-skip tile,
//              entry = j << 2 | class, in increasing j.
// count_kernel computes per-list lengths; fill_kernel writes them at the
// offsets (exclusive scan) computed by scan_kernel.
__global__ void list_count_kernel(const uint8_t* __restrict__ classes, int64_t nb,
                                  const int32_t* __restrict__ q_gid, int32_t nq,
                                  int32_t* __restrict__ row_cnt, int32_t* __restrict__ col_cnt) {
  // grid.x = nq rows; each CTA scans its row and adds to column counters
  const int j = blockIdx.x;
  const uint8_t* r = classes + (int64_t)q_gid[j] * nb;
  int cnt = 0;
  for (int64_t kb = threadIdx.x; kb < nb; kb += blockDim.x) {
    if (r[kb]) {
      ++cnt;
      atomicAdd(&col_cnt[kb], 1);
    }
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ int s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  if (lane_id() == 0) atomicAdd(&s, cnt);
  __syncthreads();
  if (threadIdx.x == 0) row_cnt[j] = s;
}

// Ordered compaction of one row (fwd) by one CTA using ballots.  With
// ``owner`` (context parallelism) the row's key blocks owned by ``rank`` come
// first, then the others, each group in increasing kb: the forward works on
// local K/V while the peers' rows are still arriving.
__global__ void list_fill_rows_kernel(const uint8_t* __restrict__ classes, int64_t nb,
                                      const int32_t* __restrict__ q_gid,
                                      const int32_t* __restrict__ row_off,
                                      int32_t* __restrict__ row_tiles,
                                      const int32_t* __restrict__ owner, int32_t rank,
                                      int32_t world) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int j = blockIdx.x;
  const uint8_t* r = classes + (int64_t)q_gid[j] * nb;
  int32_t* out = row_tiles + row_off[j];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  // under CP: the owners in rotation order rank, rank+1, ... (this rank's key
  // blocks first, then the peers in the order the copy engines pull them)
  for (int pass = 0; pass < (owner ? world : 1); ++pass) {
    const int want = (rank + pass) % (world > 0 ? world : 1);
    for (int64_t base = 0; base < nb; base += blockDim.x) {
      const int64_t kb = base + threadIdx.x;
      int cls = kb < nb ? r[kb] : 0;
      if (owner && cls && owner[kb] != want) cls = 0;
      const uint32_t m = __ballot_sync(0xffffffffu, cls != 0);
      if (lane_id() == 0) warp_tot[threadIdx.x >> 5] = __popc(m);
      __syncthreads();
      int before = carry;
      for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) before += warp_tot[w];
      if (cls) out[before + __popc(m & ((1u << lane_id()) - 1))] = (int32_t)((kb << 2) | cls);
      __syncthreads();
      if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += warp_tot[w];
        carry += t;
      }
      __syncthreads();
    }
  }
}

// Ordered compaction of one column (bwd) by one CTA.
__global__ void list_fill_cols_kernel(const uint8_t* __restrict__ classes, int64_t nb,
                                      const int32_t* __restrict__ q_gid, int32_t nq,
                                      const int32_t* __restrict__ col_off,
                                      int32_t* __restrict__ col_tiles) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int64_t kb = blockIdx.x;
  int32_t* out = col_tiles + col_off[kb];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nq; base += blockDim.x) {
    const int j = base + threadIdx.x;
    const int cls = j < nq ? classes[(int64_t)q_gid[j] * nb + kb] : 0;
    const uint32_t m = __ballot_sync(0xffffffffu, cls != 0);
    if (lane_id() == 0) warp_tot[threadIdx.x >> 5] = __popc(m);
    __syncthreads();
    int before = carry;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) before += warp_tot[w];
    if (cls) out[before + __popc(m & ((1u << lane_id()) - 1))] = (int32_t)((j << 2) | cls);
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += warp_tot[w];
      carry += t;
    }
    __syncthreads();
  }
}

// Exact number of allowed (q, k) pairs over all tiles (the algorithmic FLOP
// basis): FULL tiles count |Q||K|, PARTIAL tiles are counted element-wise.
// One CTA per query block row, one warp per tile.
__global__ void __launch_bounds__(256) count_allowed_kernel(const int64_t* __restrict__ desc,
                                                            const BamBlockSummary* __restrict__ sum,
                                                            const uint8_t* __restrict__ classes,
                                                            int64_t nb,
                                                            unsigned long long* __restrict__ out) {
  const int64_t row = blockIdx.x;
  const BamBlockSummary Q = sum[row];
  unsigned long long acc = 0;
  for (int64_t c = threadIdx.x >> 5; c < nb; c += blockDim.x >> 5) {
    const int cls = classes[row * nb + c];
    if (cls == 0) continue;
    const BamBlockSummary K = sum[c];
    if (cls == 1) {
      if (lane_id() == 0) acc += (unsigned long long)(Q.hi - Q.lo) * (K.hi - K.lo);
      continue;
    }
    for (int64_t q = Q.lo; q < Q.hi; ++q) {
      const long long dq = desc[q];
      for (int64_t k0 = K.lo; k0 < K.hi; k0 += 32) {
        const int64_t k = k0 + lane_id();
        const bool ok = k < K.hi && bam_allowed(dq, q, desc[k < K.hi ? k : K.lo], k);
        const uint32_t bits = __ballot_sync(0xffffffffu, ok);
        if (lane_id() == 0) acc += __popc(bits);
      }
    }
  }
  if (lane_id() == 0 && acc) atomicAdd(out, acc);
}

static inline int grid_for(int64_t n, int threads, int cap = 148 * 16) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace bam

using namespace bam;

extern "C" {

int bam_mask_expand(const int64_t* seg_desc, const int64_t* seg_end, int32_t nseg, int64_t T,
                    int64_t* desc, void* stream) {
  BAM_CHECK_ARG(nseg >= 1 && T >= 1, "bam_mask_expand: nseg=%d T=%lld", nseg, (long long)T);
  expand_kernel<<<grid_for(T, 256), 256, 0, (cudaStream_t)stream>>>(seg_desc, seg_end, nseg, T,
                                                                     desc);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_mask_validate(const int64_t* desc, int64_t T, unsigned long long* err, void* stream) {
  BAM_CHECK_ARG(T >= 0, "bam_mask_validate: T=%lld", (long long)T);
  BAM_CUDA_TRY(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), (cudaStream_t)stream));
  if (T == 0) return kOk;
  validate_kernel<<<grid_for(T, 256), 256, 0, (cudaStream_t)stream>>>(desc, T, err);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_block_summarize(const int64_t* desc, int64_t T, int64_t block_size,
                        BamBlockSummary* out, void* stream) {
  BAM_CHECK_ARG(T >= 1 && block_size >= 1, "bam_block_summarize: T=%lld block_size=%lld",
                (long long)T, (long long)block_size);
  const int64_t nb = (T + block_size - 1) / block_size;
  const int warps = 8;
  summarize_kernel<<<(unsigned)((nb + warps - 1) / warps), warps * 32, 0,
                     (cudaStream_t)stream>>>(desc, T, block_size, nb, out);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_classify(const int64_t* desc, const BamBlockSummary* summaries, int64_t nb,
                 uint8_t* classes, int32_t* W, void* stream) {
  BAM_CHECK_ARG(nb >= 1 && nb < (1ll << 31), "bam_classify: nb=%lld", (long long)nb);
  classify_kernel<<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(desc, summaries, nb, classes, W);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_count_allowed(const int64_t* desc, const BamBlockSummary* summaries,
                      const uint8_t* classes, int64_t nb, unsigned long long* out, void* stream) {
  BAM_CHECK_ARG(nb >= 1, "bam_count_allowed: nb=%lld", (long long)nb);
  BAM_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(unsigned long long), (cudaStream_t)stream));
  count_allowed_kernel<<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(desc, summaries, classes,
                                                                       nb, out);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_build_tile_lists(const uint8_t* classes, int64_t nb, const int32_t* q_gid, int32_t nq,
                         int32_t* row_cnt, int32_t* row_off, int32_t* row_tiles, int32_t* col_cnt,
                         int32_t* col_off, int32_t* col_tiles, void* stream) {
  BAM_CHECK_ARG(nb >= 1 && nq >= 1, "bam_build_tile_lists: nb=%lld nq=%d", (long long)nb, nq);
  cudaStream_t s = (cudaStream_t)stream;
  BAM_CUDA_TRY(cudaMemsetAsync(col_cnt, 0, sizeof(int32_t) * nb, s));
  list_count_kernel<<<nq, 256, 0, s>>>(classes, nb, q_gid, nq, row_cnt, col_cnt);
  BAM_LAUNCH_CHECK();
  scan_kernel<<<1, 1024, 0, s>>>(row_cnt, nq, row_off);
  scan_kernel<<<1, 1024, 0, s>>>(col_cnt, nb, col_off);
  BAM_LAUNCH_CHECK();
  if (row_tiles) {
    list_fill_rows_kernel<<<nq, 256, 0, s>>>(classes, nb, q_gid, row_off, row_tiles, nullptr, 0,
                                             1);
    BAM_LAUNCH_CHECK();
  }
  if (col_tiles) {
    list_fill_cols_kernel<<<(unsigned)nb, 256, 0, s>>>(classes, nb, q_gid, nq, col_off, col_tiles);
    BAM_LAUNCH_CHECK();
  }
  return kOk;
}

}  // extern "C"
