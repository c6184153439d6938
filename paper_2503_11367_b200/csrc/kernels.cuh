// Cross-translation-unit kernel declarations used by the planner (plan.cu).
// Launching a __global__ defined in another .cu needs only its declaration
// (the host stub is an ordinary external symbol; no -rdc).
#pragma once
#include <stdint.h>

namespace bam {

constexpr int kSortSmemMax = 16384;  // items sorted in one CTA's shared memory
constexpr int kOrderClasses = 16;    // forward work classes (BamAttnFwdParams.order_classes)

// mask_kernels.cu
__global__ void list_count_kernel(const uint8_t* __restrict__ classes, int64_t nb,
                                  const int32_t* __restrict__ q_gid, int32_t nq,
                                  int32_t* __restrict__ row_cnt, int32_t* __restrict__ col_cnt);
__global__ void list_fill_rows_kernel(const uint8_t* __restrict__ classes, int64_t nb,
                                      const int32_t* __restrict__ q_gid,
                                      const int32_t* __restrict__ row_off,
                                      int32_t* __restrict__ row_tiles,
                                      const int32_t* __restrict__ owner, int32_t rank,
                                      int32_t world);
__global__ void list_fill_cols_kernel(const uint8_t* __restrict__ classes, int64_t nb,
                                      const int32_t* __restrict__ q_gid, int32_t nq,
                                      const int32_t* __restrict__ col_off,
                                      int32_t* __restrict__ col_tiles);

// assign_kernels.cu: one-CTA bitonic sort of (INT32_MAX - w) << 32 | i (heavy
// first, ties by lower index); writes the keys and/or the index order
__global__ void sort_smem_kernel(const int32_t* __restrict__ w, int64_t n, int64_t n_pad,
                                 uint64_t* __restrict__ sorted, int32_t* __restrict__ order);

// attn_fwd.cu: the forward translation unit's half of bam_set_cta_clock_buffer
int fwd_set_cta_clock(void* buf);

namespace bwd {
// attn_bwd.cu: CTA-pair step lists over CSC (or CSR) lists
__global__ void pair_lists_kernel(const int32_t* __restrict__ col_off,
                                  const int32_t* __restrict__ col_tiles,
                                  const int32_t* __restrict__ order, int32_t nb,
                                  int32_t* __restrict__ slot_kb, int32_t* __restrict__ slot_cnt,
                                  const int32_t* __restrict__ slot_off, int32_t* __restrict__ tiles,
                                  int32_t* __restrict__ pair_shared);
}  // namespace bwd

}  // namespace bam
