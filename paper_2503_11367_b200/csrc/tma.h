// Host helpers building TMA tensor maps (cuTensorMapEncodeTiled through the
// runtime's driver entry point, so libbam needs no -lcuda at link time).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace bam {

// Token-major [rows, heads, 128] bf16 tensor -> 3-D map with dims
// (128, heads, rows), box (64, 1, box_rows), SWIZZLE_128B: one TMA load
// brings box_rows rows x 64 columns of one head (128-B swizzled rows).
// head_major: the tensor is [heads, rows, 128] instead; same dims and
// coordinates, only the two outer strides swap, so kernels are unchanged.
int make_tmap_rows_heads_d128(CUtensorMap* map, const void* base, int64_t rows, int heads,
                              int box_rows, bool head_major = false);

}  // namespace bam
