// Per-rank attention planner: everything between the block assignment (K3,
// ref balance.py:58-102) and the attention kernels, on one stream with no
// host synchronisation (bam_plan_build, include/bam.h).
//
//   layout_kernel        owner[nb] -> k_row[nb] (rank-major gathered block-row),
//                        q_gid[nq] (this rank's blocks, ascending)
//   list_* kernels       CSR rows (fwd) / CSC columns (bwd) of non-skip tiles
//   sort_smem_kernel     heavy-first processing orders (-count, index)
//   pair_lists_dense_kernel  CTA-pair step lists (bwd) / query-block pairs (fwd)
//   order_classes_kernel the forward's work classes over the heavy-first order
//                        (query blocks; shared query-block pairs, sorted heavy-first)
//   fwd_pairs_kernel     compaction of the shared forward pairs and the
//                        whole-row items of the others, with device counts
//                        that the forward kernels read (grid = upper bound)
//
// The caller sizes every buffer from (nb, nq, n_tiles): n_tiles = sum of W
// over this rank's blocks = the rank's LPT load, known on the host after the
// one D2H of the assignment's (off, loads) that also gives nq and max_blocks.
#include "../../include/bam.h"
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace bam {

// One CTA per rank g: ordered (ascending block id) compaction of the blocks
// with owner == g.  k_row[b] = g * max_blocks + position; rank's own blocks
// also go to q_gid.
__global__ void __launch_bounds__(1024) layout_kernel(const int32_t* __restrict__ owner,
                                                      int32_t nb, int32_t max_blocks,
                                                      int32_t rank, int32_t* __restrict__ k_row,
                                                      int32_t* __restrict__ q_gid) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int g = blockIdx.x;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += blockDim.x) {
    const int b = base + threadIdx.x;
    const bool mine = b < nb && (owner ? owner[b] : 0) == g;
    const uint32_t m = __ballot_sync(0xffffffffu, mine);
    if (lane_id() == 0) warp_tot[threadIdx.x >> 5] = __popc(m);
    __syncthreads();
    int before = carry;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) before += warp_tot[w];
    if (mine) {
      const int pos = before + __popc(m & ((1u << lane_id()) - 1));
      k_row[b] = g * max_blocks + pos;
      if (g == rank) q_gid[pos] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += warp_tot[w];
      carry += t;
    }
    __syncthreads();
  }
}

// Forward query-block pairs: the shared pairs (ascending pair id) run in the
// split-row kernel, the blocks of the other pairs (pair order, then slot) as
// whole-row items {j, 0, W_j, -1} of the one-head kernel.  counts = {#pairs,
// #items}.  One CTA, ordered ballot compaction of both lists.
__global__ void __launch_bounds__(1024) fwd_pairs_kernel(const int32_t* __restrict__ shared,
                                                         const int32_t* __restrict__ slot_q,
                                                         const int32_t* __restrict__ row_cnt,
                                                         int32_t npairs,
                                                         int32_t* __restrict__ pair_ids,
                                                         int4* __restrict__ items,
                                                         int32_t* __restrict__ counts) {
  __shared__ int wp[32], wi[32];
  __shared__ int cp, ci;
  if (threadIdx.x == 0) cp = ci = 0;
  __syncthreads();
  for (int base = 0; base < npairs; base += blockDim.x) {
    const int pr = base + threadIdx.x;
    const bool valid = pr < npairs;
    const bool sh = valid && shared[pr] != 0;
    const int a = valid ? slot_q[2 * pr] : -1, b = valid ? slot_q[2 * pr + 1] : -1;
    const int n_it = (valid && !sh) ? (a >= 0) + (b >= 0) : 0;
    const uint32_t m = __ballot_sync(0xffffffffu, sh);
    // per-warp inclusive scan of the item counts
    int x = n_it;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane_id() >= (uint32_t)o) x += y;
    }
    if (lane_id() == 31) {
      wp[threadIdx.x >> 5] = __popc(m);
      wi[threadIdx.x >> 5] = x;
    }
    __syncthreads();
    int bp = cp, bi = ci;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) {
      bp += wp[w];
      bi += wi[w];
    }
    if (sh) pair_ids[bp + __popc(m & ((1u << lane_id()) - 1))] = pr;
    int pos = bi + x - n_it;
    if (n_it) {
      if (a >= 0) items[pos++] = make_int4(a, 0, row_cnt[a], -1);
      if (b >= 0) items[pos++] = make_int4(b, 0, row_cnt[b], -1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        cp += wp[w];
        ci += wi[w];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    counts[0] = cp;
    counts[1] = ci;
  }
}

// CTA-pair step lists straight from the dense class matrix: one CTA per pair
// of lists (a, b) = (order[2 pr], order[2 pr + 1]); the same lists as
// bam_build_pair_lists' merge of the CSR/CSC arrays (tests compare them), but
// every element is tested in parallel instead of one thread walking two sorted
// lists.  kCols: lists are key-block columns over this rank's query blocks
// (element e -> classes[q_gid[e]][list]); else query-block rows over the key
// blocks (classes[q_gid[list]][e]).  Pass 1 (tiles == nullptr) counts: a pair
// is shared when its union is at most 9/8 of the longer list; pass 2 fills,
// ascending -- for rows under CP (owner != NULL) grouped by owner in the CSR
// rows' rotation order (this rank's key blocks first, then rank+1, ...), so the
// forward can start before the peers' K/V land.
template <bool kCols>
__global__ void __launch_bounds__(256) pair_lists_dense_kernel(
    const uint8_t* __restrict__ classes, int32_t nb, const int32_t* __restrict__ q_gid,
    int32_t n_elem, const int32_t* __restrict__ order, int32_t n_lists,
    int32_t* __restrict__ slot_kb, int32_t* __restrict__ slot_cnt,
    const int32_t* __restrict__ slot_off, int32_t* __restrict__ tiles,
    int32_t* __restrict__ pair_shared, const int32_t* __restrict__ owner = nullptr,
    int32_t rank = 0, int32_t world = 1) {
  __shared__ int wa[8], wb[8], wu[8];
  __shared__ int carry_a, carry_b;
  const int pr = blockIdx.x;
  const int a = order[2 * pr], b = 2 * pr + 1 < n_lists ? order[2 * pr + 1] : -1;
  const uint8_t* ra = kCols ? classes + a : classes + (int64_t)q_gid[a] * nb;
  const uint8_t* rb = b < 0 ? nullptr : (kCols ? classes + b : classes + (int64_t)q_gid[b] * nb);
  const int w = threadIdx.x >> 5;
  auto cls = [&](const uint8_t* base, int e) -> int {
    if (base == nullptr || e >= n_elem) return 0;
    return kCols ? base[(int64_t)q_gid[e] * nb] : base[e];
  };
  if (tiles == nullptr) {
    int na = 0, nbb = 0, nu = 0;
    for (int e = threadIdx.x; e < n_elem; e += 256) {
      const int ca = cls(ra, e), cb = cls(rb, e);
      na += ca != 0;
      nbb += cb != 0;
      nu += (ca | cb) != 0;
    }
    for (int o = 16; o; o >>= 1) {
      na += __shfl_xor_sync(0xffffffffu, na, o);
      nbb += __shfl_xor_sync(0xffffffffu, nbb, o);
      nu += __shfl_xor_sync(0xffffffffu, nu, o);
    }
    if (lane_id() == 0) {
      wa[w] = na;
      wb[w] = nbb;
      wu[w] = nu;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      na = nbb = nu = 0;
      for (int i = 0; i < 8; ++i) {
        na += wa[i];
        nbb += wb[i];
        nu += wu[i];
      }
      const int mx = na > nbb ? na : nbb;
      const bool sh = b >= 0 && mx > 0 && 8 * nu <= 9 * mx;
      pair_shared[pr] = sh;
      slot_kb[2 * pr] = a;
      slot_kb[2 * pr + 1] = b;
      slot_cnt[2 * pr] = sh ? nu : na;
      slot_cnt[2 * pr + 1] = sh ? nu : nbb;
    }
    return;
  }
  const bool sh = pair_shared[pr] != 0;
  int32_t* oa = tiles + slot_off[2 * pr];
  int32_t* ob = tiles + slot_off[2 * pr + 1];
  if (threadIdx.x == 0) carry_a = carry_b = 0;
  __syncthreads();
  const bool by_owner = !kCols && owner != nullptr;
  for (int pass = 0; pass < (by_owner ? world : 1); ++pass)
  for (int base = 0; base < n_elem; base += 256) {
    const int e = base + threadIdx.x;
    int ca = cls(ra, e), cb = cls(rb, e);
    if (by_owner && e < n_elem && owner[e] != (rank + pass) % world) ca = cb = 0;
    // shared: both slots walk the union (class 0 where a list lacks the element)
    const bool ka = sh ? (ca | cb) != 0 : ca != 0, kb2 = sh ? ka : cb != 0;
    const uint32_t ma = __ballot_sync(0xffffffffu, ka), mb = __ballot_sync(0xffffffffu, kb2);
    if (lane_id() == 0) {
      wa[w] = __popc(ma);
      wb[w] = __popc(mb);
    }
    __syncthreads();
    int pa = carry_a, pb = carry_b;
    for (int i = 0; i < w; ++i) {
      pa += wa[i];
      pb += wb[i];
    }
    const uint32_t below = (1u << lane_id()) - 1;
    if (ka) oa[pa + __popc(ma & below)] = (e << 2) | ca;
    if (kb2) ob[pb + __popc(mb & below)] = (e << 2) | cb;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < 8; ++i) {
        carry_a += wa[i];
        carry_b += wb[i];
      }
    }
    __syncthreads();
  }
}

// Geometric work classes over the heavy-first order (forward CTA order,
// BamAttnFwdParams.order_classes): class(i) = floor(log2(n_max / n_i)) for the
// tile count n_i of the i-th heaviest row, clamped to [0, kOrderClasses - 1]
// (empty rows: the last class).  Classes are contiguous ranges of the order;
// cls[c] = the first position of class >= c, cls[kOrderClasses] = n.
__global__ void __launch_bounds__(1024) order_classes_kernel(const int32_t* __restrict__ cnt,
                                                             const int32_t* __restrict__ order,
                                                             int32_t n, int32_t* __restrict__ cls) {
  const int n_max = cnt[order[0]];
  auto klass = [&](int i) {
    const int c = cnt[order[i]];
    if (c <= 0) return kOrderClasses - 1;
    const int k = 31 - __clz(n_max / c);   // floor(log2(n_max / c)), exact in integers
    return k > kOrderClasses - 1 ? kOrderClasses - 1 : k;
  };
  if (threadIdx.x == 0) {
    cls[0] = 0;
    cls[kOrderClasses] = n;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int prev = i == 0 ? 0 : klass(i - 1), cur = klass(i);
    for (int c = prev + 1; c <= cur; ++c) cls[c] = i;   // classes (prev, cur] start at i
  }
  // classes past the lightest present one are empty: they start at n
  __syncthreads();
  if (threadIdx.x == 0)
    for (int c = klass(n - 1) + 1; c < kOrderClasses; ++c) cls[c] = n;
}

// weight of forward query-block pair pr: its union list length if shared, else 0
__global__ void pair_weights_kernel(const int32_t* __restrict__ shared,
                                    const int32_t* __restrict__ slot_cnt, int32_t npairs,
                                    int32_t* __restrict__ w) {
  const int pr = blockIdx.x * blockDim.x + threadIdx.x;
  if (pr < npairs) w[pr] = shared[pr] ? slot_cnt[2 * pr] : 0;
}

static int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

static int heavy_first(const int32_t* cnt, int32_t n, int32_t* order, cudaStream_t s) {
  const int64_t np = next_pow2(n);
  BAM_CHECK_ARG(np <= kSortSmemMax, "bam_plan_build: %d blocks exceed the one-CTA sort (%d)", n,
                kSortSmemMax);
  const size_t smem = np * sizeof(uint64_t);
  BAM_CUDA_TRY(cudaFuncSetAttribute(sort_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  sort_smem_kernel<<<1, 1024, smem, s>>>(cnt, n, np, nullptr, order);
  BAM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace bam

using namespace bam;

extern "C" int bam_plan_build(const BamPlan* pp, void* stream) {
  BAM_CHECK_ARG(pp != nullptr, "bam_plan_build: null plan");
  const BamPlan& p = *pp;
  BAM_CHECK_ARG(p.classes && p.nb >= 1 && p.nq >= 1 && p.world >= 1 && p.rank >= 0 &&
                    p.rank < p.world && p.max_blocks >= p.nq,
                "bam_plan_build: nb=%d nq=%d world=%d rank=%d max_blocks=%d", p.nb, p.nq, p.world,
                p.rank, p.max_blocks);
  BAM_CHECK_ARG(p.world == 1 || p.owner, "bam_plan_build: world > 1 needs owner[]");
  BAM_CHECK_ARG(p.k_row && p.q_gid && p.row_cnt && p.row_off && p.row_tiles &&
                    p.col_cnt && p.col_off && p.col_tiles && p.fwd_order && p.bwd_order &&
                    p.slot_kb && p.slot_cnt && p.slot_off && p.slot_tiles && p.pair_shared &&
                    p.fwd_slot_q && p.fwd_slot_cnt && p.fwd_slot_off && p.fwd_slot_tiles &&
                    p.fwd_shared && p.fwd_pair_ids && p.fwd_rest_items && p.counts &&
                    p.fwd_classes && p.fwd_pair_w && p.fwd_pair_classes,
                "bam_plan_build: null output buffer");
  BAM_CHECK_ARG(((uintptr_t)p.fwd_rest_items & 15) == 0,
                "bam_plan_build: fwd_rest_items must be 16-byte aligned (int4 records)");
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = p.nb, nq = p.nq;
  layout_kernel<<<p.world, 1024, 0, s>>>(p.world > 1 ? p.owner : nullptr, nb, p.max_blocks, p.rank,
                                         p.k_row, p.q_gid);
  BAM_LAUNCH_CHECK();
  // tile lists: counts, offsets, ascending rows and columns
  BAM_CUDA_TRY(cudaMemsetAsync(p.col_cnt, 0, sizeof(int32_t) * nb, s));
  list_count_kernel<<<nq, 256, 0, s>>>(p.classes, nb, p.q_gid, nq, p.row_cnt, p.col_cnt);
  scan_kernel<<<1, 1024, 0, s>>>(p.row_cnt, nq, p.row_off);
  scan_kernel<<<1, 1024, 0, s>>>(p.col_cnt, nb, p.col_off);
  // rows: under CP this rank's key blocks first, then each peer's in the order
  // rank+1, rank+2, ... that the copy engines pull them (the forward works on local
  // K/V while the peers' rows are still arriving), each group ascending
  list_fill_rows_kernel<<<nq, 256, 0, s>>>(p.classes, nb, p.q_gid, p.row_off, p.row_tiles,
                                           p.world > 1 ? p.owner : nullptr, p.rank, p.world);
  list_fill_cols_kernel<<<nb, 256, 0, s>>>(p.classes, nb, p.q_gid, nq, p.col_off, p.col_tiles);
  BAM_LAUNCH_CHECK();
  // heavy-first orders (LPT's sort key: -count, then index)
  if (int rc = heavy_first(p.col_cnt, nb, p.bwd_order, s)) return rc;
  if (int rc = heavy_first(p.row_cnt, nq, p.fwd_order, s)) return rc;
  order_classes_kernel<<<1, 1024, 0, s>>>(p.row_cnt, p.fwd_order, nq, p.fwd_classes);
  // backward CTA-pair step lists over the columns, forward query-block pairs over the rows
  const int bp = (nb + 1) / 2, fp = (nq + 1) / 2;
  pair_lists_dense_kernel<true><<<bp, 256, 0, s>>>(p.classes, nb, p.q_gid, nq, p.bwd_order, nb,
                                                   p.slot_kb, p.slot_cnt, nullptr, nullptr,
                                                   p.pair_shared);
  pair_lists_dense_kernel<false><<<fp, 256, 0, s>>>(p.classes, nb, p.q_gid, nb, p.fwd_order, nq,
                                                    p.fwd_slot_q, p.fwd_slot_cnt, nullptr,
                                                    nullptr, p.fwd_shared);
  scan_kernel<<<1, 1024, 0, s>>>(p.slot_cnt, 2 * bp, p.slot_off);
  scan_kernel<<<1, 1024, 0, s>>>(p.fwd_slot_cnt, 2 * fp, p.fwd_slot_off);
  pair_lists_dense_kernel<true><<<bp, 256, 0, s>>>(p.classes, nb, p.q_gid, nq, p.bwd_order, nb,
                                                   p.slot_kb, p.slot_cnt, p.slot_off,
                                                   p.slot_tiles, p.pair_shared);
  pair_lists_dense_kernel<false><<<fp, 256, 0, s>>>(p.classes, nb, p.q_gid, nb, p.fwd_order, nq,
                                                    p.fwd_slot_q, p.fwd_slot_cnt, p.fwd_slot_off,
                                                    p.fwd_slot_tiles, p.fwd_shared,
                                                    p.world > 1 ? p.owner : nullptr, p.rank,
                                                    p.world);
  fwd_pairs_kernel<<<1, 1024, 0, s>>>(p.fwd_shared, p.fwd_slot_q, p.row_cnt, fp, p.fwd_pair_ids,
                                      reinterpret_cast<int4*>(p.fwd_rest_items), p.counts);
  // shared pairs heavy-first by union length (the others weigh 0 and sort last, so
  // the first counts[0] entries are the same pairs), and their work classes
  pair_weights_kernel<<<(fp + 255) / 256, 256, 0, s>>>(p.fwd_shared, p.fwd_slot_cnt, fp,
                                                       p.fwd_pair_w);
  BAM_LAUNCH_CHECK();
  if (int rc = heavy_first(p.fwd_pair_w, fp, p.fwd_pair_ids, s)) return rc;
  order_classes_kernel<<<1, 1024, 0, s>>>(p.fwd_pair_w, p.fwd_pair_ids, fp, p.fwd_pair_classes);
  BAM_LAUNCH_CHECK();
  return kOk;
}
