/* bam.h -- C ABI of libbam.so, the B200-native (sm_100a) hot path of Cornstarch's
 * token workload-balanced context-parallel attention under bitfield masks.
 *
 * The reference (/root/reference/pkg, Python package `mmplan`) has no FFI; its
 * hot-path interface is the Python API listed below.  Each entry point names
 * the reference function (file:line, relative to /root/reference/pkg) whose
 * work it replaces.  The Python host layer (paper_2503_11367_b200.mask /
 * .balance / .attention) binds these through ctypes with the same names,
 * argument meanings and exceptions as the reference.
 *
 * Conventions (all entry points):
 *   - return 0 on success, otherwise a BamStatus code; bam_last_error() gives
 *     a thread-local message;
 *   - every pointer argument is a caller-allocated DEVICE buffer unless the
 *     comment says "host";
 *   - work is enqueued on `stream` (a cudaStream_t passed as void*) and is
 *     asynchronous; nothing allocates device memory and nothing synchronises
 *     except where the comment says so;
 *   - re-entrant: no global mutable state besides the per-thread error text.
 */
#ifndef BAM_H_
#define BAM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum BamStatus {
  BAM_OK = 0,
  BAM_INVALID_ARGUMENT = 1,
  BAM_CUDA_ERROR = 2,
  BAM_UNSUPPORTED = 3,
  BAM_BUDGET_EXCEEDED = 4
} BamStatus;

#define BAM_SUMMARY_ALL_TEXT 1
#define BAM_SUMMARY_NO_TEXT 2

/* Per-block summary of descriptors. */
typedef struct BamBlockSummary {
  int64_t or_bits;   /* OR of the block's descriptors  */
  int64_t and_bits;  /* AND of the block's descriptors */
  int64_t lo, hi;    /* token range [lo, hi)           */
  int32_t flags;     /* BAM_SUMMARY_* bits              */
  int32_t pad;
} BamBlockSummary;

const char* bam_last_error(void);
int bam_version(void);
/* sizeof of the ABI structs as compiled ("BamAttnFwdParams", "BamAttnBwdParams",
 * "BamPlan", "BamBlockSummary"), -1 for an unknown name: lets bindings check
 * their struct layouts against the library. */
int64_t bam_sizeof(const char* name);

/* ---- bitfield masks (reference src/mmplan/mask.py) ------------------------ */

/* build_bitfield (mask.py:71-103): expand per-segment descriptors to one per
 * token.  seg_desc[i] is segment i's descriptor, seg_end[i] its exclusive end
 * token (prefix sum of counts).  desc[T] out. */
int bam_mask_expand(const int64_t* seg_desc, const int64_t* seg_end, int32_t nseg, int64_t T,
                    int64_t* desc, void* stream);

/* BitfieldMask.validate (mask.py:53-68), token checks in reference order.
 * err (device, 1 x u64) receives min over failing tokens of (t << 2 | kind),
 * kind 1 = reserved control bits, 2 = zero descriptor, 3 = pure modality
 * popcount != 1; all ones when every token is valid.  (The range check and
 * the modality-count check are done by the host before the int64 copy.) */
int bam_mask_validate(const int64_t* desc, int64_t T, unsigned long long* err, void* stream);

/* Per-block OR/AND/text summaries for blocks of `block_size` tokens. */
int bam_block_summarize(const int64_t* desc, int64_t T, int64_t block_size,
                        BamBlockSummary* out, void* stream);

/* block_workloads (mask.py:168-188) / _classify_pair (mask.py:132-165):
 * classes[nb*nb] (0 skip, 1 full, 2 partial; row = query block) and
 * W[nb] = non-skip tiles per query block.  Bit-exact with the reference. */
int bam_classify(const int64_t* desc, const BamBlockSummary* summaries, int64_t nb,
                 uint8_t* classes, int32_t* W, void* stream);

/* Exact count of allowed (q, k) pairs (materialize() true) given classes:
 * the algorithmic-FLOP basis of the attention (4*d*Hq per pair forward,
 * 10*d*Hq backward).  out: device u64. */
int bam_count_allowed(const int64_t* desc, const BamBlockSummary* summaries,
                      const uint8_t* classes, int64_t nb, unsigned long long* out, void* stream);

/* Tile lists for the attention kernels over the local query blocks q_gid[nq]:
 * CSR rows (entry kb << 2 | class, kb ascending) and CSC columns over all nb
 * key blocks (entry j << 2 | class, j = local q index ascending).
 * row_off[nq+1], col_off[nb+1]; row_tiles / col_tiles may be NULL (counts and
 * offsets only).  Counts: row_cnt[nq], col_cnt[nb]. */
int bam_build_tile_lists(const uint8_t* classes, int64_t nb, const int32_t* q_gid, int32_t nq,
                         int32_t* row_cnt, int32_t* row_off, int32_t* row_tiles, int32_t* col_cnt,
                         int32_t* col_off, int32_t* col_tiles, void* stream);

/* ---- distribution (reference src/mmplan/balance.py) ----------------------- */

/* lpt_distribute (balance.py:58-76), also the list scheduler of
 * intra_schedule (balance.py:251-259): items sorted by (-w, index), each to
 * argmin (load, unit).  0 <= w[i] < 2^31.
 * Outputs: owner[n]; flat[n] = items grouped by unit, each unit's items in
 * assignment order, unit g occupying flat[off[g] .. off[g+1]); off[G+1];
 * loads[G].  workspace: >= bam_lpt_workspace_bytes(n) bytes (device). */
int64_t bam_lpt_workspace_bytes(int64_t n);
int bam_lpt_assign(const int32_t* w, int64_t n, int32_t G, int32_t* owner, int32_t* flat,
                   int32_t* off, int64_t* loads, void* workspace, void* stream);

/* zigzag_distribute (balance.py:79-102) and the naive contiguous split
 * (BASELINE.json config 5; not in the reference).  Same outputs as LPT. */
int bam_zigzag_assign(const int32_t* w, int64_t n, int32_t G, int32_t* owner, int32_t* flat,
                      int32_t* off, int64_t* loads, void* stream);
int bam_contiguous_assign(const int32_t* w, int64_t n, int32_t G, int32_t* owner, int32_t* flat,
                          int32_t* off, int64_t* loads, void* stream);

/* split_block pieces for intra_schedule (balance.py:217-220, 237-245): for
 * block b with workload w[b], ceil(w/s) pieces of size s except a final
 * remainder.  piece_off[n+1] (exclusive scan of piece counts) is produced by
 * bam_split_count; bam_split_fill writes piece_size / piece_block /
 * piece_index in (block, index) order. */
int bam_split_count(const int32_t* w, int64_t n, int32_t s, int32_t* piece_cnt,
                    int32_t* piece_off, void* stream);
int bam_split_fill(const int32_t* w, int64_t n, int32_t s, const int32_t* piece_off,
                   int32_t* piece_size, int32_t* piece_block, int32_t* piece_index, void* stream);

/* ilp_optimal (balance.py:124-192): exact branch-and-bound makespan, then
 * the lexicographically smallest assignment.  HOST pointers; synchronous.
 * Returns BAM_BUDGET_EXCEEDED past 14 blocks or 4 GPUs (balance.py:23-24). */
int bam_ilp_optimal(const int64_t* w, int32_t n, int32_t G, int32_t* assignment,
                    int64_t* makespan);

/* ---- attention (absent in the reference) ---------------- */

/* Forward, bitfield-masked, 128x128 tiles, head_dim 128, bf16 in / fp32 acc.
 * Query rows are the local query blocks (q_gid) in local order; keys/values
 * are all nb global blocks stored at block-row k_row[kb] of k/v. */
typedef struct BamAttnFwdParams {
  const void* q;            /* bf16 [nq*128, Hq, 128]            */
  const void* k;            /* bf16 [k_rows*128, Hkv, 128]       */
  const void* v;            /* bf16 [k_rows*128, Hkv, 128]       */
  void* o;                  /* bf16 [nq*128, Hq, 128] out        */
  float* lse;               /* fp32 [Hq, nq*128] out (natural log) */
  const int64_t* desc;      /* int64 [nb*128] descriptors         */
  const int32_t* q_gid;     /* [nq]                               */
  const int32_t* k_row;     /* [nb]                               */
  const int32_t* row_off;   /* [nq+1] CSR from bam_build_tile_lists */
  const int32_t* row_tiles; /* kb << 2 | class                    */
  const int32_t* order;     /* [nq] local q-block processing order (heavy first), or NULL */
  int32_t nq, nb, k_rows, Hq, Hkv;
  float scale;              /* softmax scale, usually 1/sqrt(128) */
  int32_t h_begin, nh;      /* head group: query heads [h_begin, h_begin+nh) of q/o/lse against
                               the Hkv heads of k/v (nh = 0: all Hq heads) */
  /* Optional intra-GPU split-KV schedule (the paper's subblocks, PAPER.md:564-584;
   * ref balance.py:223-265): items[n_items] = {query block j, first tile, end
   * tile, slot}, in LPT order.  slot < 0: the item is the whole row and writes
   * o/lse; slot >= 0: a subblock writing unnormalised fp32 partials
   * part_o[slot][Hq][128][128] and (m log2, l) pairs part_ml[slot][Hq][128][2],
   * merged by bam_attn_fwd_combine.  items == NULL: one whole row per CTA. */
  const int32_t* items;     /* int4 records */
  float* part_o;
  float* part_ml;
  int32_t n_items;
  int32_t kv_flag_heads;    /* head-major kv_ready: one flag per group of this many KV
                               heads, kv_ready[g*Hkv + (h / kv_flag_heads) * kv_flag_heads]
                               (0 or 1: one flag per (rank, KV head)) */
  /* Optional CP overlap (GQA head-pair kernel): kv_ready[g] >= kv_epoch once
   * rank g's K/V rows (block-rows [g*kv_rows_per_rank, (g+1)*kv_rows_per_rank)
   * of k/v) have landed; tiles of other ranks wait for it, this rank's
   * (kv_rank) do not.  kv_ready == NULL: k/v are complete at launch.
   * kv_head_major != 0: k and v are head-major [Hkv, k_rows*128, 128] (the
   * copy-engine gather moves one contiguous chunk per (rank, KV head)), and
   * kv_ready holds one flag per (rank, KV head): kv_ready[g*Hkv + hkv]. */
  const int32_t* kv_ready;
  int32_t kv_epoch, kv_rank, kv_rows_per_rank, kv_head_major;
  /* Optional device-side work counts (bam_plan_build's counts[2]): when set, the
   * host's n_pairs (bam_attn_fwd_qpairs / _2cta) and n_items are upper bounds
   * that size the grid, and CTAs past dev_counts[0] (pairs) or dev_counts[1]
   * (items) exit at once -- the plan needs no host synchronisation. */
  const int32_t* dev_counts;
  /* Optional CTA order of the split-row kernels over whole rows (items == NULL:
   * the GQA head-pair kernel with bam_plan_build's fwd_classes; the MHA
   * query-block-pair kernel of bam_attn_fwd_qpairs with fwd_pair_classes):
   * order_classes[17] split the
   * heavy-first order into geometric work classes [c, c+1) with c = floor(
   * log2(n_max / n)); the grid walks class by class, each class head-pair
   * major, so every head pair's heaviest rows start early and the kernel ends on
   * light rows (the hardware block scheduler then acts as an LPT list scheduler
   * over the whole grid).  NULL: head pairs slowest. */
  const int32_t* order_classes;
} BamAttnFwdParams;
int bam_attn_fwd(const BamAttnFwdParams* p, void* stream);

/* The aggregation kernel of the split schedule: for each combine record
 * {query block j, first slot, n slots, 0} (combine[n_combine]) and each query
 * head of the group, O = sum_p 2^(m_p - M) O_p / sum_p 2^(m_p - M) l_p and
 * LSE = (M + log2 L) ln 2, written to o / lse of p. */
int bam_attn_fwd_combine(const BamAttnFwdParams* p, const int32_t* combine, int32_t n_combine,
                         void* stream);

/* Backward.  dq (bf16) for the local rows; dk/dv for every key row of k/v:
 * fp32 partial gradients (the contributions of the local queries, summed over
 * CP ranks by a reduce-scatter) or, with dkv_bf16, the complete bf16 gradients
 * (one GPU).  delta ([Hq, 2, nq*128] fp32) and dq_acc ([Hq, nq*128, 128] fp32,
 * head-major) are caller workspaces. */
typedef struct BamAttnBwdParams {
  const void* q;
  const void* k;
  const void* v;
  const void* o;
  const void* dout;         /* bf16 [nq*128, Hq, 128]             */
  const float* lse;         /* [Hq, nq*128] from the forward      */
  float* delta;             /* workspace [Hq, 2, nq*128]: lse*log2e, then rowsum(dO*O) */
  float* dq_acc;            /* workspace [Hq, nq*128, 128] fp32 (head-major) */
  void* dq;                 /* bf16 [nq*128, Hq, 128] out         */
  float* dk;                /* fp32 [k_rows*128, Hkv, 128] out    */
  float* dv;                /* fp32 [k_rows*128, Hkv, 128] out    */
  const int64_t* desc;
  const int32_t* q_gid;
  const int32_t* k_row;
  const int32_t* col_off;   /* [nb+1] CSC from bam_build_tile_lists */
  const int32_t* col_tiles; /* j << 2 | class                     */
  const int32_t* order;     /* [nb] key-block processing order, or NULL */
  int32_t nq, nb, k_rows, Hq, Hkv;
  float scale;
  int32_t h_begin, nh;      /* head group as in BamAttnFwdParams; k/v/dk/dv hold Hkv heads */
  /* Optional CTA-pair mode (thread-block clusters of 2 along the key blocks):
   * when pair_shared != NULL, order = slot_kb[n_slots] (-1 = padding slot),
   * col_off / col_tiles are per-slot lists from bam_build_pair_lists (class 0
   * entries allowed), and pairs with pair_shared[p] != 0 multicast each Q/dO
   * tile to both CTAs (each loads one half). */
  const int32_t* pair_shared;
  int32_t n_slots, pad_;
  int32_t kv_head_major;    /* k/v head-major [Hkv, k_rows*128, 128] */
  int32_t dkv_bf16;         /* != 0: dk / dv are bf16 [k_rows*128, Hkv, 128] (complete
                               gradients, one GPU: no partial sums follow), else fp32 */
  /* Optional CP reduce-scatter fused into the epilogue: when dkv_peers != NULL
   * (a DEVICE array of one pointer per rank, each the UVA address of this
   * rank's slot [2][Hkv][dkv_rows_per_owner][128] fp32 in that rank's
   * symmetric workspace), the dK/dV partial rows of key row r go straight to
   * dkv_peers[r / dkv_rows_per_owner] (dK at [0], dV at [1]; over NVLink for
   * other ranks) and dk / dv are not written. */
  float* const* dkv_peers;
  int32_t dkv_rows_per_owner, pad3_;
} BamAttnBwdParams;
int bam_attn_bwd(const BamAttnBwdParams* p, void* stream);
/* The three launches bam_attn_bwd performs, exposed for per-kernel timing:
 * preprocess (delta = rowsum(dO*O), zero dq_acc), main (the tcgen05 kernel),
 * finalize (dq = scale * dq_acc -> bf16). */
int bam_attn_bwd_preprocess(const BamAttnBwdParams* p, void* stream);
int bam_attn_bwd_main(const BamAttnBwdParams* p, void* stream);
int bam_attn_bwd_finalize(const BamAttnBwdParams* p, void* stream);

/* CTA-pair step lists for the backward: pairs (order[2p], order[2p+1]) of key
 * blocks; a pair shares its Q/dO stream when the union of the two CSC columns
 * is at most 9/8 of the longer one (both slots then walk the union, entries
 * j << 2 | class, class 0 = skip for that slot).  n_slots = 2 ceil(nb/2).
 * Pass slot_tiles = NULL to get counts/offsets only. */
int bam_build_pair_lists(const int32_t* col_off, const int32_t* col_tiles, const int32_t* order,
                         int32_t nb, int32_t* slot_kb, int32_t* slot_cnt, int32_t* slot_off,
                         int32_t* slot_tiles, int32_t* pair_shared, void* stream);

/* Forward on CTA pairs (tcgen05 cta_group::2, M = 256): for every shared pair
 * pr = pair_ids[i] of bam_build_pair_lists run over the ROW lists (row_off /
 * row_tiles, order = heavy-first query blocks), the two query blocks
 * slot_q[2 pr], slot_q[2 pr + 1] walk their common union list
 * slot_tiles[slot_off[s] .. slot_off[s + 1]) with the K/V operand traffic
 * split across the two SMs.  Needs an even GQA group (nh / Hkv); whole rows
 * only (p->items unused).  Query blocks of non-shared pairs go through
 * bam_attn_fwd with a whole-row items list. */
int bam_attn_fwd_2cta(const BamAttnFwdParams* p, const int32_t* pair_ids, int32_t n_pairs,
                      const int32_t* slot_q, const int32_t* slot_off, const int32_t* slot_tiles,
                      void* stream);

/* Forward on query-block pairs within one CTA (any head grouping, used for
 * MHA): the shared pairs pair_ids of bam_build_pair_lists over the row lists
 * run as one CTA per (pair, head) -- the two query blocks share every K/V
 * tile and the split-row softmax -- with the union lists slot_tiles; the
 * blocks of non-shared pairs go through bam_attn_fwd with a whole-row items
 * list.  Whole rows only. */
int bam_attn_fwd_qpairs(const BamAttnFwdParams* p, const int32_t* pair_ids, int32_t n_pairs,
                        const int32_t* slot_q, const int32_t* slot_off, const int32_t* slot_tiles,
                        void* stream);

/* ---- per-rank attention planner (no host synchronisation) -------------------
 * Builds, on `stream`, everything the attention kernels need for one rank of a
 * CP plan from the tile classes and the block assignment: the rank-major
 * gathered layout (k_row; this rank's blocks q_gid ascending), the CSR rows
 * (fwd; this rank's key blocks first when world > 1, each group ascending)
 * and CSC columns (bwd), the heavy-first orders, the backward CTA-pair step lists, the
 * forward query-block pairs and the whole-row items of the other blocks
 * (counts[0] shared pairs in fwd_pair_ids, counts[1] items in fwd_rest_items,
 * both on the device; see BamAttnFwdParams.dev_counts).
 * Sizes (int32 elements), with n_tiles = sum of W over this rank's blocks (its
 * LPT load) and P = ceil(nb/2), F = ceil(nq/2): k_row nb, q_gid nq, row_cnt nq,
 * row_off nq+1, row_tiles / col_tiles n_tiles, col_cnt nb,
 * col_off nb+1, fwd_order nq, bwd_order nb, slot_kb / slot_cnt 2P, slot_off
 * 2P+1, slot_tiles 2*n_tiles, pair_shared P, fwd_slot_q / fwd_slot_cnt 2F,
 * fwd_slot_off 2F+1, fwd_slot_tiles 2*n_tiles, fwd_shared F, fwd_pair_ids F,
 * fwd_rest_items 4*nq, counts 2, fwd_classes 17, fwd_pair_w F, fwd_pair_classes
 * 17.  nb <= 16384 (2M tokens).  fwd_classes: the forward's geometric work
 * classes over fwd_order (BamAttnFwdParams.order_classes); fwd_pair_ids lists the
 * shared pairs heavy-first by union length (fwd_pair_w), fwd_pair_classes their
 * classes (the query-block-pair kernels' order_classes). */
typedef struct BamPlan {
  const uint8_t* classes;   /* [nb, nb] from bam_classify */
  const int32_t* owner;     /* [nb] rank of each block (K3); may be NULL when world == 1 */
  int32_t nb, nq, world, rank;
  int32_t max_blocks;       /* the largest per-rank block count (gathered rank stride) */
  int32_t pad_;
  int32_t *k_row, *q_gid, *row_cnt, *row_off, *row_tiles;
  int32_t *col_cnt, *col_off, *col_tiles, *fwd_order, *bwd_order;
  int32_t *slot_kb, *slot_cnt, *slot_off, *slot_tiles, *pair_shared;
  int32_t *fwd_slot_q, *fwd_slot_cnt, *fwd_slot_off, *fwd_slot_tiles, *fwd_shared;
  int32_t *fwd_pair_ids, *fwd_rest_items, *counts, *fwd_classes, *fwd_pair_w,
      *fwd_pair_classes;
} BamPlan;
int bam_plan_build(const BamPlan* plan, void* stream);

/* Stream-ordered 32-bit store (cuStreamWriteValue32, executed without an SM
 * after the stream's prior work, with a memory barrier): the arrival flags of
 * BamAttnFwdParams.kv_ready. */
int bam_stream_write_i32(int32_t* dst, int32_t value, void* stream);
/* Strided copy on the stream's copy engine (cudaMemcpy2DAsync, UVA
 * direction, so a peer's buffer can be the source; no SM involved): height
 * rows of width bytes, dst / src row pitches in bytes.  The CP K/V pulls. */
int bam_copy_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                int64_t height, void* stream);
/* Stream-ordered wait (cuStreamWaitValue32, GEQ): the stream's later work
 * starts once *src >= value (no SM involved). */
int bam_stream_wait_i32_geq(const int32_t* src, int32_t value, void* stream);

/* ---- token permutation ----------------- */
/* The CP runtime permutes tokens into the LPT block layout before attention
 * and back afterwards.  Block-row gather / scatter for up to BAM_PERMUTE_MAX
 * tensors in one launch: a block is block_rows rows of row_bytes[t] bytes.
 *   scatter == 0 (gather):  dst[t] block i      = src[t] block idx[i]
 *   scatter != 0 (scatter): dst[t] block idx[i] = src[t] block i
 * for i < n_blocks.  Pointers and row_bytes must be 16-byte aligned; idx is a
 * device array; src / dst are device pointers (HOST arrays of them). */
#define BAM_PERMUTE_MAX 4
int bam_permute_blocks(const void* const* src, void* const* dst, const int64_t* row_bytes,
                       int32_t n_tensors, const int32_t* idx, int32_t n_blocks,
                       int32_t block_rows, int32_t scatter, void* stream);

/* Sum of n_parts fp32 partials -> bf16, the tail of the dK/dV reduce-scatter
 * (every rank's partials land in this rank's symmetric workspace):
 *   dst_c[row, h, 0:128] = bf16(sum_p src[p*part_stride + c*comp_stride +
 *                                        h*head_stride + row*row_stride + 0:128])
 * for row < n_rows, h < n_heads, c = 0 (dst0) and, when dst1 != NULL, c = 1
 * (dst1).  Outputs are token-major [n_rows, n_heads, 128] bf16; strides are
 * in floats; head dim 128, 16-byte aligned pointers and strides. */
int bam_reduce_partials_bf16(const float* src, int32_t n_parts, int64_t part_stride,
                             int64_t comp_stride, int64_t head_stride, int64_t row_stride,
                             int32_t n_heads, int64_t n_rows, void* dst0, void* dst1,
                             void* stream);

/* Token-major K and V [n, nkv, 128] bf16 -> head-major [nkv, rows_i, 128] at
 * rows [off_i, off_i + n) of destination 0 and, when k1 != NULL, destination 1,
 * in one launch: this rank's shard into its symmetric buffer (pulled by the
 * peers) and into its slot of the gathered K/V the CP forward reads.  Replaces
 * four strided copies on the forward's critical path. */
int bam_kv_head_major(const void* k, const void* v, int64_t n, int32_t nkv, void* k0, void* v0,
                      int64_t rows0, int64_t off0, void* k1, void* v1, int64_t rows1,
                      int64_t off1, void* stream);

/* fp32 -> bf16 conversion (dk/dv partials to the bf16 gradient layout). */
int bam_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream);

/* ---- diagnostics ---------------------------------------------------------- */
/* One-CTA tcgen05/TMA self test: out[3][128][128] fp32 =
 * {A*B^T (SS, both K-major), A*V (TS: A from TMEM, V MN-major),
 *  X^T*V (SS, A MN-major)} for bf16 inputs a, b, v, x of [128,128]. */
int bam_selftest_umma(const void* a, const void* b, const void* v, const void* x, float* out,
                      void* stream);

/* Development aid: install a device buffer ([events][4096] u64 clock64 stamps
 * of one CTA) for -DBAM_TRACE builds; BAM_UNSUPPORTED in normal builds. */
int bam_set_trace_buffer(void* buf);

/* Development aid: install device buffers ([CTAs][4] u64 = {start ns, end ns,
 * SM id, work items} per CTA, %globaltimer) for the forward head-pair kernel and
 * the backward kernel of -DBAM_CTA_CLOCK builds; BAM_UNSUPPORTED otherwise. */
int bam_set_cta_clock_buffer(void* fwd_buf, void* bwd_buf);

#ifdef __cplusplus
}
#endif
#endif /* BAM_H_ */
