// Bitfield-masked attention backward for sm_100a (tcgen05 + TMEM + TMA).
//
// FlashAttention-style backward parallel over key blocks: one CTA owns one
// 128-key block x one KV head and walks the CSC list of local query blocks
// that see it (non-skip tiles only; PARTIAL tiles re-evaluate the descriptor
// predicate of mask.py:106-112 in registers), for every query head of the
// GQA group.  A step is one 64-row half of a query block for one head
// (j outer, head, half inner, so CTAs running together hit the same dQ
// accumulator lines in L2).  K and V are copied into TMEM once per CTA and
// are the A operands of the TS MMAs:
//   S^T  = K Q^T      (TS, M=128 keys, N=64)  -> TMEM S        P^T = exp2(S^T c - LSE)
//                     (P^T bf16 of queries [32c, 32c+32) over S cols [32c, 32c+16))
//   dP^T = V dO^T     (TS)                    -> TMEM dP       dS^T = P^T (dP^T - D)
//   dV  += P^T dO     (TS: P^T bf16 in S, dO MN-major)         -> TMEM [0,128)
//   dK  += dS^T Q     (SS: dS^T K-major in smem, Q MN-major)   -> TMEM [128,256)
//   dQ^T = K^T dS^T   (SS: K MN-major, dS^T MN-major)          -> TMEM dP
// with S / dP single-buffered (TMEM holds dV, dK, K, V, S, dP = 512 columns):
// S(s+1) is issued right after dV(s) so it runs while the compute warps turn
// dP(s) into dS(s), and P^T(s) reaches dV(s) in two chunks.  dQ^T puts d on
// the TMEM lanes; the dQ warps stage each 64-query dQ^T tile (32 KB fp32) in
// shared memory (two stages: the freed V region and one more, so the drain
// never waits for the previous bulk reduce) and one TMA bulk reduce-add adds
// it into the head-major accumulator.  Q/dO half tiles (+ the (lse, D) pairs)
// stream through a 3-stage TMA ring.
// Warp roles (448 threads, 1 CTA / SM):
//   warps 0-7 compute (two warpgroups, 32 query columns each; thread r = key
//   row r), warps 8-11 dQ epilogue (thread r = head-dim column r), warp 12
//   MMA issuer + TMEM alloc, warp 13 TMA producer (Q/dO half tiles + LSE/D).
// CTA pairs (clusters of 2 along the slot axis) whose key blocks share one
// step list multicast each Q/dO stage to both CTAs.
// Bounds (profiles/r01/bwd_variants.md, profiles/r02/): the fp32
// dQ reduce-adds into L2 (357 GB per config-4 launch), the shared-memory port
// (128 B/clk: MMA operands, TMA writes, dS^T and dQ staging) and the
// single-buffered S/dP chain.  Alternatives measured slower and removed: the
// all-SS double-buffered kernel (975-985 vs 1075 TFLOP/s), dQ by red.global
// from registers (931-956 / 891-896), the CTA-pair DSMEM dQ sum (469-523), lse/D
// by warp shuffles instead of broadcast loads (-2%).  BAM_TRACE builds record
// per-step events for tools/trace_bwd.py.
#include "../../include/bam.h"
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"
#include "tma.h"

namespace bam {
namespace bwd {

constexpr int kThreads = 448;
// warp roles
constexpr uint32_t kWarpDQ = 8, kWarpMMA = 12, kWarpTMA = 13;
constexpr int kStages = 3;       // Q/dO half-tile ring (the dQ staging takes the 4th slot)
// P^T(s) reaches the dV MMAs in two chunks of 16 queries per warpgroup
constexpr int kBwdPChunks = 2;
// lse and D reach P = 2^(c S - lse) and dS = P (dP - D) through the tensor core:
// one extra K = 16 MMA per S^T / dP^T adds -lse / c and -D (as bf16 hi/mid/lo
// splits, exact to ~2^-24) from a per-step bias tile [64 queries x 16] times a
// constant ones tile [128 keys x 16], so the compute warps need no per-query
// values -- the broadcast loads that fed them were ~12% of the shared-memory
// port traffic, the kernel's binding resource (measured +1.3%,
// profiles/r02/ab_bwd_bias.txt)
#ifndef BAM_DQ_SLEEP_NS
#define BAM_DQ_SLEEP_NS 64
#endif
// Grid order: slot-major (key blocks fastest, one KV head after the other): the
// ~148 CTAs resident together are key blocks of ONE KV head, so their dQ
// reductions land in that head group's quarter-GiB slice of dq_acc, whose
// active window stays in L2 (DRAM traffic per config-4 launch 94 -> 14.8 GB).
constexpr uint32_t kTileBytes = 128 * 128 * 2;   // K, V: 128 rows x 128 cols (two 64-col boxes)
constexpr uint32_t kHalfBytes = 64 * 128 * 2;    // Q, dO half tile: 64 rows x 128 cols
constexpr uint32_t kDsBytes = 128 * 64 * 2;      // dS^T: 128 key rows x 64 query cols
// TMEM columns: dV, dK accumulators; K, V as bf16 pairs; single S and dP/dQ^T buffers
constexpr uint32_t kColDV = 0, kColDK = 128, kColK = 256, kColV = 320, kColS = 384,
                   kColDP = 448;

struct Stage {
  alignas(1024) uint8_t q[kHalfBytes];
  alignas(1024) uint8_t dout[kHalfBytes];
  // bias B operands [64 queries x 16] bf16, SWIZZLE_NONE K-major core matrices
  // ([k chunk][row group][8 rows][8]): [0] -lse/c, [1] -D as (hi, mid, lo, 0...)
  alignas(1024) __nv_bfloat16 bias[2][64 * 16];
};

struct Smem {
  alignas(1024) uint8_t k[kTileBytes];
  alignas(1024) uint8_t v[kTileBytes];
  alignas(1024) uint8_t ds[kDsBytes];
  Stage st[kStages];
  alignas(128) float dq_stage[64 * 128];  // dQ tile [64 queries][128 d] fp32 for the bulk reduce
  alignas(128) __nv_bfloat16 ones[128 * 16];  // A operand [128 keys x 16]: 1 in k = 0, 1, 2
  uint64_t bar_kv, bar_full[kStages], bar_empty[kStages];
  uint64_t bar_s_full, bar_p_ready[kBwdPChunks], bar_mma_done, bar_dq_full, bar_dq_empty;
  uint64_t bar_kvt, bar_dp_full, bar_ds_ready;
  uint32_t tmem_base;
};

// Shared-memory matrix descriptor, no swizzle (K-major core matrices of 8 rows x
// 16 B): lbo = byte stride between k-adjacent core matrices, sbo = between
// row-adjacent ones (tools/umma_k16_test.cu checks the convention).
__device__ __forceinline__ uint64_t sdesc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// bf16 (hi, mid, lo) with hi + mid + lo == x to ~2^-24 relative
__device__ __forceinline__ uint4 bias_chunk(float x) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(hi);
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
  return make_uint4(uint32_t(__bfloat16_as_ushort(hi)) | (uint32_t(__bfloat16_as_ushort(mid)) << 16),
                    uint32_t(__bfloat16_as_ushort(lo)), 0u, 0u);
}

// P = 2^(S c - lse) for a pair of queries (packed FMUL2, exponentials on MUFU:
// the backward's MUFU is ~25% busy, a polynomial share measured slower), masked by
// the PARTIAL-tile allow bits.  The S columns already hold S - lse / c (bias MMA).
template <bool kMasked>
__device__ __forceinline__ float2 p_pair(uint32_t s0, uint32_t s1, float sc, int i2,
                                         uint32_t allow) {
  const float2 x = fmul2(make_float2(__uint_as_float(s0), __uint_as_float(s1)),
                         make_float2(sc, sc));
  float2 p = make_float2(ex2(x.x), ex2(x.y));
  if constexpr (kMasked) {
    p.x = (allow >> (2 * i2)) & 1 ? p.x : 0.f;
    p.y = (allow >> (2 * i2 + 1)) & 1 ? p.y : 0.f;
  }
  return p;
}
template <bool B>
struct BoolC {
  static constexpr bool value = B;
};
// dS = P (dP - D) for the same pair (the dP columns hold dP - D: bias MMA)
__device__ __forceinline__ float2 ds_pair(float2 p, uint32_t dp0, uint32_t dp1) {
  return fmul2(p, make_float2(__uint_as_float(dp0), __uint_as_float(dp1)));
}

struct StepInfo {
  int h, jq, cls, half;
};

// Step s = (column entry s / (2 grp), head (s / 2) % grp, half s % 2), walked
// incrementally (no integer division in the loops).
struct StepIter {
  const int32_t* col;
  int per_j, h0, ci = 0, r = 0;
  __device__ __forceinline__ StepIter(const int32_t* c, int grp, int hkv, int h_begin)
      : col(c), per_j(2 * grp), h0(h_begin + hkv * grp) {}
  __device__ __forceinline__ StepInfo get() const {
    const int e = col[ci];
    return {h0 + (r >> 1), e >> 2, e & 3, r & 1};
  }
  __device__ __forceinline__ void next() {
    if (++r == per_j) {
      r = 0;
      ++ci;
    }
  }
};

__global__ void __maxnreg__(128)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const BamAttnBwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  BAM_CTA_CLOCK_BEGIN();
  const uint32_t warp = warp_id(), lane = lane_id();
  const int hkv = blockIdx.y;
  // CTA-pair mode: clusters of 2 along x (slots); slot lists; shared pairs multicast Q/dO
  const bool cluster_mode = p.pair_shared != nullptr;
  const int slot = blockIdx.x;
  const int kb = p.order ? p.order[slot] : slot;   // -1: padding slot (cluster mode)
  const int li = cluster_mode ? slot : kb;         // step-list index
  const uint32_t crank = cluster_mode ? cluster_ctarank() : 0;
  const bool shared = cluster_mode && p.pair_shared[slot >> 1] != 0;
  const int grp = (p.nh > 0 ? p.nh : p.Hq) / p.Hkv;
  int ncol = 0, krow0 = 0;
  const int32_t* col = p.col_tiles;
  if (kb >= 0) {
    const int c0 = p.col_off[li];
    ncol = p.col_off[li + 1] - c0;
    col = p.col_tiles + c0;
    krow0 = p.k_row[kb] * 128;
  }
  const int nsteps = ncol * grp * 2;
  const int64_t Tq = (int64_t)p.nq * 128;
  const bool trace_cta = blockIdx.x == 0 && blockIdx.y == 0;
  (void)trace_cta;
#ifdef BAM_TRACE
  unsigned long long* const bam_trace_ptr = trace_cta ? g_bam_trace : nullptr;
#endif

  if (threadIdx.x == 0) {
    if ((smem_u32(smem_raw) & 1023) != 0) __trap();  // SWIZZLE_128B needs 1024-B alignment
    mbar_init(&sm.bar_kv, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.bar_full[i], 2);  // TMA bytes + the bias tile's arrival
      mbar_init(&sm.bar_empty[i], shared ? 2 : 1);  // shared: both CTAs' MMAs release a stage
    }
    mbar_init(&sm.bar_s_full, 1);
    for (int j = 0; j < kBwdPChunks; ++j) mbar_init(&sm.bar_p_ready[j], 256);
    mbar_init(&sm.bar_mma_done, 1);
    mbar_init(&sm.bar_dq_full, 1);
    mbar_init(&sm.bar_dq_empty, 128);
    mbar_init(&sm.bar_kvt, 256);
    mbar_init(&sm.bar_dp_full, 1);
    mbar_init(&sm.bar_ds_ready, 256);
    fence_mbar_init();
  }
  if (warp == kWarpMMA) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  if (cluster_mode) cluster_sync_all();  // peer barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == kWarpTMA) {
    // ------------------------------------------------------------ TMA producer (whole warp)
    const uint32_t leader = elect_one();
    if (nsteps > 0) {
      if (leader) {
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        prefetch_tmap(&tm_v);
        prefetch_tmap(&tm_do);
      }
      mbar_expect_tx_w(&sm.bar_kv, 2 * kTileBytes, leader);
      tma_load_3d_w(&tm_k, &sm.bar_kv, sm.k, 0, hkv, krow0, leader);
      tma_load_3d_w(&tm_k, &sm.bar_kv, sm.k + kTileBytes / 2, 64, hkv, krow0, leader);
      tma_load_3d_w(&tm_v, &sm.bar_kv, sm.v, 0, hkv, krow0, leader);
      tma_load_3d_w(&tm_v, &sm.bar_kv, sm.v + kTileBytes / 2, 64, hkv, krow0, leader);
      StepIter it(col, grp, hkv, p.h_begin);
      for (int s = 0; s < nsteps; ++s) {
        const int st = s % kStages;
        const StepInfo si = it.get();
        it.next();
        const int row0 = si.jq * 128 + si.half * 64;
        if (s >= kStages) mbar_wait_sleep(&sm.bar_empty[st], ((s / kStages) - 1) & 1);
        BAM_TRACE_EV(trace_cta && leader, 10, s);
        Stage& S = sm.st[st];
        mbar_expect_tx_w(&sm.bar_full[st], 2 * kHalfBytes, leader);
        if (shared) {  // this CTA loads column box `crank` of Q and dO for both CTAs
          const uint32_t off = crank * (kHalfBytes / 2);
          tma_load_3d_mc_w(&tm_q, &sm.bar_full[st], S.q + off, crank * 64, si.h, row0, 0x3,
                           leader);
          tma_load_3d_mc_w(&tm_do, &sm.bar_full[st], S.dout + off, crank * 64, si.h, row0, 0x3,
                           leader);
        } else {
          tma_load_3d_w(&tm_q, &sm.bar_full[st], S.q, 0, si.h, row0, leader);
          tma_load_3d_w(&tm_q, &sm.bar_full[st], S.q + kHalfBytes / 2, 64, si.h, row0, leader);
          tma_load_3d_w(&tm_do, &sm.bar_full[st], S.dout, 0, si.h, row0, leader);
          tma_load_3d_w(&tm_do, &sm.bar_full[st], S.dout + kHalfBytes / 2, 64, si.h, row0,
                        leader);
        }
        {  // bias tiles: lane l writes queries 2l, 2l+1 (k chunk 0; chunk 1 stays zero)
          const float* ld = p.delta + (int64_t)si.h * 2 * Tq + row0;
          const float2 lse2 = *reinterpret_cast<const float2*>(ld + 2 * lane);
          const float2 dd = *reinterpret_cast<const float2*>(ld + Tq + 2 * lane);
          const float inv_sc = 1.f / (p.scale * 1.4426950408889634f);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int q = 2 * lane + u;
            const int off = ((q >> 3) * 8 + (q & 7)) * 8;   // element of (q, k = 0)
            *reinterpret_cast<uint4*>(S.bias[0] + off) = bias_chunk(-(u ? lse2.y : lse2.x) * inv_sc);
            *reinterpret_cast<uint4*>(S.bias[1] + off) = bias_chunk(-(u ? dd.y : dd.x));
          }
          fence_async_smem();   // generic-proxy stores -> the tensor core's reads
          __syncwarp();
          if (leader) mbar_arrive(&sm.bar_full[st]);
        }
      }
    }
  } else if (warp == kWarpMMA) {
    // ------------------------------------------------------------ MMA issuer (whole warp)
    // Descriptors are built once; per MMA only the 14-bit start-address field
    // advances (adding offset >> 4 to the 64-bit descriptor cannot carry out).
    const uint32_t leader = elect_one();
    if (nsteps > 0) {
      const uint32_t id_s = idesc_bf16(128, 64, 0, 0);    // S^T, dP^T: K-major x K-major
      const uint32_t id_kv = idesc_bf16(128, 128, 0, 1);  // dV, dK: (TMEM|K-major) x MN-major
      const uint32_t id_q = idesc_bf16(128, 64, 1, 1);    // dQ^T: MN-major x MN-major
      const uint64_t dk_kmn = sdesc_sw128(smem_u32(sm.k), kTileBytes / 2, 1024);  // K, MN-major
      const uint64_t d_q0 = sdesc_sw128(smem_u32(sm.st[0].q), 16, 1024);         // K-major
      const uint64_t d_q0mn = sdesc_sw128(smem_u32(sm.st[0].q), kHalfBytes / 2, 1024);
      const uint64_t d_ds0 = sdesc_sw128(smem_u32(sm.ds), 16, 1024);
      constexpr uint32_t kStage16 = sizeof(Stage) >> 4, kDo16 = kHalfBytes >> 4;
      // ones [128 x 16]: k-chunk stride 16 row groups x 128 B; bias [64 x 16]: 8 x 128 B
      const uint64_t d_ones = sdesc_noswz(smem_u32(sm.ones), 2048, 128);
      const uint64_t d_bias0 = sdesc_noswz(smem_u32(sm.st[0].bias[0]), 1024, 128);
      constexpr uint32_t kBias16 = (64 * 16 * 2) >> 4;
      const uint32_t tK = tmem + kColK, tV = tmem + kColV, tS = tmem + kColS, tDP = tmem + kColDP;
      mbar_wait(&sm.bar_kvt, 0);  // K / V rows stored into TMEM by the compute warps
      // S^T(s) = K Q^T (A = K from TMEM) -> S; S(s) overwrites P^T(s-1), the A operand of
      // dV(s-1): issued earlier by this thread, and tcgen05.mma ops execute in issue order.
      auto issue_s = [&](int s) {
        const int st = s % kStages;
        mbar_wait(&sm.bar_full[st], (s / kStages) & 1);
        BAM_TRACE_EV(trace_cta && leader, 11, s);
        tc_fence_after();
        const uint64_t dq = d_q0 + st * kStage16;
        mma_ss_w(tS, d_ones, d_bias0 + st * kStage16, id_s, 0, leader);   // S := -lse / c
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t kq = ((kk >> 2) * (kHalfBytes / 2) + (kk & 3) * 32) >> 4;
          mma_ts_w(tS, tK + 8 * kk, dq + kq, id_s, 1, leader);   // accumulates onto the bias
        }
        tc_commit_w(&sm.bar_s_full, leader);
      };
      // dP^T(s) = V dO^T (A = V from TMEM) -> dP, once dQ^T(s-1) has been drained from it
      auto issue_dp = [&](int s) {
        const int st = s % kStages;
        if (s > 0) mbar_wait(&sm.bar_dq_empty, (s - 1) & 1);
        BAM_TRACE_EV(trace_cta && leader, 1, s);
        tc_fence_after();
        const uint64_t ddo = d_q0 + st * kStage16 + kDo16;
        mma_ss_w(tDP, d_ones, d_bias0 + st * kStage16 + kBias16, id_s, 0, leader);   // dP := -D
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t kq = ((kk >> 2) * (kHalfBytes / 2) + (kk & 3) * 32) >> 4;
          mma_ts_w(tDP, tV + 8 * kk, ddo + kq, id_s, 1, leader);
        }
        tc_commit_w(&sm.bar_dp_full, leader);
        BAM_TRACE_EV(trace_cta && leader, 12, s);
      };
      issue_s(0);
      issue_dp(0);
      for (int s = 0; s < nsteps; ++s) {
        const int st = s % kStages;
        const uint32_t ph = s & 1;
        const uint64_t dqmn = d_q0mn + st * kStage16, ddomn = dqmn + kDo16;
        // dV += P^T dO  (A = P^T bf16 in the S columns).  P^T(s) arrives in two chunks
        // of 16 queries per warpgroup (bar_p_ready[j]): chunk j feeds the 16-query
        // steps kk = j (warpgroup 0) and 2 + j (warpgroup 1), so half of dV(s) runs
        // while the compute warps finish the other half of P
#pragma unroll
        for (int j = 0; j < kBwdPChunks; ++j) {
          mbar_wait(&sm.bar_p_ready[j], ph);
          BAM_TRACE_EV(trace_cta && leader, 2, s);
          tc_fence_after();
#pragma unroll
          for (int u = 0; u < 4 / kBwdPChunks; ++u) {
            const int kk = 2 * u + j;
            mma_ts_w(tmem + kColDV, tS + (kk >> 1) * 32 + (kk & 1) * 8, ddomn + kk * 128, id_kv,
                     (s > 0 || j > 0 || u > 0), leader);
          }
        }
        if (s + 1 < nsteps) issue_s(s + 1);  // overlaps the compute warps' dS(s)
        mbar_wait(&sm.bar_ds_ready, ph);
        BAM_TRACE_EV(trace_cta && leader, 14, s);
        tc_fence_after();
        // dQ^T first and committed on its own: the dQ warps drain it (and dP(s+1),
        // which reuses its columns, can start) while dK(s) runs
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dQ^T = K^T dS^T -> the dP columns
          mma_ss_w(tDP, dk_kmn + kk * 128, d_ds0 + kk * 128, id_q, kk > 0, leader);
        tc_commit_w(&sm.bar_dq_full, leader);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dK += dS^T Q  (A = dS^T K-major in shared memory)
          mma_ss_w(tmem + kColDK, d_ds0 + 2 * kk, dqmn + kk * 128, id_kv, (s > 0 || kk > 0),
                   leader);
        if (shared)
          tc_commit_mc_w(&sm.bar_empty[st], 0x3, leader);
        else
          tc_commit_w(&sm.bar_empty[st], leader);
        BAM_TRACE_EV(trace_cta && leader, 3, s);
        if (s + 1 < nsteps) issue_dp(s + 1);
      }
      tc_commit_w(&sm.bar_mma_done, leader);
    }
  } else if (warp < kWarpDQ) {
    // ------------------------------------------------------------ compute warps 0-7
    // Two warpgroups split the 64 queries of a step: warpgroup c takes query
    // columns [32c, 32c+32); thread r = key row r = TMEM lane r in both.
    const int c = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    const long long kg = (long long)kb * 128 + r;
    const long long dk = p.desc[kg];
    const float scale_log2 = p.scale * 1.4426950408889634f;
    StepIter it(col, grp, hkv, p.h_begin);
    if (nsteps > 0) {
      // Row r of K (warpgroup 0) / V (warpgroup 1) from the swizzled tile into
      // TMEM lane r as bf16 pairs: column j = head-dim elements 2j, 2j+1.
      mbar_wait_sleep(&sm.bar_kv, 0);
      const uint8_t* src = (c == 0 ? sm.k : sm.v) + r * 128;
#pragma unroll
      for (int hb = 0; hb < 2; ++hb) {
        uint32_t w[32];
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const uint4 x = *reinterpret_cast<const uint4*>(src + hb * (kTileBytes / 2) +
                                                          ((ch ^ (r & 7)) << 4));
          w[4 * ch] = x.x;
          w[4 * ch + 1] = x.y;
          w[4 * ch + 2] = x.z;
          w[4 * ch + 3] = x.w;
        }
        BAM_TMEM_ST32(tmem + lane_base + (c == 0 ? kColK : kColV) + 32 * hb, w);
      }
      tmem_wait_st();
      {  // ones tile (thread t: row t % 128, k chunk t / 128) and the bias tiles' zero chunk
        const int t = c * 128 + r;
        const uint32_t one = 0x3F80u | (0x3F80u << 16);   // bf16 1.0 pairs
        const uint4 v = t < 128 ? make_uint4(one, 0x3F80u, 0u, 0u) : make_uint4(0u, 0u, 0u, 0u);
        const int rr = t & 127;
        *reinterpret_cast<uint4*>(sm.ones + ((t >> 7) * 16 * 8 + (rr >> 3) * 8 + (rr & 7)) * 8) = v;
        for (int i = t; i < kStages * 2 * 64; i += 256) {   // (stage, tile, query), k chunk 1
          const int q = i & 63, tile = (i >> 6) & 1, stg = i >> 7;
          *reinterpret_cast<uint4*>(sm.st[stg].bias[tile] + (64 + (q >> 3) * 8 + (q & 7)) * 8) =
              make_uint4(0u, 0u, 0u, 0u);
        }
        fence_async_smem();
      }
      tc_fence_before();
      mbar_arrive(&sm.bar_kvt);
    }
    for (int s = 0; s < nsteps; ++s) {
      const uint32_t ph = s & 1;
      const StepInfo si = it.get();
      it.next();
      const uint32_t tS = tmem + kColS + lane_base, tdP = tmem + kColDP + lane_base;
      const uint32_t ds_row = smem_u32(sm.ds) + r * 128;
      mbar_wait_sleep<BAM_COMPUTE_SLEEP_NS>(&sm.bar_s_full, ph);
      BAM_TRACE_EV(trace_cta && threadIdx.x == 0, 4, s);
      tc_fence_after();
      uint32_t sr[32];
      BAM_TMEM_LD32(tS + c * 32, sr);
      uint32_t allow = si.cls ? 0xFFFFFFFFu : 0u;
      if (si.cls == 2) {
        const long long qg0 = (long long)p.q_gid[si.jq] * 128 + si.half * 64 + c * 32;
        allow = 0;
#pragma unroll 1
        for (int i = 0; i < 32; ++i)
          allow |= uint32_t(bam_allowed(__ldg(p.desc + qg0 + i), qg0 + i, dk, kg)) << i;
      }
      tmem_wait_ld();
      // P^T over this warpgroup's own S columns, released in kBwdPChunks chunks
      // (FULL tiles -- nearly all of them -- skip the per-element allow test)
      auto p_chunks = [&](auto masked) {
#pragma unroll
        for (int j = 0; j < kBwdPChunks; ++j) {
          constexpr int kPer = 16 / kBwdPChunks;
          uint32_t pk[kPer];
#pragma unroll
          for (int u = 0; u < kPer; ++u) {
            const int i2 = j * kPer + u;
            const float2 pp = p_pair<decltype(masked)::value>(sr[2 * i2], sr[2 * i2 + 1],
                                                              scale_log2, i2, allow);
            sr[2 * i2] = __float_as_uint(pp.x);
            sr[2 * i2 + 1] = __float_as_uint(pp.y);
            pk[u] = pack_bf16(pp.x, pp.y);
          }
          if constexpr (kPer == 16)
            BAM_TMEM_ST16(tS + c * 32, pk);
          else
            BAM_TMEM_ST8(tS + c * 32 + j * 8, pk);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&sm.bar_p_ready[j]);
        }
      };
      if (si.cls == 1)
        p_chunks(BoolC<false>{});
      else
        p_chunks(BoolC<true>{});
      BAM_TRACE_EV(trace_cta && threadIdx.x == 0, 5, s);
      mbar_wait_sleep<BAM_COMPUTE_SLEEP_NS>(&sm.bar_dp_full, ph);
      BAM_TRACE_EV(trace_cta && threadIdx.x == 0, 6, s);
      tc_fence_after();
      uint32_t dr[32], dsk[16];
      BAM_TMEM_LD32(tdP + c * 32, dr);
      tmem_wait_ld();
      BAM_TRACE_EV(trace_cta && threadIdx.x == 0, 16, s);
#pragma unroll
      for (int i2 = 0; i2 < 16; ++i2) {
        const float2 ds = ds_pair(make_float2(__uint_as_float(sr[2 * i2]),
                                              __uint_as_float(sr[2 * i2 + 1])),
                                  dr[2 * i2], dr[2 * i2 + 1]);
        dsk[i2] = pack_bf16(ds.x, ds.y);
      }
      // dS^T row r, query columns 32c .. 32c+31 (the A operand of dK, B of dQ^T)
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const uint32_t chunk = (uint32_t)(c * 4 + q4) ^ (uint32_t)(r & 7);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ds_row + chunk * 16),
                     "r"(dsk[q4 * 4]), "r"(dsk[q4 * 4 + 1]), "r"(dsk[q4 * 4 + 2]),
                     "r"(dsk[q4 * 4 + 3])
                     : "memory");
      }
      BAM_TRACE_EV(trace_cta && threadIdx.x == 0, 17, s);
      fence_async_smem();
      BAM_TRACE_EV(trace_cta && threadIdx.x == 0, 18, s);
      tc_fence_before();
      BAM_TRACE_EV(trace_cta && threadIdx.x == 0, 7, s);
      mbar_arrive(&sm.bar_ds_ready);
    }
    // epilogue: warpgroup 0 writes dV, warpgroup 1 writes dK (scaled), fp32 rows
    if (kb < 0) goto done;  // padding slot of the last cluster
    {
    const int64_t row = (int64_t)krow0 + r;
    float* dst;
    if (p.dkv_peers != nullptr) {  // fused reduce-scatter: the owner's workspace slot
      const int owner = krow0 / p.dkv_rows_per_owner;
      const int64_t lr = row - (int64_t)owner * p.dkv_rows_per_owner;
      dst = p.dkv_peers[owner] +
            (((int64_t)(c == 0 ? 1 : 0) * p.Hkv + hkv) * p.dkv_rows_per_owner + lr) * 128;
    } else {
      dst = (c == 0 ? p.dv : p.dk) + (row * p.Hkv + hkv) * 128;
    }
    const float mul = c == 0 ? 1.f : p.scale;
    if (nsteps > 0) {
      mbar_wait_sleep(&sm.bar_mma_done, 0);
      tc_fence_after();
      if (p.dkv_peers != nullptr) {
        // fused reduce-scatter: rows staged in the (now idle) Q/dO stages, 272-B
        // pitch (conflict-free 16-B stores), then one 256-B bulk copy per half
        // row; the CTA waits only for the shared-memory reads, not for the
        // NVLink writes to land
        static_assert(kStages * sizeof(Stage) >= 2 * 128 * 272, "staging space");
        const uint32_t s_row = smem_u32(reinterpret_cast<uint8_t*>(&sm.st[0])) +
                               (uint32_t)(c * 128 * 272 + r * 272);
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          if (hh) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#pragma unroll
          for (int q2 = 0; q2 < 2; ++q2) {
            uint32_t a[32];
            BAM_TMEM_LD32(tmem + lane_base + (c == 0 ? kColDV : kColDK) + (hh * 2 + q2) * 32, a);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i)
              asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(s_row + q2 * 128 + i * 16),
                           "f"(__uint_as_float(a[4 * i]) * mul),
                           "f"(__uint_as_float(a[4 * i + 1]) * mul),
                           "f"(__uint_as_float(a[4 * i + 2]) * mul),
                           "f"(__uint_as_float(a[4 * i + 3]) * mul)
                           : "memory");
          }
          fence_async_smem();
          asm volatile(
              "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;\n\t"
              "cp.async.bulk.commit_group;" ::"l"(dst + hh * 64),
              "r"(s_row)
              : "memory");
        }
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      } else if (p.dkv_bf16) {
        // one GPU: the complete gradient row, rounded to bf16 here (no fp32 round trip)
        uint4* d16 = reinterpret_cast<uint4*>(
            reinterpret_cast<__nv_bfloat16*>(c == 0 ? p.dv : p.dk) + (row * p.Hkv + hkv) * 128);
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          uint32_t a[32];
          BAM_TMEM_LD32(tmem + lane_base + (c == 0 ? kColDV : kColDK) + q * 32, a);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 4; ++i)
            d16[q * 4 + i] = make_uint4(
                pack_bf16(__uint_as_float(a[8 * i]) * mul, __uint_as_float(a[8 * i + 1]) * mul),
                pack_bf16(__uint_as_float(a[8 * i + 2]) * mul, __uint_as_float(a[8 * i + 3]) * mul),
                pack_bf16(__uint_as_float(a[8 * i + 4]) * mul, __uint_as_float(a[8 * i + 5]) * mul),
                pack_bf16(__uint_as_float(a[8 * i + 6]) * mul, __uint_as_float(a[8 * i + 7]) * mul));
        }
      } else
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        uint32_t a[32];
        BAM_TMEM_LD32(tmem + lane_base + (c == 0 ? kColDV : kColDK) + q * 32, a);
        tmem_wait_ld();
        float4* d4 = reinterpret_cast<float4*>(dst + q * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          d4[i] = make_float4(__uint_as_float(a[4 * i]) * mul, __uint_as_float(a[4 * i + 1]) * mul,
                              __uint_as_float(a[4 * i + 2]) * mul,
                              __uint_as_float(a[4 * i + 3]) * mul);
      }
    } else if (p.dkv_bf16 && p.dkv_peers == nullptr) {
      uint4* d16 = reinterpret_cast<uint4*>(
          reinterpret_cast<__nv_bfloat16*>(c == 0 ? p.dv : p.dk) + (row * p.Hkv + hkv) * 128);
      for (int i = 0; i < 16; ++i) d16[i] = make_uint4(0u, 0u, 0u, 0u);
    } else {
      float4* d4 = reinterpret_cast<float4*>(dst);
      for (int i = 0; i < 32; ++i) d4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    }
  done:;
  } else {
    // ------------------------------------------------------------ dQ epilogue warps 8-11
    // TMEM lane = head-dim column d; columns = the 64 queries of the step.  The
    // accumulator is head-major [Hq, rows, 128] fp32, so the 64 rows of a step
    // sit at compile-time 512-B strides from one base (immediate offsets).
    const int d = (warp - kWarpDQ) * 32 + lane;
    const uint32_t lane_base = ((warp - kWarpDQ) * 32) << 16;
    StepIter it(col, grp, hkv, p.h_begin);
    float* const dq_stage0 = reinterpret_cast<float*>(sm.v);  // V lives in TMEM by now
    int n_export = 0;
    for (int s = 0; s < nsteps; ++s) {
      const uint32_t tDQ = tmem + kColDP;
      const StepInfo si = it.get();
      it.next();
      float* dst = p.dq_acc + ((int64_t)si.h * Tq + si.jq * 128 + si.half * 64) * 128 + d;
      // on the K/V-in-TMEM chain (dP(s+1) waits for this drain): short back-off
      mbar_wait_sleep<BAM_DQ_SLEEP_NS>(&sm.bar_dq_full, s & 1);
      BAM_TRACE_EV(trace_cta && threadIdx.x == kWarpDQ * 32, 8, s);
      tc_fence_after();
      uint32_t a[32], c2[32];
      BAM_TMEM_LD32(tDQ + lane_base, a);
      BAM_TMEM_LD32(tDQ + lane_base + 32, c2);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&sm.bar_dq_empty);
      if (si.cls == 0) continue;  // pair step this key block skips: dQ^T is zero
      // staging buffer free once the bulk reduce that last used it has read it
      const bool dq_leader = threadIdx.x == kWarpDQ * 32;
      float* const dq_stage = (n_export++ & 1) ? sm.dq_stage : dq_stage0;
      if (dq_leader) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      BAM_TRACE_EV(trace_cta && dq_leader, 13, s);
      named_bar_sync(1, 128);
#pragma unroll
      for (int i = 0; i < 32; ++i) dq_stage[i * 128 + d] = __uint_as_float(a[i]);
#pragma unroll
      for (int i = 0; i < 32; ++i) dq_stage[(32 + i) * 128 + d] = __uint_as_float(c2[i]);
      fence_async_smem();
      named_bar_sync(1, 128);
      BAM_TRACE_EV(trace_cta && dq_leader, 15, s);
      if (dq_leader) {
        float* gdst = dst - d;   // 64 rows x 512 B contiguous in the head-major accumulator
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;\n\t"
            "cp.async.bulk.commit_group;" ::"l"(gdst),
            "r"(smem_u32(dq_stage)), "n"(64 * 128 * 4)
            : "memory");
      }
      BAM_TRACE_EV(trace_cta && threadIdx.x == kWarpDQ * 32, 9, s);
    }
    if (threadIdx.x == kWarpDQ * 32) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (cluster_mode) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == kWarpMMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  BAM_CTA_CLOCK_END(nsteps);
}

// ld[h, 0, row] = lse[h, row] * log2e, ld[h, 1, row] = sum_d dO[row, h, d] * O[row, h, d],
// and the dQ accumulator row dq_acc[h, row, :] = 0 (one warp per (row, h); the
// zeroing replaces a separate 2-GB memset at config 4)
__global__ void bwd_delta_kernel(const __nv_bfloat16* __restrict__ o,
                                 const __nv_bfloat16* __restrict__ dout,
                                 const float* __restrict__ lse, int64_t rows, int H,
                                 float* __restrict__ ld, float* __restrict__ dq_acc) {
  // one warp per 4 (row, head) items: 8 independent 8-B loads in flight per lane
  const int64_t nw = rows * H;
  const int lane = lane_id();
  for (int64_t w0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 4; w0 < nw;
       w0 += (((int64_t)gridDim.x * blockDim.x) >> 5) * 4) {
    uint2 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t w = w0 + u < nw ? w0 + u : nw - 1;
      a[u] = __ldcs(reinterpret_cast<const uint2*>(o + w * 128) + lane);
      b[u] = __ldcs(reinterpret_cast<const uint2*>(dout + w * 128) + lane);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (w0 + u < nw) {
        const int64_t w = w0 + u, row = w / H, h = w - row * H;
        reinterpret_cast<float4*>(dq_acc + (h * rows + row) * 128)[lane] =
            make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    float acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a[u]);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b[u]);
      float t = 0.f;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(b2[i]);
        t = fmaf(x.x, y.x, fmaf(x.y, y.y, t));
      }
      acc[u] = t;
    }
#pragma unroll
    for (int s = 16; s; s >>= 1)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], s);
    if (lane < 4 && w0 + lane < nw) {
      const float mine = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
      const int64_t w = w0 + lane, row = w / H, h = w % H;
      ld[h * 2 * rows + row] = lse[h * rows + row] * 1.4426950408889634f;
      ld[h * 2 * rows + rows + row] = mine;
    }
  }
}

// dq[row, h, :] (bf16) = scale * dq_acc[h, row, :]   (one warp per (row, h))
__global__ void bwd_dq_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                                      int64_t rows, int H, float scale) {
  const int64_t nw = rows * H;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = w / H, h = w % H;
    const float4 v = reinterpret_cast<const float4*>(acc + (h * rows + row) * 128)[lane_id()];
    reinterpret_cast<uint2*>(dq + w * 128)[lane_id()] =
        make_uint2(pack_bf16(v.x * scale, v.y * scale), pack_bf16(v.z * scale, v.w * scale));
  }
}

// CTA-pair step lists (bam_build_pair_lists): one thread per pair merges the
// two ascending CSC columns.  Pass 1 (tiles == nullptr) counts, pass 2 fills.
__global__ void pair_lists_kernel(const int32_t* __restrict__ col_off,
                                  const int32_t* __restrict__ col_tiles,
                                  const int32_t* __restrict__ order, int32_t nb,
                                  int32_t* __restrict__ slot_kb, int32_t* __restrict__ slot_cnt,
                                  const int32_t* __restrict__ slot_off, int32_t* __restrict__ tiles,
                                  int32_t* __restrict__ pair_shared) {
  const int npairs = (nb + 1) / 2;
  for (int pr = blockIdx.x * blockDim.x + threadIdx.x; pr < npairs; pr += gridDim.x * blockDim.x) {
    const int a = order[2 * pr], b = 2 * pr + 1 < nb ? order[2 * pr + 1] : -1;
    const int32_t* ca = col_tiles + col_off[a];
    const int na = col_off[a + 1] - col_off[a];
    const int32_t* cb = b >= 0 ? col_tiles + col_off[b] : nullptr;
    const int nbb = b >= 0 ? col_off[b + 1] - col_off[b] : 0;
    if (tiles == nullptr) {
      slot_kb[2 * pr] = a;
      slot_kb[2 * pr + 1] = b;
      int u = 0, i = 0, k = 0;
      while (i < na || k < nbb) {
        const int ja = i < na ? ca[i] >> 2 : 0x7fffffff, jb = k < nbb ? cb[k] >> 2 : 0x7fffffff;
        i += ja <= jb;
        k += jb <= ja;
        ++u;
      }
      const int mx = na > nbb ? na : nbb;
      const bool sh = b >= 0 && mx > 0 && 8 * u <= 9 * mx;
      pair_shared[pr] = sh;
      slot_cnt[2 * pr] = sh ? u : na;
      slot_cnt[2 * pr + 1] = sh ? u : nbb;
    } else {
      int32_t* oa = tiles + slot_off[2 * pr];
      int32_t* ob = tiles + slot_off[2 * pr + 1];
      if (pair_shared[pr]) {  // union walk: both slots get every j, class 0 where absent
        int i = 0, k = 0, n = 0;
        while (i < na || k < nbb) {
          const int ja = i < na ? ca[i] >> 2 : 0x7fffffff, jb = k < nbb ? cb[k] >> 2 : 0x7fffffff;
          const int j = ja < jb ? ja : jb;
          oa[n] = (j << 2) | (ja == j ? (ca[i] & 3) : 0);
          ob[n] = (j << 2) | (jb == j ? (cb[k] & 3) : 0);
          i += ja == j;
          k += jb == j;
          ++n;
        }
      } else {
        for (int i = 0; i < na; ++i) oa[i] = ca[i];
        for (int k = 0; k < nbb; ++k) ob[k] = cb[k];
      }
    }
  }
}

}  // namespace bwd
}  // namespace bam

using namespace bam;

static int check_bwd(const BamAttnBwdParams* pp) {
  BAM_CHECK_ARG(pp != nullptr, "bam_attn_bwd: null params");
  const BamAttnBwdParams& p = *pp;
  BAM_CHECK_ARG(p.nq >= 1 && p.nb >= 1 && p.k_rows >= 1, "bam_attn_bwd: nq=%d nb=%d k_rows=%d",
                p.nq, p.nb, p.k_rows);
  const int nh = p.nh > 0 ? p.nh : p.Hq;
  BAM_CHECK_ARG(p.Hq >= 1 && p.Hkv >= 1 && nh % p.Hkv == 0 && p.h_begin >= 0 &&
                    p.h_begin + nh <= p.Hq,
                "bam_attn_bwd: head group [%d, %d) of Hq=%d over Hkv=%d", p.h_begin,
                p.h_begin + nh, p.Hq, p.Hkv);
  BAM_CHECK_ARG(p.nb <= 65535, "bam_attn_bwd: nb=%d > 65535", p.nb);
  BAM_CHECK_ARG(!(p.dkv_bf16 && p.dkv_peers), "bam_attn_bwd: dkv_bf16 with dkv_peers");
  BAM_CHECK_ARG(p.dkv_peers == nullptr ||
                    (p.dkv_rows_per_owner >= 128 && p.dkv_rows_per_owner % 128 == 0 &&
                     (int64_t)p.k_rows * 128 % p.dkv_rows_per_owner == 0),
                "bam_attn_bwd: dkv_rows_per_owner=%d must be a multiple of 128 dividing %d",
                p.dkv_rows_per_owner, p.k_rows * 128);
  return kOk;
}

extern "C" {

// Development aid: install the per-step trace buffer of -DBAM_TRACE builds of
// the backward kernel (returns BAM_UNSUPPORTED otherwise).
int bam_set_trace_buffer(void* buf) {
#ifdef BAM_TRACE
  BAM_CUDA_TRY(cudaMemcpyToSymbol(g_bam_trace, &buf, sizeof(buf)));
  return BAM_OK;
#else
  (void)buf;
  set_last_error("libbam built without -DBAM_TRACE");
  return BAM_UNSUPPORTED;
#endif
}

// Development aid: install the per-CTA clock buffers ([CTAs][4] u64 of the
// forward head-pair / backward kernels) of -DBAM_CTA_CLOCK builds.
int bam_set_cta_clock_buffer(void* fwd_buf, void* bwd_buf) {
#ifdef BAM_CTA_CLOCK
  BAM_CUDA_TRY(cudaMemcpyToSymbol(g_bam_cta_clock, &bwd_buf, sizeof(bwd_buf)));
  return fwd_set_cta_clock(fwd_buf);
#else
  (void)fwd_buf;
  (void)bwd_buf;
  set_last_error("libbam built without -DBAM_CTA_CLOCK");
  return BAM_UNSUPPORTED;
#endif
}

int bam_attn_bwd_preprocess(const BamAttnBwdParams* pp, void* stream) {
  if (int rc = check_bwd(pp)) return rc;
  const BamAttnBwdParams& p = *pp;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rows = (int64_t)p.nq * 128;
  bwd::bwd_delta_kernel<<<148 * 8, 256, 0, s>>>((const __nv_bfloat16*)p.o,
                                                (const __nv_bfloat16*)p.dout, p.lse, rows, p.Hq,
                                                p.delta, p.dq_acc);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_attn_bwd_main(const BamAttnBwdParams* pp, void* stream) {
  if (int rc = check_bwd(pp)) return rc;
  const BamAttnBwdParams& p = *pp;
  const int64_t rows = (int64_t)p.nq * 128;
  CUtensorMap mq, mk, mv, mdo;
  int rc;
  if ((rc = make_tmap_rows_heads_d128(&mq, p.q, rows, p.Hq, 64))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mdo, p.dout, rows, p.Hq, 64))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mk, p.k, (int64_t)p.k_rows * 128, p.Hkv, 128,
                                      p.kv_head_major)))
    return rc;
  if ((rc = make_tmap_rows_heads_d128(&mv, p.v, (int64_t)p.k_rows * 128, p.Hkv, 128,
                                      p.kv_head_major)))
    return rc;
  const int smem = (int)sizeof(bwd::Smem);
  BAM_CUDA_TRY(cudaFuncSetAttribute(bwd::attn_bwd_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (p.pair_shared) {  // CTA pairs: clusters of 2 along the (slot) y dimension
    BAM_CHECK_ARG(p.n_slots >= 2 && p.n_slots % 2 == 0 && p.order != nullptr,
                  "bam_attn_bwd: pair mode needs an even n_slots=%d and slot_kb", p.n_slots);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.n_slots, p.Hkv);
    cfg.blockDim = dim3(bwd::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    BAM_CUDA_TRY(cudaLaunchKernelEx(&cfg, bwd::attn_bwd_kernel, mq, mk, mv, mdo, p));
  } else {
    const dim3 grid(p.nb, p.Hkv);
    bwd::attn_bwd_kernel<<<grid, bwd::kThreads, smem, (cudaStream_t)stream>>>(mq, mk, mv, mdo, p);
  }
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_attn_bwd_finalize(const BamAttnBwdParams* pp, void* stream) {
  if (int rc = check_bwd(pp)) return rc;
  const BamAttnBwdParams& p = *pp;
  bwd::bwd_dq_convert_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
      p.dq_acc, reinterpret_cast<__nv_bfloat16*>(p.dq), (int64_t)p.nq * 128, p.Hq, p.scale);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_build_pair_lists(const int32_t* col_off, const int32_t* col_tiles, const int32_t* order,
                         int32_t nb, int32_t* slot_kb, int32_t* slot_cnt, int32_t* slot_off,
                         int32_t* slot_tiles, int32_t* pair_shared, void* stream) {
  BAM_CHECK_ARG(nb >= 1 && order != nullptr, "bam_build_pair_lists: nb=%d", nb);
  cudaStream_t s = (cudaStream_t)stream;
  const int npairs = (nb + 1) / 2;
  const int grid = (npairs + 127) / 128;
  if (slot_tiles == nullptr) {
    bwd::pair_lists_kernel<<<grid, 128, 0, s>>>(col_off, col_tiles, order, nb, slot_kb, slot_cnt,
                                                nullptr, nullptr, pair_shared);
    BAM_LAUNCH_CHECK();
    scan_kernel<<<1, 1024, 0, s>>>(slot_cnt, 2 * npairs, slot_off);
  } else {
    bwd::pair_lists_kernel<<<grid, 128, 0, s>>>(col_off, col_tiles, order, nb, slot_kb, slot_cnt,
                                                slot_off, slot_tiles, pair_shared);
  }
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_attn_bwd(const BamAttnBwdParams* pp, void* stream) {
  int rc;
  if ((rc = bam_attn_bwd_preprocess(pp, stream))) return rc;
  if ((rc = bam_attn_bwd_main(pp, stream))) return rc;
  return bam_attn_bwd_finalize(pp, stream);
}

}  // extern "C"
