// Bitfield-masked attention forward for sm_100a (tcgen05 + TMEM + TMA).
//
// Semantics: O = softmax(scale * Q K^T, masked by materialize()) V per query
// head, mask per reference mask.py:106-112, computed blockwise over the
// non-skip 128x128 tiles only: FULL tiles take no mask,
// PARTIAL tiles evaluate the 64-bit descriptor predicate in registers.
//
// One CTA = one 128-row query block x one query head; 2 CTAs per SM so one
// CTA's softmax overlaps the other's MMAs.
//   warps 0-3  softmax: thread r owns row r (= TMEM lane r); online softmax
//              with lazy (2^8) rescaling of the TMEM O accumulator
//   warp 4     TMA producer: Q once, then K / V tiles (single-buffered each;
//              K(t+1) streams in during softmax(t), V(t+1) during S(t+1))
//   warp 5     TMEM allocator + MMA issuer (one thread):
//              S = Q K^T (SS, K-major x K-major) -> TMEM cols [0,128)
//              O += P V  (TS: P bf16 in TMEM cols [0,64), V MN-major) -> [128,256)
#include "../../include/bam.h"
#include "common.cuh"
#include "kernels.cuh"
#include "tma.h"

namespace bam {

namespace fwd {

constexpr int kThreads = 192;
constexpr uint32_t kTileBytes = 128 * 128 * 2;  // one 128x128 bf16 tile (two 64-col boxes)
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kColS = 0, kColO = 128;

struct Smem {
  alignas(1024) uint8_t q[kTileBytes];
  alignas(1024) uint8_t k[kTileBytes];
  alignas(1024) uint8_t v[kTileBytes];
  uint64_t bar_q, bar_k_full, bar_k_empty, bar_v_full, bar_v_empty;
  uint64_t bar_s_full, bar_p_full, bar_pv_done;
  uint32_t tmem_base;
};

__device__ __forceinline__ void load_tile(const CUtensorMap* m, uint64_t* bar, uint8_t* dst,
                                          int head, int row0) {
  tma_load_3d(m, bar, dst, 0, head, row0);
  tma_load_3d(m, bar, dst + kTileBytes / 2, 64, head, row0);
}

// The CP arrival flag guarding rank `owner`'s rows of KV head hkv
// (BamAttnFwdParams.kv_ready / kv_head_major / kv_flag_heads)
__device__ __forceinline__ int kv_flag_index(const BamAttnFwdParams& p, int owner, int hkv) {
  if (!p.kv_head_major) return owner;
  const int g = p.kv_flag_heads > 1 ? p.kv_flag_heads : 1;
  return owner * p.Hkv + (hkv / g) * g;
}

// One CTA's work: a whole query-block row (items == NULL: heavy-first order)
// or a split-KV subblock [first, end) of its tile list (LPT-ordered items).
struct WorkItem {
  int j, n, slot;
  const int32_t* tiles;
};
__device__ __forceinline__ WorkItem work_item(const BamAttnFwdParams& p, int y) {
  WorkItem w;
  if (p.items) {
    const int4 it = reinterpret_cast<const int4*>(p.items)[y];
    w.j = it.x;
    w.tiles = p.row_tiles + p.row_off[it.x] + it.y;
    w.n = it.z - it.y;
    w.slot = it.w;
  } else {
    w.j = p.order ? p.order[y] : y;
    w.tiles = p.row_tiles + p.row_off[w.j];
    w.n = p.row_off[w.j + 1] - p.row_off[w.j];
    w.slot = -1;
  }
  return w;
}

// One in kPolyEvery exponential PAIRS runs on the FMA pipe (ex2_poly2) so the MUFU
// unit (16 ex2 / clk / SM) is not the softmax bottleneck.  Measured on B200:
// the MHA kernel (two CTAs per SM) is fastest at 1 in 3; the CTA-pair kernel
// (one softmax thread per row at its 168-register ceiling) with none; the
// split-row head-pair kernel at 1 in 4 (BAM_FWD_POLY_SPLIT).
#ifndef BAM_FWD_POLY_MHA
#define BAM_FWD_POLY_MHA 3
#endif
#ifndef BAM_FWD_POLY_PAIR
#define BAM_FWD_POLY_PAIR 0
#endif

// Softmax / epilogue role of one 128-row query tile: thread (warp w, lane)
// owns row r = 32 w + lane = TMEM lane r.  Per key tile t: wait S(t), mask
// PARTIAL tiles, online softmax (log2 domain, lazy 2^8 rescale of O in TMEM),
// P -> bf16 into the S columns, arrive p_ready.  Finally O / l -> bf16, LSE.
// Grid order.  Row-major (query blocks / work items fastest, heads slowest):
// the CTAs resident together read the K/V tiles of one KV head, which stay in
// L2; head-major spreads every wave over all KV heads.
#ifndef BAM_FWD_ROW_MAJOR
#define BAM_FWD_ROW_MAJOR 1
#endif
constexpr bool kRowMajor = BAM_FWD_ROW_MAJOR;
// P(t) released to the PV MMAs in chunks (2: keys 32 apart per thread half; 4: 16).
// Measured on config 4: one release 1210, 2 chunks 1320-1330 TFLOP/s
#ifndef BAM_FWD_P_CHUNKS
#define BAM_FWD_P_CHUNKS 2
#endif
constexpr int kPChunks = BAM_FWD_P_CHUNKS;

template <int kPolyEvery>
__device__ __forceinline__ void softmax_role(const BamAttnFwdParams& p, uint32_t tmem,
                                             uint32_t colS, uint32_t colO, uint64_t* bar_s_full,
                                             uint64_t* bar_p_ready, uint64_t* bar_pv_done, int j,
                                             int h, uint32_t warp, uint32_t lane,
                                             const int32_t* tiles, int n, int slot,
                                             uint32_t p_ready_remote = 0) {
  const int r = (warp & 3) * 32 + lane;
  const uint32_t lane_base = ((warp & 3) * 32) << 16;
  const long long qg = (long long)p.q_gid[j] * 128 + r;
  const float scale_log2 = p.scale * 1.4426950408889634f;
  float m = -INFINITY, l = 0.f;
  for (int t = 0; t < n; ++t) {
    const int e = tiles[t];
    const int cls = e & 3;
    const long long kg0 = (long long)(e >> 2) * 128;
    // allow bits first (descriptors only): overlaps the wait for S(t) and keeps the
    // predicate's temporaries out of the S row's live range
    uint32_t bits[4] = {~0u, ~0u, ~0u, ~0u};
    if (cls == 2) {  // PARTIAL: descriptor predicate per element, 32 columns at a time
      const long long* dk = reinterpret_cast<const long long*>(p.desc) + kg0;
      const long long dq = __ldg(reinterpret_cast<const long long*>(p.desc) + qg);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t b = 0;
#pragma unroll 4
        for (int i = 0; i < 32; ++i) {
          const long long d = __ldg(dk + c * 32 + i);
          b |= uint32_t(bam_allowed(dq, qg, d, kg0 + c * 32 + i)) << i;
        }
        bits[c] = b;
      }
    } else if (cls == 0) {  // a tile only the other CTA of a pair sees: fully masked here
      bits[0] = bits[1] = bits[2] = bits[3] = 0u;
    }
    mbar_wait_sleep<BAM_COMPUTE_SLEEP_NS>(bar_s_full, t & 1);
    tc_fence_after();
    uint32_t sr[128];  // S row as fp32 bits: four TMEM loads in flight, one wait
#pragma unroll
    for (int c = 0; c < 4; ++c) BAM_TMEM_LD32(tmem + lane_base + colS + c * 32, (sr + c * 32));
    tmem_wait_ld();
    if (cls != 1) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (!((bits[c] >> i) & 1)) sr[c * 32 + i] = 0xff800000u;  // -inf
    }
    // row max: eight independent FMNMX3 chains instead of one serial chain
    float mx[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) mx[k] = fmaxf(__uint_as_float(sr[2 * k]), __uint_as_float(sr[2 * k + 1]));
#pragma unroll
    for (int c = 16; c < 128; c += 16)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        mx[k] = fmaxf(mx[k], fmaxf(__uint_as_float(sr[c + 2 * k]), __uint_as_float(sr[c + 2 * k + 1])));
    const float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                           fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
    const float m_new = fmaxf(m, mt * scale_log2);
    // lazy rescale: only when the running max grows by more than 2^8
    const bool rescale = m_new > m + 8.f;
    const float alpha = rescale ? ex2(m - m_new) : 1.f;  // m = -inf -> 0
    if (rescale) {
      l *= alpha;
      m = m_new;
    }
    const float mb = (m == -INFINITY) ? 0.f : m;
    const float2 sc2 = make_float2(scale_log2, scale_log2), nmb2 = make_float2(-mb, -mb);
    float2 ls = make_float2(0.f, 0.f);  // one chain: its FADD2 latency hides under MUFU
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 x = ffma2(make_float2(__uint_as_float(sr[c * 32 + 2 * i]),
                                           __uint_as_float(sr[c * 32 + 2 * i + 1])),
                               sc2, nmb2);
        const float2 pp = (kPolyEvery > 0 && (c * 16 + i) % (kPolyEvery > 0 ? kPolyEvery : 1) ==
                                                 kPolyEvery - 1)
                              ? ex2_poly2(x)
                              : make_float2(ex2(x.x), ex2(x.y));
        ls = fadd2(ls, pp);
        pk[i] = pack_bf16(pp.x, pp.y);
      }
      BAM_TMEM_ST16(tmem + lane_base + colS + c * 16, pk);
    }
    l += ls.x + ls.y;
    // warp-uniform branch: tcgen05.ld/st are .sync.aligned (alpha == 1 for rows that keep m).
    // O(t-1) is complete: S(t) was issued after PV(t-1) and its commit covers it.
    if (__any_sync(0xffffffffu, rescale) && t > 0) {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t rr[32];
        BAM_TMEM_LD32(tmem + lane_base + colO + c * 32, rr);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) rr[i] = __float_as_uint(__uint_as_float(rr[i]) * alpha);
        BAM_TMEM_ST32(tmem + lane_base + colO + c * 32, rr);
      }
    }
    tmem_wait_st();
    tc_fence_before();
    if (p_ready_remote) {  // the pair leader's barrier: one arrival per warp
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(p_ready_remote);
    } else {
      mbar_arrive(bar_p_ready);
    }
  }
  // epilogue of a split-KV subblock: unnormalised fp32 O and (m, l) for the combine
  if (slot >= 0) {
    float* po = p.part_o + (((int64_t)slot * p.Hq + h) * 128 + r) * 128;
    if (n > 0) {
      mbar_wait_sleep(bar_pv_done, (n - 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t rr[32];
        BAM_TMEM_LD32(tmem + lane_base + colO + c * 32, rr);
        tmem_wait_ld();
        float4* dst = reinterpret_cast<float4*>(po + c * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[i] = make_float4(__uint_as_float(rr[4 * i]), __uint_as_float(rr[4 * i + 1]),
                               __uint_as_float(rr[4 * i + 2]), __uint_as_float(rr[4 * i + 3]));
      }
    } else {
      for (int i = 0; i < 32; ++i) reinterpret_cast<float4*>(po)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    reinterpret_cast<float2*>(p.part_ml)[((int64_t)slot * p.Hq + h) * 128 + r] =
        make_float2(n > 0 ? m : -INFINITY, n > 0 ? l : 0.f);
    return;
  }
  // epilogue: O / l -> bf16, LSE
  const int64_t Tq = (int64_t)p.nq * 128;
  const int64_t row = (int64_t)j * 128 + r;
  __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o) + (row * p.Hq + h) * 128;
  if (n > 0) {
    mbar_wait_sleep(bar_pv_done, (n - 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t rr[32];
      BAM_TMEM_LD32(tmem + lane_base + colO + c * 32, rr);
      tmem_wait_ld();
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 v;
        v.x = pack_bf16(__uint_as_float(rr[8 * i + 0]) * inv, __uint_as_float(rr[8 * i + 1]) * inv);
        v.y = pack_bf16(__uint_as_float(rr[8 * i + 2]) * inv, __uint_as_float(rr[8 * i + 3]) * inv);
        v.z = pack_bf16(__uint_as_float(rr[8 * i + 4]) * inv, __uint_as_float(rr[8 * i + 5]) * inv);
        v.w = pack_bf16(__uint_as_float(rr[8 * i + 6]) * inv, __uint_as_float(rr[8 * i + 7]) * inv);
        dst[i] = v;
      }
    }
    p.lse[(int64_t)h * Tq + row] = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
  } else {
    uint4* dst = reinterpret_cast<uint4*>(orow);
    for (int i = 0; i < 16; ++i) dst[i] = make_uint4(0, 0, 0, 0);
    p.lse[(int64_t)h * Tq + row] = -INFINITY;
  }
}

__global__ void __launch_bounds__(kThreads, 2)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const BamAttnFwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  const uint32_t warp = warp_id(), lane = lane_id();
  const int nh = p.nh > 0 ? p.nh : p.Hq;
  const int h = p.h_begin + (kRowMajor ? blockIdx.y : blockIdx.x);
  // device-counted items (bam_plan_build): the grid is an upper bound
  if (p.dev_counts && p.items && (int)(kRowMajor ? blockIdx.x : blockIdx.y) >= p.dev_counts[1])
    return;
  const WorkItem wi = work_item(p, kRowMajor ? blockIdx.x : blockIdx.y);
  const int j = wi.j, n = wi.n, slot = wi.slot;
  const int32_t* tiles = wi.tiles;
  const int hkv = (h - p.h_begin) / (nh / p.Hkv);

  if (threadIdx.x == 0) {
    mbar_init(&sm.bar_q, 1);
    mbar_init(&sm.bar_k_full, 1);
    mbar_init(&sm.bar_k_empty, 1);
    mbar_init(&sm.bar_v_full, 1);
    mbar_init(&sm.bar_v_empty, 1);
    mbar_init(&sm.bar_s_full, 1);
    mbar_init(&sm.bar_p_full, 128);
    mbar_init(&sm.bar_pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 5) {
    tmem_alloc(&sm.tmem_base, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer (whole warp)
    const uint32_t leader = elect_one();
    if (n > 0) {
      if (leader) {
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        prefetch_tmap(&tm_v);
      }
      mbar_expect_tx_w(&sm.bar_q, kTileBytes, leader);
      tma_load_3d_w(&tm_q, &sm.bar_q, sm.q, 0, h, j * 128, leader);
      tma_load_3d_w(&tm_q, &sm.bar_q, sm.q + kTileBytes / 2, 64, h, j * 128, leader);
      uint64_t ready = 0;  // CP overlap: ranks whose K/V rows are known to have landed
      for (int t = 0; t < n; ++t) {
        const int kblk = p.k_row[tiles[t] >> 2];
        const int krow = kblk * 128;
        if (p.kv_ready) {
          const int owner = kblk / p.kv_rows_per_rank;
          if (owner != p.kv_rank && !((ready >> owner) & 1)) {
            if (lane == 0)
              wait_flag_geq(p.kv_ready + kv_flag_index(p, owner, hkv),
                            p.kv_epoch);
            __syncwarp();
            fence_proxy_async_global();
            ready |= 1ull << owner;
          }
        }
        if (t > 0) mbar_wait_sleep(&sm.bar_k_empty, (t - 1) & 1);
        mbar_expect_tx_w(&sm.bar_k_full, kTileBytes, leader);
        tma_load_3d_w(&tm_k, &sm.bar_k_full, sm.k, 0, hkv, krow, leader);
        tma_load_3d_w(&tm_k, &sm.bar_k_full, sm.k + kTileBytes / 2, 64, hkv, krow, leader);
        if (t > 0) mbar_wait_sleep(&sm.bar_v_empty, (t - 1) & 1);
        mbar_expect_tx_w(&sm.bar_v_full, kTileBytes, leader);
        tma_load_3d_w(&tm_v, &sm.bar_v_full, sm.v, 0, hkv, krow, leader);
        tma_load_3d_w(&tm_v, &sm.bar_v_full, sm.v + kTileBytes / 2, 64, hkv, krow, leader);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer (whole warp)
    const uint32_t leader = elect_one();
    if (n > 0) {
      const uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
      const uint32_t idesc_o = idesc_bf16(128, 128, 0, 1);
      const uint64_t dq = sdesc_sw128(smem_u32(sm.q), 16, 1024);
      const uint64_t dk = sdesc_sw128(smem_u32(sm.k), 16, 1024);
      const uint64_t dv = sdesc_sw128(smem_u32(sm.v), kTileBytes / 2, 1024);
      mbar_wait(&sm.bar_q, 0);
      for (int t = 0; t < n; ++t) {
        mbar_wait(&sm.bar_k_full, t & 1);
        if (t > 0) mbar_wait(&sm.bar_pv_done, (t - 1) & 1);  // P(t-1) in S cols consumed
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * (kTileBytes / 2) + (kk & 3) * 32) >> 4;
          mma_ss_w(tmem + kColS, dq + off, dk + off, idesc_s, kk > 0, leader);
        }
        tc_commit_w(&sm.bar_s_full, leader);
        tc_commit_w(&sm.bar_k_empty, leader);
        mbar_wait(&sm.bar_p_full, t & 1);
        mbar_wait(&sm.bar_v_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts_w(tmem + kColO, tmem + kColS + kk * 8, dv + kk * 128, idesc_o, (t > 0 || kk > 0),
                   leader);
        tc_commit_w(&sm.bar_pv_done, leader);
        tc_commit_w(&sm.bar_v_empty, leader);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps 0-3
    softmax_role<BAM_FWD_POLY_MHA>(p, tmem, kColS, kColO, &sm.bar_s_full, &sm.bar_p_full, &sm.bar_pv_done, j, h,
                 warp, lane, tiles, n, slot);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// GQA head pairs: one CTA = one 128-row query block x two query heads of the
// same KV group (identical tile lists and masks, shared K/V tiles), 1 CTA per
// SM.  TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).  The MMA warp
// ping-pongs the two tiles so one head's softmax overlaps the other head's
// MMAs:  S0(0) S1(0) | PV0(0) S0(1) | PV1(0) S1(1) | PV0(1) S0(2) | ...
// K/V tiles stream through a 2-stage ring.  (A 320-thread variant with one
// softmax thread per row sat at its 168-register launch ceiling -- registers
// are allocated per warpgroup, 12 x 32 x 168 -- and spilled; the split-row
// kernel below replaced it: config 4 forward 1125 -> 1220 TFLOP/s.)
constexpr int kPairThreads = 320;   // the CTA-pair kernel's block size

// ---------------------------------------------------------------------------
// Split-row softmax: TWO threads per query row (warps q and q+4 of a head's
// eight softmax warps share TMEM lane quadrant q; thread half hf owns S / O
// columns [64 hf, 64 hf + 64)).  Each thread carries 64 S values instead of
// 128, so (a) a head-tile's 128 exponentials per row run on two warps' MUFU
// turns, halving the softmax latency the MMA ping-pong must hide, and (b) the
// row fits in ~100 registers.  The row max is combined through shared memory
// (one 64-thread named barrier per tile); both threads then make the same
// rescale decision.
template <int kPolyEvery>
__device__ __forceinline__ void softmax_half_role(
    const BamAttnFwdParams& p, uint32_t tmem, uint32_t colS, uint32_t colO, uint64_t* bar_s_full,
    uint64_t* bar_p_ready /* [2]: P chunk 0, 1 */, uint64_t* bar_pv_done, int j, int h,
    uint32_t lw, uint32_t lane, const int32_t* tiles, int n, int slot,
    float* xch /* [2][2][128] */, uint32_t bar_id) {
  const uint32_t q = lw & 3, hf = lw >> 2;
  const int r = q * 32 + lane;
  const uint32_t lane_base = (q * 32) << 16;
  const uint32_t cS = colS + 64 * hf, cP = colS + 32 * hf, cO = colO + 64 * hf;
  const long long qg = (long long)p.q_gid[j] * 128 + r;
  const float scale_log2 = p.scale * 1.4426950408889634f;
  float m = -INFINITY, l = 0.f;
  for (int t = 0; t < n; ++t) {
    const int e = tiles[t];
    const int cls = e & 3;
    const long long kg0 = (long long)(e >> 2) * 128 + 64 * hf;
    uint32_t bits[2] = {~0u, ~0u};
    if (cls == 2) {
      const long long* dk = reinterpret_cast<const long long*>(p.desc) + kg0;
      const long long dq = __ldg(reinterpret_cast<const long long*>(p.desc) + qg);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t b = 0;
#pragma unroll 4
        for (int i = 0; i < 32; ++i) {
          const long long d = __ldg(dk + c * 32 + i);
          b |= uint32_t(bam_allowed(dq, qg, d, kg0 + c * 32 + i)) << i;
        }
        bits[c] = b;
      }
    } else if (cls == 0) {
      bits[0] = bits[1] = 0u;
    }
    mbar_wait_sleep<BAM_COMPUTE_SLEEP_NS>(bar_s_full, t & 1);
    tc_fence_after();
    uint32_t sr[64];
    BAM_TMEM_LD32(tmem + lane_base + cS, sr);
    BAM_TMEM_LD32(tmem + lane_base + cS + 32, (sr + 32));
    tmem_wait_ld();
    if (cls != 1) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (!((bits[c] >> i) & 1)) sr[c * 32 + i] = 0xff800000u;
    }
    float mx[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      mx[k] = fmaxf(__uint_as_float(sr[2 * k]), __uint_as_float(sr[2 * k + 1]));
#pragma unroll
    for (int c = 8; c < 64; c += 8)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mx[k] = fmaxf(mx[k], fmaxf(__uint_as_float(sr[c + 2 * k]), __uint_as_float(sr[c + 2 * k + 1])));
    float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
    // combine with the other half of the row (double-buffered by tile parity); the
    // barrier also orders the partner's S loads before this thread's P stores
    float* xb = xch + (t & 1) * 256;
    xb[hf * 128 + r] = mt;
    named_bar_sync(bar_id, 64);
    mt = fmaxf(mt, xb[(hf ^ 1) * 128 + r]);
    const float m_new = fmaxf(m, mt * scale_log2);
    const bool rescale = m_new > m + 8.f;
    const float alpha = rescale ? ex2(m - m_new) : 1.f;
    if (rescale) {
      l *= alpha;
      m = m_new;
    }
    const float mb = (m == -INFINITY) ? 0.f : m;
    const float2 sc2 = make_float2(scale_log2, scale_log2), nmb2 = make_float2(-mb, -mb);
    float2 ls = make_float2(0.f, 0.f);
    // P in kPChunks key chunks per thread (keys [64 hf + c 64/kPChunks, ...)), each
    // released on its own barrier: the MMA warp starts PV on the first chunks while
    // the later chunks' exponentials are still running
    constexpr int kPairsPerChunk = 32 / kPChunks;
#pragma unroll
    for (int c = 0; c < kPChunks; ++c) {
      uint32_t pk[kPairsPerChunk];
#pragma unroll
      for (int i = 0; i < kPairsPerChunk; ++i) {
        const int i2 = c * kPairsPerChunk + i;   // pair index within the thread's 64 keys
        const float2 x = ffma2(make_float2(__uint_as_float(sr[2 * i2]),
                                           __uint_as_float(sr[2 * i2 + 1])),
                               sc2, nmb2);
        const float2 pp = (kPolyEvery > 0 && i2 % (kPolyEvery > 0 ? kPolyEvery : 1) ==
                                                 kPolyEvery - 1)
                              ? ex2_poly2(x)
                              : make_float2(ex2(x.x), ex2(x.y));
        ls = fadd2(ls, pp);
        pk[i] = pack_bf16(pp.x, pp.y);
      }
      if constexpr (kPairsPerChunk == 16)
        BAM_TMEM_ST16(tmem + lane_base + cP + c * 16, pk);
      else
        BAM_TMEM_ST8(tmem + lane_base + cP + c * 8, pk);
      // the lazy rescale of O precedes the release of P(t)'s first chunk (PV(t-1) has
      // completed: S(t), committed after it by the same thread, is done); here, once
      // chunk 0's S values are dead, it fits the register budget (16-column pieces)
      if (c == 0 && __any_sync(0xffffffffu, rescale) && t > 0) {
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t rr[16];
          BAM_TMEM_LD16(tmem + lane_base + cO + cc * 16, rr);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) rr[i] = __float_as_uint(__uint_as_float(rr[i]) * alpha);
          BAM_TMEM_ST16(tmem + lane_base + cO + cc * 16, rr);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar_p_ready + c);
    }
    l += ls.x + ls.y;
  }
  // row sum of both halves (same m in both threads)
  xch[512 + hf * 128 + r] = l;
  named_bar_sync(bar_id, 64);
  const float l_row = l + xch[512 + (hf ^ 1) * 128 + r];
  if (slot >= 0) {  // split-KV subblock: unnormalised fp32 O and (m, l)
    float* po = p.part_o + (((int64_t)slot * p.Hq + h) * 128 + r) * 128 + 64 * hf;
    if (n > 0) {
      mbar_wait_sleep(bar_pv_done, (n - 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t rr[32];
        BAM_TMEM_LD32(tmem + lane_base + cO + c * 32, rr);
        tmem_wait_ld();
        float4* dst = reinterpret_cast<float4*>(po + c * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[i] = make_float4(__uint_as_float(rr[4 * i]), __uint_as_float(rr[4 * i + 1]),
                               __uint_as_float(rr[4 * i + 2]), __uint_as_float(rr[4 * i + 3]));
      }
    } else {
      for (int i = 0; i < 16; ++i) reinterpret_cast<float4*>(po)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (hf == 0)
      reinterpret_cast<float2*>(p.part_ml)[((int64_t)slot * p.Hq + h) * 128 + r] =
          make_float2(n > 0 ? m : -INFINITY, n > 0 ? l_row : 0.f);
    return;
  }
  const int64_t Tq = (int64_t)p.nq * 128;
  const int64_t row = (int64_t)j * 128 + r;
  __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o) + (row * p.Hq + h) * 128 + 64 * hf;
  if (n > 0) {
    mbar_wait_sleep(bar_pv_done, (n - 1) & 1);
    tc_fence_after();
    const float inv = l_row > 0.f ? 1.f / l_row : 0.f;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t rr[32];
      BAM_TMEM_LD32(tmem + lane_base + cO + c * 32, rr);
      tmem_wait_ld();
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 v;
        v.x = pack_bf16(__uint_as_float(rr[8 * i + 0]) * inv, __uint_as_float(rr[8 * i + 1]) * inv);
        v.y = pack_bf16(__uint_as_float(rr[8 * i + 2]) * inv, __uint_as_float(rr[8 * i + 3]) * inv);
        v.z = pack_bf16(__uint_as_float(rr[8 * i + 4]) * inv, __uint_as_float(rr[8 * i + 5]) * inv);
        v.w = pack_bf16(__uint_as_float(rr[8 * i + 6]) * inv, __uint_as_float(rr[8 * i + 7]) * inv);
        dst[i] = v;
      }
    }
    if (hf == 0)
      p.lse[(int64_t)h * Tq + row] =
          l_row > 0.f ? (m + __log2f(l_row)) * 0.6931471805599453f : -INFINITY;
  } else {
    uint4* dst = reinterpret_cast<uint4*>(orow);
    for (int i = 0; i < 8; ++i) dst[i] = make_uint4(0, 0, 0, 0);
    if (hf == 0) p.lse[(int64_t)h * Tq + row] = -INFINITY;
  }
}

// GQA head-pair kernel with split-row softmax: 16 softmax warps (8 per head:
// 2 per TMEM lane quadrant), warp 16 TMA, warp 17 MMA.
constexpr int kSplitThreads = 576;
#ifndef BAM_FWD_POLY_SPLIT
#define BAM_FWD_POLY_SPLIT 4
#endif

struct SplitSmem {
  alignas(1024) uint8_t q[2][kTileBytes];
  alignas(1024) uint8_t k[2][kTileBytes];
  alignas(1024) uint8_t v[2][kTileBytes];
  float xch[2][768];  // per head: max exchange [2 parity][2 halves][128] + row sums [2][128]
  uint64_t bar_q, bar_k_full[2], bar_k_empty[2], bar_v_full[2], bar_v_empty[2];
  uint64_t bar_s_full[2], bar_p_ready[2][kPChunks], bar_pv_done[2];  // p_ready[head][chunk]
  uint32_t tmem_base;
};

// kQPair = false: tile i = head h0 + i of query block j (GQA head pair).
// kQPair = true: tile i = query block slot_q[2 pr + i] of head h (MHA query-block
// pair of bam_build_pair_lists' shared pairs: one union tile list, class 0 where
// a block does not see the key tile), so the two tiles still share K/V.
template <bool kQPair>
__global__ void __launch_bounds__(kSplitThreads, 1)
    attn_fwd_split_kernel(const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const BamAttnFwdParams p,
                          const int32_t* __restrict__ pair_ids, const int32_t* __restrict__ slot_q,
                          const int32_t* __restrict__ slot_off,
                          const int32_t* __restrict__ slot_tiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SplitSmem& sm = *reinterpret_cast<SplitSmem*>(smem_raw);
  BAM_CTA_CLOCK_BEGIN();
  const uint32_t warp = warp_id(), lane = lane_id();
  const int nh = p.nh > 0 ? p.nh : p.Hq;
  int bx = kRowMajor ? blockIdx.x : blockIdx.y, by = kRowMajor ? blockIdx.y : blockIdx.x;
  if (p.order_classes && (kQPair || !p.items)) {
    // class-major CTA order: linear CTA L walks the work classes of the
    // heavy-first order (rows, or shared query-block pairs), each class head-pair
    // (head) major (BamAttnFwdParams.order_classes)
    const int npairs = kRowMajor ? gridDim.y : gridDim.x;
    const int L = blockIdx.x + gridDim.x * blockIdx.y;   // the block scheduler's dispatch order
    int lo = p.order_classes[0];
#pragma unroll 1
    for (int c = 1; c <= kOrderClasses; ++c) {
      const int hi = p.order_classes[c];
      if (L < npairs * hi) {
        const int len = hi - lo, off = L - npairs * lo;
        by = off / len;
        bx = lo + (off - by * len);
        break;
      }
      lo = hi;
    }
  }
  int jj[2], hh[2], n, slot;
  const int32_t* tl[2];
  // device-counted pairs / items (bam_plan_build): the grid is an upper bound
  if (p.dev_counts && (kQPair || p.items) && bx >= p.dev_counts[kQPair ? 0 : 1]) return;
  if constexpr (kQPair) {
    const int pr = pair_ids[bx];
    for (int i = 0; i < 2; ++i) {
      jj[i] = slot_q[2 * pr + i];
      hh[i] = p.h_begin + by;
      tl[i] = slot_tiles + slot_off[2 * pr + i];
    }
    n = slot_off[2 * pr + 1] - slot_off[2 * pr];
    slot = -1;
  } else {
    const WorkItem wi = work_item(p, bx);
    for (int i = 0; i < 2; ++i) {
      jj[i] = wi.j;
      hh[i] = p.h_begin + 2 * by + i;
      tl[i] = wi.tiles;
    }
    n = wi.n;
    slot = wi.slot;
  }
  const int32_t* tiles = tl[0];   // the key-tile order (identical in both lists)
  const int hkv = (hh[0] - p.h_begin) / (nh / p.Hkv);
  constexpr uint32_t kWarpTma = 16, kWarpMma = 17;

  if (threadIdx.x == 0) {
    if ((smem_u32(smem_raw) & 1023) != 0) __trap();
    mbar_init(&sm.bar_q, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.bar_k_full[i], 1);
      mbar_init(&sm.bar_k_empty[i], 1);
      mbar_init(&sm.bar_v_full[i], 1);
      mbar_init(&sm.bar_v_empty[i], 1);
      mbar_init(&sm.bar_s_full[i], 1);
      for (int c = 0; c < kPChunks; ++c) mbar_init(&sm.bar_p_ready[i][c], 256);
      mbar_init(&sm.bar_pv_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == kWarpMma) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == kWarpTma) {
    const uint32_t leader = elect_one();
    if (n > 0) {
      if (leader) {
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        prefetch_tmap(&tm_v);
      }
      mbar_expect_tx_w(&sm.bar_q, 2 * kTileBytes, leader);
      for (int i = 0; i < 2; ++i) {
        tma_load_3d_w(&tm_q, &sm.bar_q, sm.q[i], 0, hh[i], jj[i] * 128, leader);
        tma_load_3d_w(&tm_q, &sm.bar_q, sm.q[i] + kTileBytes / 2, 64, hh[i], jj[i] * 128, leader);
      }
      uint64_t ready = 0;  // CP overlap: ranks whose K/V rows are known to have landed
#ifdef BAM_CTA_CLOCK
      unsigned long long flag_wait_ns = 0;
#endif
      for (int t = 0; t < n; ++t) {
        const int st = t & 1;
        const int kblk = p.k_row[tiles[t] >> 2];
        const int krow = kblk * 128;
        if (p.kv_ready) {
          const int owner = kblk / p.kv_rows_per_rank;
          if (owner != p.kv_rank && !((ready >> owner) & 1)) {
#ifdef BAM_CTA_CLOCK
            const unsigned long long w0 = bam_globaltimer();
#endif
            if (lane == 0)
              wait_flag_geq(p.kv_ready + kv_flag_index(p, owner, hkv),
                            p.kv_epoch);
            __syncwarp();
            fence_proxy_async_global();  // the copy engine's data before the TMA reads
            ready |= 1ull << owner;
#ifdef BAM_CTA_CLOCK
            flag_wait_ns += bam_globaltimer() - w0;
#endif
          }
        }
        if (t >= 2) mbar_wait_sleep(&sm.bar_k_empty[st], ((t >> 1) - 1) & 1);
        mbar_expect_tx_w(&sm.bar_k_full[st], kTileBytes, leader);
        tma_load_3d_w(&tm_k, &sm.bar_k_full[st], sm.k[st], 0, hkv, krow, leader);
        tma_load_3d_w(&tm_k, &sm.bar_k_full[st], sm.k[st] + kTileBytes / 2, 64, hkv, krow, leader);
        if (t >= 2) mbar_wait_sleep(&sm.bar_v_empty[st], ((t >> 1) - 1) & 1);
        mbar_expect_tx_w(&sm.bar_v_full[st], kTileBytes, leader);
        tma_load_3d_w(&tm_v, &sm.bar_v_full[st], sm.v[st], 0, hkv, krow, leader);
        tma_load_3d_w(&tm_v, &sm.bar_v_full[st], sm.v[st] + kTileBytes / 2, 64, hkv, krow, leader);
      }
#ifdef BAM_CTA_CLOCK
      if (leader) BAM_CTA_CLOCK_FLAG_WAIT(flag_wait_ns);
#endif
    }
  } else if (warp == kWarpMma) {
    const uint32_t leader = elect_one();
    if (n > 0) {
      const uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
      const uint32_t idesc_o = idesc_bf16(128, 128, 0, 1);
      const uint64_t dq0 = sdesc_sw128(smem_u32(sm.q[0]), 16, 1024);
      const uint64_t dk0 = sdesc_sw128(smem_u32(sm.k[0]), 16, 1024);
      const uint64_t dv0 = sdesc_sw128(smem_u32(sm.v[0]), kTileBytes / 2, 1024);
      constexpr uint32_t kTile16 = kTileBytes >> 4;
      auto issue_s = [&](int i, int t) {
        const uint64_t dq = dq0 + i * kTile16, dk = dk0 + (t & 1) * kTile16;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * (kTileBytes / 2) + (kk & 3) * 32) >> 4;
          mma_ss_w(tmem + 128 * i, dq + off, dk + off, idesc_s, kk > 0, leader);
        }
        tc_commit_w(&sm.bar_s_full[i], leader);
      };
      // PV(t) of head i in kPChunks parts as the softmax releases the P chunks: chunk c
      // covers the 16-key MMA steps kk = hf 4 + c (4 / kPChunks) + u of both thread
      // halves hf
      auto issue_pv = [&](int i, int t) {
        const uint64_t dv = dv0 + (t & 1) * kTile16;
        constexpr int kKPer = 4 / kPChunks;
#pragma unroll
        for (int c = 0; c < kPChunks; ++c) {
          mbar_wait(&sm.bar_p_ready[i][c], t & 1);
          tc_fence_after();
#pragma unroll
          for (int u = 0; u < 2 * kKPer; ++u) {
            const int kk = (u / kKPer) * 4 + c * kKPer + u % kKPer;
            mma_ts_w(tmem + 256 + 128 * i, tmem + 128 * i + kk * 8, dv + kk * 128, idesc_o,
                     (t > 0 || c > 0 || u > 0), leader);
          }
        }
        tc_commit_w(&sm.bar_pv_done[i], leader);
      };
      mbar_wait(&sm.bar_q, 0);
      mbar_wait(&sm.bar_k_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      tc_commit_w(&sm.bar_k_empty[0], leader);
      for (int t = 0; t < n; ++t) {
        const int st = t & 1, st1 = (t + 1) & 1;
        mbar_wait(&sm.bar_v_full[st], (t >> 1) & 1);
        issue_pv(0, t);
        if (t + 1 < n) {
          mbar_wait(&sm.bar_k_full[st1], ((t + 1) >> 1) & 1);
          tc_fence_after();
          issue_s(0, t + 1);
        }
        issue_pv(1, t);
        tc_commit_w(&sm.bar_v_empty[st], leader);
        if (t + 1 < n) {
          issue_s(1, t + 1);
          tc_commit_w(&sm.bar_k_empty[st1], leader);
        }
      }
    }
  } else {
    const int i = warp >> 3;  // head: warps 0-7 / 8-15
    const uint32_t lw = warp & 7;
    softmax_half_role<BAM_FWD_POLY_SPLIT>(p, tmem, 128 * i, 256 + 128 * i, &sm.bar_s_full[i],
                                          sm.bar_p_ready[i], &sm.bar_pv_done[i], jj[i], hh[i],
                                          lw, lane, tl[i], n, slot, sm.xch[i],
                                          1 + i * 4 + (lw & 3));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  BAM_CTA_CLOCK_END(n);
}

// ---------------------------------------------------------------------------
// CTA-pair (cta_group::2) head-pair kernel: a cluster of two CTAs = two query
// blocks whose key-tile lists are (nearly) the same (the union list of a
// "shared" pair from bam_build_pair_lists; a tile only one of them sees is
// class 0 = fully masked for the other) x two query heads.  The even CTA
// issues M = 256 MMAs: Q rows come from each CTA's own shared memory, K / V
// are split by N -- each CTA loads 64 keys of K and 64 head-dim columns of V
// per tile, half of the one-CTA kernel's K/V traffic, and each SM's shared
// memory feeds 160 KB per key tile instead of 256 KB (tensor time 2048 clk).
// Softmax / epilogue are the one-CTA kernel's, per CTA on its own TMEM rows.
constexpr int k2Stages = 3;
constexpr uint32_t kHalfTile = kTileBytes / 2;   // 64 keys x 128 d, or 128 keys x 64 d

struct Pair2Smem {
  alignas(1024) uint8_t q[2][kTileBytes];
  alignas(1024) uint8_t k[k2Stages][kHalfTile];  // this CTA's 64 keys: two 64-col boxes of 8 KB
  alignas(1024) uint8_t v[k2Stages][kHalfTile];  // this CTA's 64 d-columns of all 128 keys
  uint64_t bar_q, bar_k_full[k2Stages], bar_k_empty[k2Stages], bar_v_full[k2Stages],
      bar_v_empty[k2Stages];
  uint64_t bar_s_full[2], bar_p_ready[2], bar_pv_done[2];
  uint32_t tmem_base;
};

__global__ void __maxnreg__(168)
    attn_fwd_2cta_kernel(const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_k64,
                         const __grid_constant__ CUtensorMap tm_v, const BamAttnFwdParams p,
                         const int32_t* __restrict__ pair_ids, const int32_t* __restrict__ slot_q,
                         const int32_t* __restrict__ slot_off,
                         const int32_t* __restrict__ slot_tiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Pair2Smem& sm = *reinterpret_cast<Pair2Smem*>(smem_raw);
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t crank = cluster_ctarank();
  const int nh = p.nh > 0 ? p.nh : p.Hq;
  const int h0 = p.h_begin + 2 * blockIdx.y;
  if (p.dev_counts && (int)(blockIdx.x >> 1) >= p.dev_counts[0]) return;  // both CTAs of the pair
  const int slot = 2 * pair_ids[blockIdx.x >> 1] + (int)crank;
  const int j = slot_q[slot];
  const int32_t* tiles = slot_tiles + slot_off[slot];
  const int n = slot_off[slot + 1] - slot_off[slot];  // equal in both CTAs (union list)
  const int hkv = (h0 - p.h_begin) / (nh / p.Hkv);

  if (threadIdx.x == 0) {
    if ((smem_u32(smem_raw) & 1023) != 0) __trap();
    mbar_init(&sm.bar_q, 1);
    for (int i = 0; i < k2Stages; ++i) {
      mbar_init(&sm.bar_k_full[i], 1);
      mbar_init(&sm.bar_k_empty[i], 1);
      mbar_init(&sm.bar_v_full[i], 1);
      mbar_init(&sm.bar_v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.bar_s_full[i], 1);
      mbar_init(&sm.bar_p_ready[i], 128 + 4);  // own warpgroup i per thread + the peer's per warp
      mbar_init(&sm.bar_pv_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 9) {
    tmem_alloc_2cta(&sm.tmem_base, 512);
    tmem_relinquish_2cta();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    const uint32_t leader = elect_one();
    if (n > 0) {
      if (leader) {
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k64);
        prefetch_tmap(&tm_v);
      }
      if (crank == 0) mbar_expect_tx_w(&sm.bar_q, 4 * kTileBytes, leader);
      const uint32_t lbar_q = mapa_shared(smem_u32(&sm.bar_q), 0);
      for (int i = 0; i < 2; ++i) {
        tma_load_3d_2cta_w(&tm_q, lbar_q, sm.q[i], 0, h0 + i, j * 128, leader);
        tma_load_3d_2cta_w(&tm_q, lbar_q, sm.q[i] + kTileBytes / 2, 64, h0 + i, j * 128, leader);
      }
      for (int t = 0; t < n; ++t) {
        const int st = t % k2Stages;
        const int krow = p.k_row[tiles[t] >> 2] * 128;
        if (t >= k2Stages) mbar_wait_sleep(&sm.bar_k_empty[st], ((t / k2Stages) - 1) & 1);
        if (crank == 0) mbar_expect_tx_w(&sm.bar_k_full[st], 2 * kHalfTile, leader);
        const uint32_t lbar_k = mapa_shared(smem_u32(&sm.bar_k_full[st]), 0);
        tma_load_3d_2cta_w(&tm_k64, lbar_k, sm.k[st], 0, hkv, krow + 64 * (int)crank, leader);
        tma_load_3d_2cta_w(&tm_k64, lbar_k, sm.k[st] + kHalfTile / 2, 64, hkv,
                           krow + 64 * (int)crank, leader);
        if (t >= k2Stages) mbar_wait_sleep(&sm.bar_v_empty[st], ((t / k2Stages) - 1) & 1);
        if (crank == 0) mbar_expect_tx_w(&sm.bar_v_full[st], 2 * kHalfTile, leader);
        tma_load_3d_2cta_w(&tm_v, mapa_shared(smem_u32(&sm.bar_v_full[st]), 0), sm.v[st],
                           64 * (int)crank, hkv, krow, leader);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer (even CTA)
    const uint32_t leader = elect_one() && crank == 0;
    if (n > 0 && crank == 0) {
      const uint32_t idesc_s = idesc_bf16(256, 128, 0, 0);
      const uint32_t idesc_o = idesc_bf16(256, 128, 0, 1);
      const uint64_t dq0 = sdesc_sw128(smem_u32(sm.q[0]), 16, 1024);
      const uint64_t dk0 = sdesc_sw128(smem_u32(sm.k[0]), 16, 1024);
      const uint64_t dv0 = sdesc_sw128(smem_u32(sm.v[0]), 16, 1024);
      constexpr uint32_t kTile16 = kTileBytes >> 4, kHalf16 = kHalfTile >> 4;
      auto issue_s = [&](int i, int t) {  // S_i(t) = Q_i K(t)^T, M = 256 over the pair
        const uint64_t dq = dq0 + i * kTile16, dk = dk0 + (t % k2Stages) * kHalf16;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t oq = ((kk >> 2) * (kTileBytes / 2) + (kk & 3) * 32) >> 4;
          const uint32_t ok = ((kk >> 2) * (kHalfTile / 2) + (kk & 3) * 32) >> 4;
          mma_ss_2cta_w(tmem + 128 * i, dq + oq, dk + ok, idesc_s, kk > 0, leader);
        }
        tc_commit_2cta_mc_w(&sm.bar_s_full[i], 0x3, leader);
      };
      auto issue_pv = [&](int i, int t) {  // O_i += P_i(t) V(t), P_i bf16 in the S_i columns
        const uint64_t dv = dv0 + (t % k2Stages) * kHalf16;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts_2cta_w(tmem + 256 + 128 * i, tmem + 128 * i + kk * 8, dv + kk * 128, idesc_o,
                        (t > 0 || kk > 0), leader);
        tc_commit_2cta_mc_w(&sm.bar_pv_done[i], 0x3, leader);
      };
      mbar_wait(&sm.bar_q, 0);
      mbar_wait(&sm.bar_k_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      tc_commit_2cta_mc_w(&sm.bar_k_empty[0], 0x3, leader);
      for (int t = 0; t < n; ++t) {
        const int st = t % k2Stages, st1 = (t + 1) % k2Stages;
        mbar_wait(&sm.bar_p_ready[0], t & 1);
        mbar_wait(&sm.bar_v_full[st], (t / k2Stages) & 1);
        tc_fence_after();
        issue_pv(0, t);
        if (t + 1 < n) {
          mbar_wait(&sm.bar_k_full[st1], ((t + 1) / k2Stages) & 1);
          tc_fence_after();
          issue_s(0, t + 1);
        }
        mbar_wait(&sm.bar_p_ready[1], t & 1);
        tc_fence_after();
        issue_pv(1, t);
        tc_commit_2cta_mc_w(&sm.bar_v_empty[st], 0x3, leader);
        if (t + 1 < n) {
          issue_s(1, t + 1);
          tc_commit_2cta_mc_w(&sm.bar_k_empty[st1], 0x3, leader);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warpgroups
    const int i = warp >> 2;
    const uint32_t p_ready_remote =
        crank == 0 ? 0u : mapa_shared(smem_u32(&sm.bar_p_ready[i]), 0);
    softmax_role<BAM_FWD_POLY_PAIR>(p, tmem, 128 * i, 256 + 128 * i, &sm.bar_s_full[i],
                                    &sm.bar_p_ready[i], &sm.bar_pv_done[i], j, h0 + i, warp, lane,
                                    tiles, n, -1, p_ready_remote);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the leader's MMAs into this CTA's TMEM are complete
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc_2cta(tmem, 512);
  }
}

// Aggregation kernel: merge the split-KV subblock partials
// of a query block; one CTA per (combine record, head), thread = row.
__global__ void __launch_bounds__(128) combine_kernel(const BamAttnFwdParams p,
                                                      const int4* __restrict__ combine) {
  const int4 c = combine[blockIdx.x];
  const int nh = p.nh > 0 ? p.nh : p.Hq;
  const int h = p.h_begin + blockIdx.y;
  if (blockIdx.y >= nh) return;
  const int r = threadIdx.x;
  const float2* ml = reinterpret_cast<const float2*>(p.part_ml);
  float M = -INFINITY;
  for (int q = 0; q < c.z; ++q) M = fmaxf(M, ml[((int64_t)(c.y + q) * p.Hq + h) * 128 + r].x);
  const float mb = M == -INFINITY ? 0.f : M;
  float L = 0.f;
  float acc[128];
#pragma unroll
  for (int d = 0; d < 128; ++d) acc[d] = 0.f;
  for (int q = 0; q < c.z; ++q) {
    const int64_t base = ((int64_t)(c.y + q) * p.Hq + h) * 128 + r;
    const float2 v = ml[base];
    const float w = ex2(v.x - mb);
    L += w * v.y;
    const float4* po = reinterpret_cast<const float4*>(p.part_o + base * 128);
#pragma unroll
    for (int d4 = 0; d4 < 32; ++d4) {
      const float4 o = po[d4];
      acc[4 * d4] = fmaf(w, o.x, acc[4 * d4]);
      acc[4 * d4 + 1] = fmaf(w, o.y, acc[4 * d4 + 1]);
      acc[4 * d4 + 2] = fmaf(w, o.z, acc[4 * d4 + 2]);
      acc[4 * d4 + 3] = fmaf(w, o.w, acc[4 * d4 + 3]);
    }
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  const int64_t row = (int64_t)c.x * 128 + r;
  uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o) +
                                        (row * p.Hq + h) * 128);
#pragma unroll
  for (int i = 0; i < 16; ++i)
    dst[i] = make_uint4(pack_bf16(acc[8 * i] * inv, acc[8 * i + 1] * inv),
                        pack_bf16(acc[8 * i + 2] * inv, acc[8 * i + 3] * inv),
                        pack_bf16(acc[8 * i + 4] * inv, acc[8 * i + 5] * inv),
                        pack_bf16(acc[8 * i + 6] * inv, acc[8 * i + 7] * inv));
  p.lse[(int64_t)h * p.nq * 128 + row] =
      L > 0.f ? (M + __log2f(L)) * 0.6931471805599453f : -INFINITY;
}

}  // namespace fwd

// bam_set_cta_clock_buffer's forward half (this translation unit's symbol)
int fwd_set_cta_clock(void* buf) {
#ifdef BAM_CTA_CLOCK
  BAM_CUDA_TRY(cudaMemcpyToSymbol(g_bam_cta_clock, &buf, sizeof(buf)));
  return kOk;
#else
  (void)buf;
  set_last_error("libbam built without -DBAM_CTA_CLOCK");
  return BAM_UNSUPPORTED;
#endif
}

}  // namespace bam

using namespace bam;

// CP-overlap flags: ``ready`` is a 64-bit per-rank mask in the kernels and the owner
// of a block-row is k_row / kv_rows_per_rank (validate both on the host)
#define BAM_CHECK_KV_READY(p, fn)                                                          \
  BAM_CHECK_ARG(!(p).kv_ready ||                                                           \
                    ((p).kv_rows_per_rank >= 1 &&                                          \
                     ((p).k_rows + (p).kv_rows_per_rank - 1) / (p).kv_rows_per_rank <= 64 && \
                     (p).kv_rank >= 0 && (p).kv_rank < 64 && (p).kv_flag_heads >= 0 &&     \
                     ((p).kv_flag_heads <= 1 || (p).Hkv % (p).kv_flag_heads == 0)),         \
                fn ": kv_ready needs kv_rows_per_rank >= 1 and at most 64 ranks "          \
                   "(kv_rows_per_rank=%d k_rows=%d kv_rank=%d)",                           \
                (p).kv_rows_per_rank, (p).k_rows, (p).kv_rank)

extern "C" int bam_attn_fwd_combine(const BamAttnFwdParams* pp, const int32_t* combine,
                                    int32_t n_combine, void* stream) {
  BAM_CHECK_ARG(pp != nullptr && combine != nullptr && n_combine >= 0,
                "bam_attn_fwd_combine: bad arguments");
  if (n_combine == 0) return kOk;
  const int nh = pp->nh > 0 ? pp->nh : pp->Hq;
  fwd::combine_kernel<<<dim3(n_combine, nh), 128, 0, (cudaStream_t)stream>>>(
      *pp, reinterpret_cast<const int4*>(combine));
  BAM_LAUNCH_CHECK();
  return kOk;
}

extern "C" int bam_attn_fwd(const BamAttnFwdParams* pp, void* stream) {
  BAM_CHECK_ARG(pp != nullptr, "bam_attn_fwd: null params");
  const BamAttnFwdParams& p = *pp;
  BAM_CHECK_ARG(p.nq >= 1 && p.nb >= 1 && p.k_rows >= 1, "bam_attn_fwd: nq=%d nb=%d k_rows=%d",
                p.nq, p.nb, p.k_rows);
  const int nh = p.nh > 0 ? p.nh : p.Hq;
  BAM_CHECK_ARG(p.Hq >= 1 && p.Hkv >= 1 && nh % p.Hkv == 0 && p.h_begin >= 0 &&
                    p.h_begin + nh <= p.Hq,
                "bam_attn_fwd: head group [%d, %d) of Hq=%d over Hkv=%d", p.h_begin,
                p.h_begin + nh, p.Hq, p.Hkv);
  BAM_CHECK_ARG(p.nq <= 65535, "bam_attn_fwd: nq=%d > 65535", p.nq);
  BAM_CHECK_KV_READY(p, "bam_attn_fwd");
  BAM_CHECK_ARG(!p.kv_ready || !p.part_o, "bam_attn_fwd: kv_ready needs whole rows");
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = make_tmap_rows_heads_d128(&mq, p.q, (int64_t)p.nq * 128, p.Hq, 128))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mk, p.k, (int64_t)p.k_rows * 128, p.Hkv, 128,
                                      p.kv_head_major)))
    return rc;
  if ((rc = make_tmap_rows_heads_d128(&mv, p.v, (int64_t)p.k_rows * 128, p.Hkv, 128,
                                      p.kv_head_major)))
    return rc;
  const int grp = nh / p.Hkv;
  if (grp % 2 == 0) {  // GQA head pairs, split-row softmax
    const int smem = (int)sizeof(fwd::SplitSmem);
    BAM_CUDA_TRY(cudaFuncSetAttribute(fwd::attn_fwd_split_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int rows = p.items ? p.n_items : p.nq;
    const dim3 grid = fwd::kRowMajor ? dim3(rows, nh / 2) : dim3(nh / 2, rows);
    fwd::attn_fwd_split_kernel<false><<<grid, fwd::kSplitThreads, smem, (cudaStream_t)stream>>>(
        mq, mk, mv, p, nullptr, nullptr, nullptr, nullptr);
  } else {
    const int smem = (int)sizeof(fwd::Smem) + 1024;
    BAM_CUDA_TRY(cudaFuncSetAttribute(fwd::attn_fwd_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int rows = p.items ? p.n_items : p.nq;
    const dim3 grid = fwd::kRowMajor ? dim3(rows, nh) : dim3(nh, rows);
    fwd::attn_fwd_kernel<<<grid, fwd::kThreads, smem, (cudaStream_t)stream>>>(mq, mk, mv, p);
  }
  BAM_LAUNCH_CHECK();
  return kOk;
}

extern "C" int bam_attn_fwd_2cta(const BamAttnFwdParams* pp, const int32_t* pair_ids,
                                 int32_t n_pairs, const int32_t* slot_q, const int32_t* slot_off,
                                 const int32_t* slot_tiles, void* stream) {
  BAM_CHECK_ARG(pp != nullptr && pair_ids && slot_q && slot_off && slot_tiles,
                "bam_attn_fwd_2cta: null argument");
  const BamAttnFwdParams& p = *pp;
  const int nh = p.nh > 0 ? p.nh : p.Hq;
  BAM_CHECK_ARG(p.nq >= 1 && p.k_rows >= 1 && p.Hkv >= 1 && nh % p.Hkv == 0 &&
                    (nh / p.Hkv) % 2 == 0 && p.h_begin >= 0 && p.h_begin + nh <= p.Hq,
                "bam_attn_fwd_2cta: needs an even GQA group (nh=%d Hkv=%d)", nh, p.Hkv);
  BAM_CHECK_ARG(n_pairs >= 0, "bam_attn_fwd_2cta: n_pairs=%d", n_pairs);
  BAM_CHECK_ARG(!p.kv_ready, "bam_attn_fwd_2cta: the CTA-pair kernel does not wait on kv_ready");
  if (n_pairs == 0) return kOk;
  CUtensorMap mq, mk64, mv;
  int rc;
  if ((rc = make_tmap_rows_heads_d128(&mq, p.q, (int64_t)p.nq * 128, p.Hq, 128))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mk64, p.k, (int64_t)p.k_rows * 128, p.Hkv, 64,
                                      p.kv_head_major)))
    return rc;
  if ((rc = make_tmap_rows_heads_d128(&mv, p.v, (int64_t)p.k_rows * 128, p.Hkv, 128,
                                      p.kv_head_major)))
    return rc;
  const int smem = (int)sizeof(fwd::Pair2Smem);
  BAM_CUDA_TRY(cudaFuncSetAttribute(fwd::attn_fwd_2cta_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * n_pairs, nh / 2);
  cfg.blockDim = dim3(fwd::kPairThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BAM_CUDA_TRY(cudaLaunchKernelEx(&cfg, fwd::attn_fwd_2cta_kernel, mq, mk64, mv, p, pair_ids,
                                  slot_q, slot_off, slot_tiles));
  BAM_LAUNCH_CHECK();
  return kOk;
}

extern "C" int bam_attn_fwd_qpairs(const BamAttnFwdParams* pp, const int32_t* pair_ids,
                                   int32_t n_pairs, const int32_t* slot_q, const int32_t* slot_off,
                                   const int32_t* slot_tiles, void* stream) {
  BAM_CHECK_ARG(pp != nullptr && pair_ids && slot_q && slot_off && slot_tiles,
                "bam_attn_fwd_qpairs: null argument");
  const BamAttnFwdParams& p = *pp;
  const int nh = p.nh > 0 ? p.nh : p.Hq;
  BAM_CHECK_ARG(p.nq >= 1 && p.k_rows >= 1 && p.Hkv >= 1 && nh % p.Hkv == 0 && p.h_begin >= 0 &&
                    p.h_begin + nh <= p.Hq,
                "bam_attn_fwd_qpairs: head group [%d, %d) of Hq=%d over Hkv=%d", p.h_begin,
                p.h_begin + nh, p.Hq, p.Hkv);
  BAM_CHECK_ARG(n_pairs >= 0, "bam_attn_fwd_qpairs: n_pairs=%d", n_pairs);
  BAM_CHECK_KV_READY(p, "bam_attn_fwd_qpairs");
  if (n_pairs == 0) return kOk;
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = make_tmap_rows_heads_d128(&mq, p.q, (int64_t)p.nq * 128, p.Hq, 128))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mk, p.k, (int64_t)p.k_rows * 128, p.Hkv, 128,
                                      p.kv_head_major)))
    return rc;
  if ((rc = make_tmap_rows_heads_d128(&mv, p.v, (int64_t)p.k_rows * 128, p.Hkv, 128,
                                      p.kv_head_major)))
    return rc;
  const int smem = (int)sizeof(fwd::SplitSmem);
  BAM_CUDA_TRY(cudaFuncSetAttribute(fwd::attn_fwd_split_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const dim3 grid = fwd::kRowMajor ? dim3(n_pairs, nh) : dim3(nh, n_pairs);
  fwd::attn_fwd_split_kernel<true><<<grid, fwd::kSplitThreads, smem, (cudaStream_t)stream>>>(
      mq, mk, mv, p, pair_ids, slot_q, slot_off, slot_tiles);
  BAM_LAUNCH_CHECK();
  return kOk;
}
