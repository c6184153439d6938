// Bitfield-masked attention backward for sm_100a (tcgen05 + TMEM + TMA).
//
// FlashAttention-style backward parallel over key blocks: one CTA owns one
// 128-key block x one KV head and walks the CSC list of local query blocks
// that see it (non-skip tiles only; PARTIAL tiles re-evaluate the descriptor
// predicate of mask.py:106-112 in registers), for every query head of the
// GQA group.  Per step (query block j, query head h):
//   S^T  = K Q^T            (SS)  -> TMEM [0,128)     P^T = exp(S^T*scale - LSE)
//   dP^T = V dO^T           (SS)  -> TMEM [128,256)   dS^T = P^T (dP^T - D)
//   dQ   = dS K             (SS, both MN-major) -> TMEM [128,256) -> red.add fp32
//   dV  += P^T dO           (TS: P^T bf16 in TMEM [0,64), dO MN-major) -> [256,384)
//   dK  += dS^T Q           (SS: dS^T smem K-major, Q MN-major)        -> [384,512)
// Warp roles (320 threads, 1 CTA / SM):
//   warps 0-3 compute (thread r = key row r), warps 4-7 dQ epilogue
//   (thread r = query row r), warp 8 TMA producer, warp 9 TMEM alloc + MMA.
#include "../../include/bam.h"
#include "common.cuh"
#include "tma.h"

namespace bam {
namespace bwd {

constexpr int kThreads = 320;
constexpr uint32_t kTileBytes = 128 * 128 * 2;
constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 384;

struct Smem {
  alignas(1024) uint8_t k[kTileBytes];
  alignas(1024) uint8_t v[kTileBytes];
  alignas(1024) uint8_t q[2][kTileBytes];
  alignas(1024) uint8_t dout[2][kTileBytes];
  alignas(1024) uint8_t ds[kTileBytes];
  uint64_t bar_kv, bar_in_full[2], bar_in_empty[2];
  uint64_t bar_sdp_full, bar_p_ready, bar_mma_done, bar_dq_full, bar_dq_empty;
  uint32_t tmem_base;
};

__device__ __forceinline__ void load_tile(const CUtensorMap* m, uint64_t* bar, uint8_t* dst,
                                          int head, int row0) {
  tma_load_3d(m, bar, dst, 0, head, row0);
  tma_load_3d(m, bar, dst + kTileBytes / 2, 64, head, row0);
}

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const BamAttnBwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  const uint32_t warp = warp_id(), lane = lane_id();
  const int hkv = blockIdx.x;
  const int kb = p.order ? p.order[blockIdx.y] : (int)blockIdx.y;
  const int grp = p.Hq / p.Hkv;
  const int c0 = p.col_off[kb], ncol = p.col_off[kb + 1] - c0;
  const int32_t* col = p.col_tiles + c0;
  const int nsteps = ncol * grp;
  const int64_t Tq = (int64_t)p.nq * 128;
  const int krow0 = p.k_row[kb] * 128;

  if (threadIdx.x == 0) {
    mbar_init(&sm.bar_kv, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.bar_in_full[i], 1);
      mbar_init(&sm.bar_in_empty[i], 1);
    }
    mbar_init(&sm.bar_sdp_full, 1);
    mbar_init(&sm.bar_p_ready, 128);
    mbar_init(&sm.bar_mma_done, 1);
    mbar_init(&sm.bar_dq_full, 1);
    mbar_init(&sm.bar_dq_empty, 128);
    fence_mbar_init();
  }
  if (warp == 9) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && nsteps > 0) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_k);
      prefetch_tmap(&tm_v);
      prefetch_tmap(&tm_do);
      mbar_expect_tx(&sm.bar_kv, 2 * kTileBytes);
      load_tile(&tm_k, &sm.bar_kv, sm.k, hkv, krow0);
      load_tile(&tm_v, &sm.bar_kv, sm.v, hkv, krow0);
      for (int s = 0; s < nsteps; ++s) {
        const int st = s & 1;
        const int h = hkv * grp + s / ncol;
        const int jq = col[s % ncol] >> 2;
        if (s >= 2) mbar_wait(&sm.bar_in_empty[st], ((s >> 1) - 1) & 1);
        mbar_expect_tx(&sm.bar_in_full[st], 2 * kTileBytes);
        load_tile(&tm_q, &sm.bar_in_full[st], sm.q[st], h, jq * 128);
        load_tile(&tm_do, &sm.bar_in_full[st], sm.dout[st], h, jq * 128);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && nsteps > 0) {
      const uint32_t id_kk = idesc_bf16(128, 128, 0, 0);   // K-major A, K-major B
      const uint32_t id_kmn = idesc_bf16(128, 128, 0, 1);  // K-major A (or TMEM), MN-major B
      const uint32_t id_mnmn = idesc_bf16(128, 128, 1, 1); // MN-major A and B
      const uint32_t sk = smem_u32(sm.k), sv = smem_u32(sm.v), sds = smem_u32(sm.ds);
      mbar_wait(&sm.bar_kv, 0);
      for (int s = 0; s < nsteps; ++s) {
        const int st = s & 1;
        const uint32_t sq = smem_u32(sm.q[st]), sdo = smem_u32(sm.dout[st]);
        mbar_wait(&sm.bar_in_full[st], (s >> 1) & 1);
        if (s > 0) mbar_wait(&sm.bar_mma_done, (s - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * (kTileBytes / 2) + (kk & 3) * 32;
          mma_ss(tmem + kColS, sdesc_sw128(sk + off, 16, 1024), sdesc_sw128(sq + off, 16, 1024),
                 id_kk, kk > 0);
        }
        if (s > 0) mbar_wait(&sm.bar_dq_empty, (s - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * (kTileBytes / 2) + (kk & 3) * 32;
          mma_ss(tmem + kColDP, sdesc_sw128(sv + off, 16, 1024), sdesc_sw128(sdo + off, 16, 1024),
                 id_kk, kk > 0);
        }
        tc_commit(&sm.bar_sdp_full);
        mbar_wait(&sm.bar_p_ready, s & 1);
        tc_fence_after();
        // dQ = dS K  (A = dS^T smem viewed MN-major, B = K MN-major)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem + kColDP, sdesc_sw128(sds + kk * 2048, kTileBytes / 2, 1024),
                 sdesc_sw128(sk + kk * 2048, kTileBytes / 2, 1024), id_mnmn, kk > 0);
        tc_commit(&sm.bar_dq_full);
        // dV += P^T dO  (A = P^T in TMEM, B = dO MN-major)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tmem + kColDV, tmem + kColS + kk * 8,
                 sdesc_sw128(sdo + kk * 2048, kTileBytes / 2, 1024), id_kmn, (s > 0 || kk > 0));
        // dK += dS^T Q  (A = dS^T smem K-major, B = Q MN-major)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * (kTileBytes / 2) + (kk & 3) * 32;
          mma_ss(tmem + kColDK, sdesc_sw128(sds + off, 16, 1024),
                 sdesc_sw128(sq + kk * 2048, kTileBytes / 2, 1024), id_kmn, (s > 0 || kk > 0));
        }
        tc_commit(&sm.bar_in_empty[st]);
        tc_commit(&sm.bar_mma_done);
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ compute warps 0-3
    const int r = warp * 32 + lane;
    const uint32_t lane_base = (warp * 32) << 16;
    const long long kg = (long long)kb * 128 + r;
    const long long dk = p.desc[kg];
    const float scale_log2 = p.scale * 1.4426950408889634f;
    const float log2e = 1.4426950408889634f;
    const uint32_t ds_row = smem_u32(sm.ds) + r * 128;
    for (int s = 0; s < nsteps; ++s) {
      const int h = hkv * grp + s / ncol;
      const int e = col[s % ncol];
      const int jq = e >> 2, cls = e & 3;
      const long long qg0 = (long long)p.q_gid[jq] * 128;
      const float* lse = p.lse + (int64_t)h * Tq + (int64_t)jq * 128;
      const float* dlt = p.delta + (int64_t)h * Tq + (int64_t)jq * 128;
      mbar_wait(&sm.bar_sdp_full, s & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sr[32], dr[32];
        BAM_TMEM_LD32(tmem + lane_base + kColS + c * 32, sr);
        BAM_TMEM_LD32(tmem + lane_base + kColDP + c * 32, dr);
        tmem_wait_ld();
        uint32_t pk[16], dsk[16];
#pragma unroll
        for (int i4 = 0; i4 < 8; ++i4) {
          const float4 l4 = __ldg(reinterpret_cast<const float4*>(lse + c * 32) + i4);
          const float4 d4 = __ldg(reinterpret_cast<const float4*>(dlt + c * 32) + i4);
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
          const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
          float pv[4], dsv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i4 * 4 + u;
            float pp = ex2(fmaf(__uint_as_float(sr[i]), scale_log2, -lv[u] * log2e));
            if (cls == 2) {
              const long long qg = qg0 + c * 32 + i;
              if (!bam_allowed(__ldg(p.desc + qg), qg, dk, kg)) pp = 0.f;
            }
            pv[u] = pp;
            dsv[u] = pp * (__uint_as_float(dr[i]) - dv[u]);
          }
          pk[i4 * 2] = pack_bf16(pv[0], pv[1]);
          pk[i4 * 2 + 1] = pack_bf16(pv[2], pv[3]);
          dsk[i4 * 2] = pack_bf16(dsv[0], dsv[1]);
          dsk[i4 * 2 + 1] = pack_bf16(dsv[2], dsv[3]);
        }
        BAM_TMEM_ST16(tmem + lane_base + kColS + c * 16, pk);
        // dS^T row r, columns 32c .. 32c+31: four 16-B chunks, 128-B swizzle
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t colq = c * 32 + q4 * 8;
          const uint32_t box = colq >> 6;
          const uint32_t chunk = ((colq & 63) >> 3) ^ (r & 7);
          const uint32_t addr = ds_row + box * (kTileBytes / 2) + chunk * 16;
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(dsk[q4 * 4]),
                       "r"(dsk[q4 * 4 + 1]), "r"(dsk[q4 * 4 + 2]), "r"(dsk[q4 * 4 + 3])
                       : "memory");
        }
      }
      tmem_wait_st();
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&sm.bar_p_ready);
    }
    // epilogue: dV, dK (scaled) -> fp32 rows of the key block
    const int64_t row = (int64_t)krow0 + r;
    float* dvrow = p.dv + (row * p.Hkv + hkv) * 128;
    float* dkrow = p.dk + (row * p.Hkv + hkv) * 128;
    if (nsteps > 0) {
      mbar_wait(&sm.bar_mma_done, (nsteps - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t a[32], b[32];
        BAM_TMEM_LD32(tmem + lane_base + kColDV + c * 32, a);
        BAM_TMEM_LD32(tmem + lane_base + kColDK + c * 32, b);
        tmem_wait_ld();
        float4* dv4 = reinterpret_cast<float4*>(dvrow + c * 32);
        float4* dk4 = reinterpret_cast<float4*>(dkrow + c * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          dv4[i] = make_float4(__uint_as_float(a[4 * i]), __uint_as_float(a[4 * i + 1]),
                               __uint_as_float(a[4 * i + 2]), __uint_as_float(a[4 * i + 3]));
          dk4[i] = make_float4(__uint_as_float(b[4 * i]) * p.scale, __uint_as_float(b[4 * i + 1]) * p.scale,
                               __uint_as_float(b[4 * i + 2]) * p.scale, __uint_as_float(b[4 * i + 3]) * p.scale);
        }
      }
    } else {
      float4* dv4 = reinterpret_cast<float4*>(dvrow);
      float4* dk4 = reinterpret_cast<float4*>(dkrow);
      for (int i = 0; i < 32; ++i) {
        dv4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        dk4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  } else {
    // ------------------------------------------------------------ dQ epilogue warps 4-7
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lane_base = ((warp - 4) * 32) << 16;
    for (int s = 0; s < nsteps; ++s) {
      const int h = hkv * grp + s / ncol;
      const int jq = col[s % ncol] >> 2;
      float* dst = p.dq_acc + (((int64_t)jq * 128 + r) * p.Hq + h) * 128;
      mbar_wait(&sm.bar_dq_full, s & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t a[32];
        BAM_TMEM_LD32(tmem + lane_base + kColDP + c * 32, a);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          red_add_v4(dst + c * 32 + 4 * i, __uint_as_float(a[4 * i]), __uint_as_float(a[4 * i + 1]),
                     __uint_as_float(a[4 * i + 2]), __uint_as_float(a[4 * i + 3]));
      }
      tc_fence_before();
      mbar_arrive(&sm.bar_dq_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// delta[h, row] = sum_d dO[row, h, d] * O[row, h, d]   (one warp per (row, h))
__global__ void bwd_delta_kernel(const __nv_bfloat16* __restrict__ o,
                                 const __nv_bfloat16* __restrict__ dout, int64_t rows, int H,
                                 float* __restrict__ delta) {
  const int64_t nw = rows * H;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint2 a = reinterpret_cast<const uint2*>(o + w * 128)[lane_id()];
    const uint2 b = reinterpret_cast<const uint2*>(dout + w * 128)[lane_id()];
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(b2[i]);
      acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
    }
    for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane_id() == 0) {
      const int64_t row = w / H, h = w % H;
      delta[h * rows + row] = acc;
    }
  }
}

// dq (bf16) = dq_acc * scale
__global__ void bwd_dq_convert_kernel(const float4* __restrict__ acc, uint2* __restrict__ dq,
                                      int64_t n4, float scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = acc[i];
    dq[i] = make_uint2(pack_bf16(v.x * scale, v.y * scale), pack_bf16(v.z * scale, v.w * scale));
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
  BAM_CHECK_ARG(p.Hq >= 1 && p.Hkv >= 1 && p.Hq % p.Hkv == 0,
                "bam_attn_bwd: Hq=%d must be a multiple of Hkv=%d", p.Hq, p.Hkv);
  BAM_CHECK_ARG(p.nb <= 65535, "bam_attn_bwd: nb=%d > 65535", p.nb);
  return kOk;
}

extern "C" {

int bam_attn_bwd_preprocess(const BamAttnBwdParams* pp, void* stream) {
  if (int rc = check_bwd(pp)) return rc;
  const BamAttnBwdParams& p = *pp;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rows = (int64_t)p.nq * 128;
  bwd::bwd_delta_kernel<<<148 * 8, 256, 0, s>>>((const __nv_bfloat16*)p.o,
                                                (const __nv_bfloat16*)p.dout, rows, p.Hq, p.delta);
  BAM_LAUNCH_CHECK();
  BAM_CUDA_TRY(cudaMemsetAsync(p.dq_acc, 0, sizeof(float) * rows * p.Hq * 128, s));
  return kOk;
}

int bam_attn_bwd_main(const BamAttnBwdParams* pp, void* stream) {
  if (int rc = check_bwd(pp)) return rc;
  const BamAttnBwdParams& p = *pp;
  const int64_t rows = (int64_t)p.nq * 128;
  CUtensorMap mq, mk, mv, mdo;
  int rc;
  if ((rc = make_tmap_rows_heads_d128(&mq, p.q, rows, p.Hq, 128))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mdo, p.dout, rows, p.Hq, 128))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mk, p.k, (int64_t)p.k_rows * 128, p.Hkv, 128))) return rc;
  if ((rc = make_tmap_rows_heads_d128(&mv, p.v, (int64_t)p.k_rows * 128, p.Hkv, 128))) return rc;
  const int smem = (int)sizeof(bwd::Smem) + 1024;
  BAM_CUDA_TRY(cudaFuncSetAttribute(bwd::attn_bwd_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid(p.Hkv, p.nb);
  bwd::attn_bwd_kernel<<<grid, bwd::kThreads, smem, (cudaStream_t)stream>>>(mq, mk, mv, mdo, p);
  BAM_LAUNCH_CHECK();
  return kOk;
}

int bam_attn_bwd_finalize(const BamAttnBwdParams* pp, void* stream) {
  if (int rc = check_bwd(pp)) return rc;
  const BamAttnBwdParams& p = *pp;
  const int64_t n4 = (int64_t)p.nq * 128 * p.Hq * 32;
  bwd::bwd_dq_convert_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(p.dq_acc), reinterpret_cast<uint2*>(p.dq), n4, p.scale);
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
