// Shared device helpers for the bam (bitfield attention mask) kernels: sm_100a only.
//
// Raw PTX wrappers for mbarrier, TMA (cp.async.bulk*), tcgen05 (alloc / mma /
// commit / ld / st / fences) and the shared-memory matrix descriptors UMMA
// consumes.  Everything here is written for B200 (compute capability 10.0a).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "bam kernels target sm_100a only"
#endif

namespace bam {

// ----------------------------------------------------------------------------- errors
// Status codes returned by every C-ABI entry point (include/bam.h).
enum Status : int {
  kOk = 0,
  kInvalidArgument = 1,
  kCudaError = 2,
  kUnsupported = 3,
};

void set_last_error(const char* fmt, ...);

#define BAM_CHECK_ARG(cond, ...)                                   \
  do {                                                             \
    if (!(cond)) {                                                 \
      ::bam::set_last_error(__VA_ARGS__);                          \
      return ::bam::kInvalidArgument;                              \
    }                                                              \
  } while (0)

#define BAM_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      ::bam::set_last_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                            __FILE__, __LINE__);                                        \
      return ::bam::kCudaError;                                                         \
    }                                                                                   \
  } while (0)

#define BAM_LAUNCH_CHECK() BAM_CUDA_TRY(cudaGetLastError())

// ----------------------------------------------------------------------------- basics
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t warp_id() {
  return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// ----------------------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint32_t mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok;
}
// Bounded waits: a protocol bug traps (a reported launch failure) instead of
// hanging the GPU.  mbar_wait spins tightly (latency-critical roles: the MMA
// issuer); mbar_wait_sleep backs off with nanosleep so waiting warps do not
// steal issue slots from the warps sharing their SM sub-partition.
static __device__ __noinline__ void mbar_timeout_trap() {
  printf("bam: mbarrier wait timeout (block %d thread %d)\n", blockIdx.x, threadIdx.x);
  __trap();
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t iters = 0;
  while (!mbar_try_wait(addr, parity)) {
    if (++iters > (1u << 28)) mbar_timeout_trap();
  }
}
template <int kSleepNs = 64>
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t iters = 0;
  while (!mbar_try_wait(addr, parity)) {
    if constexpr (kSleepNs > 0) __nanosleep(kSleepNs);
    if (++iters > (1u << 28)) mbar_timeout_trap();
  }
}

#ifndef BAM_COMPUTE_SLEEP_NS
#define BAM_COMPUTE_SLEEP_NS 32   // back-off of the softmax / compute warps' waits
#endif

// ----------------------------------------------------------------------------- tracing
// -DBAM_TRACE builds record clock64() per (event, step) for one CTA into a
// device buffer installed with bam_set_trace_buffer (development aid).
#ifdef BAM_TRACE
constexpr int kTraceSteps = 4096;
static __device__ unsigned long long* g_bam_trace = nullptr;   // per translation unit
// kernels load the pointer once: unsigned long long* const bam_trace_ptr = g_bam_trace;
#define BAM_TRACE_EV(cond, ev, step)                                                 \
  do {                                                                               \
    if ((cond) && bam_trace_ptr && (step) < ::bam::kTraceSteps)                      \
      bam_trace_ptr[(ev) * ::bam::kTraceSteps + (step)] = clock64();                 \
  } while (0)
#else
#define BAM_TRACE_EV(cond, ev, step) \
  do {                               \
  } while (0)
#endif

// -DBAM_CTA_CLOCK builds record, per CTA of the attention kernels, {start, end}
// %globaltimer ns, the SM id, the CTA's work count and (forward) the ns its TMA
// warp spent waiting on CP arrival flags into a buffer installed with
// bam_set_cta_clock_buffer (tools/cta_tail.py: the intra-GPU tail that a
// persistent work queue could remove; the exposed exchange).
#ifdef BAM_CTA_CLOCK
static __device__ unsigned long long* g_bam_cta_clock = nullptr;   // per translation unit
__device__ __forceinline__ unsigned long long bam_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BAM_CTA_CLOCK_BEGIN() const unsigned long long bam_cta_t0 = ::bam::bam_globaltimer()
#define BAM_CTA_CLOCK_END(work)                                                           \
  do {                                                                                    \
    if (threadIdx.x == 0 && g_bam_cta_clock) {                                            \
      uint32_t smid_;                                                                     \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                                  \
      unsigned long long* r_ =                                                            \
          g_bam_cta_clock + 8 * (blockIdx.x + (size_t)gridDim.x * blockIdx.y);            \
      r_[0] = bam_cta_t0;                                                                 \
      r_[1] = ::bam::bam_globaltimer();                                                   \
      r_[2] = smid_;                                                                      \
      r_[3] = (unsigned long long)(work);                                                 \
    }                                                                                     \
  } while (0)
#define BAM_CTA_CLOCK_FLAG_WAIT(ns)                                                       \
  do {                                                                                    \
    if (g_bam_cta_clock)                                                                  \
      g_bam_cta_clock[8 * (blockIdx.x + (size_t)gridDim.x * blockIdx.y) + 4] = (ns);      \
  } while (0)
#else
#define BAM_CTA_CLOCK_FLAG_WAIT(ns) \
  do {                              \
  } while (0)
#define BAM_CTA_CLOCK_BEGIN() \
  do {                        \
  } while (0)
#define BAM_CTA_CLOCK_END(work) \
  do {                          \
  } while (0)
#endif

// ----------------------------------------------------------------------------- TMA
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 3D tiled load (coords innermost first) completing on an mbarrier.
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* m, uint64_t* bar, void* dst,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// 1D bulk copy global -> shared (bytes % 16 == 0, both 16-B aligned).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// named barrier among `count` threads (ids 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// Spin (with back-off, bounded) until *flag >= value, acquire at GPU scope.
__device__ __forceinline__ void wait_flag_geq(const int32_t* flag, int32_t value) {
  uint32_t iters = 0;
  while (true) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= value) break;
    __nanosleep(128);
    if (++iters > (1u << 26)) mbar_timeout_trap();
  }
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// generic-proxy smem writes -> visible to the async proxy (tcgen05.mma reads)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ----------------------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Arrive on `bar` when every tcgen05 op issued so far by this thread completes.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Warp-uniform variants: the whole warp executes the call (no divergent
// branch around a uniform-datapath instruction, so no ELECT/BRA.U.ANY loop),
// and only the lane with `leader` != 0 issues it.
__device__ __forceinline__ void mma_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(leader)
      : "memory");
}
__device__ __forceinline__ void mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(leader)
      : "memory");
}
__device__ __forceinline__ void tc_commit_w(uint64_t* bar, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::
          "r"(smem_u32(bar)),
      "r"(leader)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_w(const CUtensorMap* m, uint64_t* bar, void* dst,
                                              int c0, int c1, int c2, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %6, 0;\n\t"
      "@q cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];\n\t}\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(leader)
      : "memory");
}
__device__ __forceinline__ void bulk_load_w(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
      "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      "\n\t}\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "r"(leader)
      : "memory");
}
// Multicast variant: the same box lands at the same smem offset in every CTA
// of `cta_mask` and completes each CTA's mbarrier at the same offset.
__device__ __forceinline__ void tma_load_3d_mc_w(const CUtensorMap* m, uint64_t* bar, void* dst,
                                                 int c0, int c1, int c2, uint16_t cta_mask,
                                                 uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %7, 0;\n\t"
      "@q cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;\n\t}\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "h"(cta_mask), "r"(leader)
      : "memory");
}
// tcgen05.commit arriving on the mbarrier at `bar`'s offset in every CTA of cta_mask
__device__ __forceinline__ void tc_commit_mc_w(uint64_t* bar, uint16_t cta_mask, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}\n" ::"r"(smem_u32(bar)),
      "h"(cta_mask), "r"(leader)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Distributed shared memory: this CTA's shared address `saddr` in cluster CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// remote arrive with the default (CTA-scope) semantics: orders this thread's
// tcgen05 work (after tcgen05.wait + fence::before_thread_sync) without the
// GPU-scope memory barrier a cluster-scope release compiles to
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// ---- CTA-pair (cta_group::2) tensor-core helpers -----------------------------
// One MMA issued by the even CTA of a cluster pair computes an M = 256 tile:
// A rows 0-127 come from CTA 0's shared memory / TMEM, rows 128-255 from CTA
// 1's (same addresses); B is split by N (each CTA holds N/2 rows of B at the
// same address); D rows land in each CTA's own TMEM.
__device__ __forceinline__ void tmem_alloc_2cta(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish_2cta() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_2cta(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void mma_ss_2cta_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate,
                                              uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(leader)
      : "memory");
}
__device__ __forceinline__ void mma_ts_2cta_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate,
                                              uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(leader)
      : "memory");
}
// commit of the pair's MMAs, arriving on `bar`'s offset in every CTA of cta_mask
__device__ __forceinline__ void tc_commit_2cta_mc_w(uint64_t* bar, uint16_t cta_mask,
                                                    uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}\n" ::"r"(smem_u32(bar)),
      "h"(cta_mask), "r"(leader)
      : "memory");
}
// TMA into this CTA's shared memory, completing the transaction bytes on the
// PAIR LEADER's mbarrier (cluster address `bar_cluster`)
__device__ __forceinline__ void tma_load_3d_2cta_w(const CUtensorMap* m, uint32_t bar_cluster,
                                                   void* dst, int c0, int c1, int c2,
                                                   uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %6, 0;\n\t"
      "@q cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];\n\t}\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2),
      "r"(leader)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_w(uint64_t* bar, uint32_t bytes, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n\t}\n" ::"r"(
          smem_u32(bar)),
      "r"(bytes), "r"(leader)
      : "memory");
}

// Instruction descriptor: bf16 x bf16 -> fp32, dense, M x N, operand majors
// (0 = K-major, 1 = MN-major).  Bit layout per the sm_100 UMMA instruction
// descriptor: c_fmt[4:6) a_fmt[7:10) b_fmt[10:13) a_major[15] b_major[16]
// n>>3 [17:23) m>>4 [24:29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_major, int b_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_major) << 15) |
         (uint32_t(b_major) << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bit set.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes,
                                                uint32_t sbo_bytes) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

// TMEM loads: 32 lanes x 32 bits, each thread gets N consecutive columns of its lane.
#define BAM_TMEM_LD32(taddr, r)                                                              \
  asm volatile(                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"  \
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),  \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),           \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),        \
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),        \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),        \
        "=r"(r[31])                                                                          \
      : "r"(taddr))

#define BAM_TMEM_ST8(taddr, r)                                                           \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: \
                   "r"(taddr),                                                          \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), \
               "r"(r[7])                                                                \
               : "memory")

#define BAM_TMEM_LD16(taddr, r)                                                              \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10," \
               "%11,%12,%13,%14,%15}, [%16];"                                              \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),    \
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),  \
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                         \
               : "r"(taddr))

#define BAM_TMEM_ST16(taddr, r)                                                           \
  asm volatile(                                                                           \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11," \
      "%12,%13,%14,%15,%16};" ::"r"(taddr),                                               \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),        \
      "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),    \
      "r"(r[14]), "r"(r[15])                                                              \
      : "memory")

#define BAM_TMEM_ST32(taddr, r)                                                               \
  asm volatile(                                                                               \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12," \
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::  \
          "r"(taddr),                                                                         \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),            \
      "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),        \
      "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),     \
      "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),     \
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])                                          \
      : "memory")

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ----------------------------------------------------------------------------- math
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2: two lanes per instruction).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 a, b, c, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mov.b64 c, {%6, %7};\n\tfma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// 2^x for a pair on the FMA pipe (packed FFMA2): x = n + f, f in [-0.5, 0.5]
// (round via the 1.5*2^23 magic constant), 2^f by a degree-4 polynomial
// (rel. err < 4e-6, well below bf16 P rounding), exponent n added to the
// float bits.  x <= 8 (the forward's lazy rescale; x <= 0 in the backward); clamping at -127 makes 2^x flush
// to ~0 like ex2.approx.ftz.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  constexpr float kMagic = 12582912.f;
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 t = fadd2(x, make_float2(kMagic, kMagic));  // integer part in the low bits
  const float2 f = ffma2(fadd2(t, make_float2(-kMagic, -kMagic)), make_float2(-1.f, -1.f), x);
  float2 p = ffma2(make_float2(1.3333558e-3f, 1.3333558e-3f), f,
                   make_float2(9.6181291e-3f, 9.6181291e-3f));
  p = ffma2(p, f, make_float2(5.5504109e-2f, 5.5504109e-2f));
  p = ffma2(p, f, make_float2(2.4022651e-1f, 2.4022651e-1f));
  p = ffma2(p, f, make_float2(6.9314718e-1f, 6.9314718e-1f));
  p = ffma2(p, f, make_float2(1.0f, 1.0f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Byte offset of element (row, col) of a [rows x 128] bf16 tile stored as two
// TMA SWIZZLE_128B boxes of 64 columns (box b at b * rows * 128 bytes).
__device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t col, uint32_t rows) {
  const uint32_t box = col >> 6;
  const uint32_t chunk = ((col & 63) >> 3) ^ (row & 7);
  return box * rows * 128 + row * 128 + chunk * 16 + (col & 7) * 2;
}

// The mask predicate (reference mask.py:106-112), on global token indices.
__device__ __forceinline__ bool bam_allowed(long long dq, long long qg, long long dk,
                                            long long kg) {
  return (dq & 1) ? (kg <= qg && (dq & dk) != 0) : (dk == dq);
}

}  // namespace bam
