// sm100_ptx.cuh -- thin inline-PTX wrappers for the Blackwell (sm_100a) features the
// LSTM kernels use: mbarriers, TMA (cp.async.bulk.tensor), tcgen05 (alloc / mma / commit /
// ld), UMMA shared-memory and instruction descriptors, cluster DSMEM and gpu-scope
// acquire/release flags. Everything is written directly against the PTX ISA; descriptor
// bit layouts follow the sm_100 UMMA encoding (start>>4 @0, LBO>>4 @16, SBO>>4 @32,
// version=1 @46, swizzle mode @61; instruction descriptor c_fmt @4, a_fmt @7, b_fmt @10,
// a_major @15, b_major @16, N>>3 @17, M>>4 @24).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#define RW_DEVICE __device__ __forceinline__

namespace rw {

// ------------------------------------------------------------------ basics
RW_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
RW_DEVICE uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}
RW_DEVICE bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
RW_DEVICE uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------ mbarrier
// try_wait suspend-time hint (the waiting thread sleeps in hardware until the phase completes
// or this many ns pass); keeps waiting warps from spinning on issue slots the working warps
// of the SM need. Same order of magnitude as CUTLASS's barrier wait.
constexpr uint32_t kSuspendHintNs = 10000000;
RW_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
RW_DEVICE void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
RW_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
RW_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
RW_DEVICE bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase), "r"(kSuspendHintNs)
      : "memory");
  return ok != 0;
}
// Every mbarrier wait is bounded. A kernel stores its context's error word in `rw_wait_err`
// (set_wait_error, before its first __syncthreads). A wait still incomplete after kWaitNs records
// kWaitTimeoutCode there and returns; once the word is set, every later slow wait of the
// launch returns too, so a lost arrival ends the launch within seconds and the host reports
// RW_ESTATE (rw_sync) instead of a GPU that never returns or a sticky trap. Only a kernel
// without an error word (none in this library) traps. The fast path is one try_wait.
constexpr unsigned long long kWaitNs = 20ULL * 1000000000ULL;
constexpr int kWaitTimeoutCode = (1 << 30) | (3 << 28) | 15;
static __shared__ int* rw_wait_err;
RW_DEVICE void set_wait_error(int* e) { rw_wait_err = e; }
// out of line: inlined at every wait site it would add its timer / error-word code to each
// producer, MMA and epilogue loop
static __device__ __noinline__ bool mbar_wait_slow(uint64_t* bar, uint32_t phase) {
  const uint64_t t0 = globaltimer();
  int* const err = rw_wait_err;
#pragma unroll 1
  while (!mbar_try_wait(bar, phase)) {
    const uint64_t dt = globaltimer() - t0;
    if (dt > 1000000ULL && err && *reinterpret_cast<volatile int*>(err) != 0) return false;  // abandoned launch
    if (dt > kWaitNs) {
      if (!err) __trap();
      atomicCAS(err, 0, kWaitTimeoutCode);
      return false;
    }
  }
  return true;
}
RW_DEVICE void mbar_wait(uint64_t* bar, uint32_t phase) {
  if (!mbar_try_wait(bar, phase)) mbar_wait_slow(bar, phase);
}
RW_DEVICE void mbar_wait_bounded(uint64_t* bar, uint32_t phase) { mbar_wait(bar, phase); }

// ------------------------------------------------------------------ TMA
RW_DEVICE void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// L2 prefetch of one 2-D box (no shared-memory destination, no completion).
RW_DEVICE void tma_prefetch_2d(const CUtensorMap* m, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1)
               : "memory");
}
// 2-D tiled load global -> shared, completion signalled on `bar` (complete_tx bytes).
RW_DEVICE void tma_load_2d(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                           int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// Order this thread's prior generic-proxy global writes / acquired reads against later
// async-proxy (TMA) accesses.
RW_DEVICE void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
RW_DEVICE void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------ tcgen05
template <uint32_t kCols>
RW_DEVICE void tmem_alloc(uint32_t* smem_result) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_result)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t kCols>
RW_DEVICE void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
RW_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
RW_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 inputs) or kind::tf32, fp32 accumulate.
template <bool kTF32>
RW_DEVICE void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                    uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}
// Warp-converged variants: the whole warp executes them and elect.sync picks the issuing lane
// inside the instruction block. Issued from a lane-0-only branch instead, every tcgen05.mma
// gets wrapped in an ELECT/R2UR.BROADCAST waterfall loop whose fixed latencies bounded the
// issue rate at ~155 cycles per MMA in the recurrent kernels (ncu source view: stall_wait).
RW_DEVICE void umma_bf16_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
template <bool kTF32>
RW_DEVICE void umma_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    umma_bf16_warp(tmem_d, adesc, bdesc, idesc, accumulate);
  }
}
// A operand from TENSOR MEMORY ("TS"): D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16. A is
// M = 128 rows on the 128 lanes, K along the columns with two 16-bit elements per 32-bit column
// (element k of the row in column k/2, even k in the low half): one K = 16 step reads 8 columns
// (layout checked on B200 by profiles/ubench/f16x2_ts_check.cu).
RW_DEVICE void umma_ts_f16_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
RW_DEVICE void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
// Arrive (once) on `bar` when all previously issued tcgen05.mma of this thread complete.
RW_DEVICE void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 consecutive columns of 32-bit: thread i of the warp gets lane (quarter*32+i).
RW_DEVICE void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
RW_DEVICE void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}
// registers -> 8 consecutive 32-bit columns of this warp's 32 lanes (lane quarter = warp % 4)
RW_DEVICE void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
RW_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
RW_DEVICE void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ UMMA descriptors
// Shared-memory matrix descriptor, SWIZZLE_128B (mode 2), version 1 (sm_100).
//   K-major tile : rows of 128 B, 8-row groups 1024 B apart (SBO); LBO unused.
//   MN-major tile: 128 B lines along MN, consecutive K rows 128 B apart, 8-row groups at
//                  SBO = 1024 B, successive 128-B MN chunks at LBO bytes.
RW_DEVICE uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}
// Advance a shared-memory matrix descriptor by `bytes` (the start-address field, bits 0..13,
// holds addr >> 4; shared memory < 256 KB never carries out of it). Lets the MMA issuer build
// each descriptor with one 64-bit add instead of re-encoding (measured: re-encoding in the
// uniform datapath bounded a single issuing thread at ~85-165 cycles per tcgen05.mma,
// profiles/ubench/mma_ubench.cu).
RW_DEVICE uint64_t desc_add(uint64_t d, uint32_t bytes) { return d + (uint64_t)(bytes >> 4); }
// Instruction descriptor: fp32 accumulate; fmt 1 = bf16, 2 = tf32.
__host__ __device__ constexpr uint32_t idesc_make(uint32_t fmt, bool a_mn_major, bool b_mn_major,
                                                  uint32_t M, uint32_t N) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((a_mn_major ? 1u : 0u) << 15) |
         ((b_mn_major ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// ------------------------------------------------------------------ cluster / DSMEM
RW_DEVICE uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
RW_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
RW_DEVICE uint32_t map_dsmem(uint32_t local_saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_saddr), "r"(rank));
  return r;
}
RW_DEVICE float ld_dsmem_f32(uint32_t cluster_saddr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(cluster_saddr) : "memory");
  return v;
}
RW_DEVICE float4 ld_dsmem_f32x4(uint32_t cluster_saddr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_saddr)
               : "memory");
  return v;
}

// ------------------------------------------------------------------ gpu-scope flags
RW_DEVICE uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Relaxed gpu-scope load: observes other SMs' writes (bypasses L1) without the L1
// invalidation (CCTL.IVALL) an acquire load carries -- for spin loops.
RW_DEVICE uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
RW_DEVICE void red_release_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
RW_DEVICE void red_relaxed_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
RW_DEVICE void nanosleep(uint32_t ns) { asm volatile("nanosleep.u32 %0;" ::"r"(ns)); }

// Named barrier among `nthreads` threads (id 1..15; 0 is __syncthreads).
RW_DEVICE void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- CTA pairs (cta_group::2): both CTAs' TMA loads complete on the leader's (rank 0)
// barrier, the leader issues M = 256 MMAs over both CTAs' operands, commits multicast to both.
namespace g2 {
// shared::cluster address of the same object in the pair's leader (cluster rank 0)
RW_DEVICE uint32_t leader_addr(const void* p) { return map_dsmem(smem_u32(p), 0); }
RW_DEVICE void tma_load_2d_pair(void* smem_dst, const CUtensorMap* m, uint64_t* bar_any,
                                                 int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_addr(bar_any)), "r"(c0), "r"(c1)
      : "memory");
}
RW_DEVICE void umma2_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// commit to the barrier at the same offset in both CTAs of the pair
RW_DEVICE void commit2_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
      ::"r"(smem_u32(bar)), "h"((uint16_t)3)
      : "memory");
}
}  // namespace g2

}  // namespace rw
