// mma_ubench.cu -- tcgen05.mma issue/throughput on B200 for the recurrent kernels' shapes:
// one CTA per SM issues `reps` x (K/16) MMAs (M=128, N in {32,64,128,256}, bf16, A and B
// resident in SWIZZLE_128B shared memory, K-major) into one TMEM accumulator, commits once and
// waits. Reports cycles per MMA instruction and TFLOP/s per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1604_01946_b200/csrc mma_ubench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "sm100_ptx.cuh"

using namespace rw;

// mode 8/9: per rep, bulk-load the B k-blocks (kblocks x N*128 B) from global `src` into the
// B region (one mbarrier per k-block), then (mode 8) issue the MMAs of each k-block as it lands,
// (mode 9) only wait for the loads. Measures L2 -> SMEM bulk-copy bandwidth with/without MMAs.
// L2 -> SMEM bulk-copy ingress per SM: each rep one CTA receives 64 KB as 64K/csz bulk copies
// (all in flight), completion on one mbarrier; no cluster.
__global__ void __launch_bounds__(128, 1) k_load(int N, int kblocks, int reps, const uint8_t* src,
                                                 unsigned long long* out, int csz, int mc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  const long long c0 = clock64();
  if (threadIdx.x == 0) {
    for (int r = 0; r < reps; ++r) {
      const uint8_t* s0 = src + (size_t)(r % 16) * 65536;
      mbar_arrive_expect_tx(&bar, 65536);
      for (int o = 0; o < 65536; o += csz)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sm + o)), "l"(s0 + o), "r"(csz), "r"(smem_u32(&bar)) : "memory");
      mbar_wait(&bar, r & 1);
    }
  }
  __syncthreads();
  const long long c1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2 + 0] = c1 - c0;
    out[blockIdx.x * 2 + 1] = c1 - c0;
  }
  (void)N; (void)kblocks; (void)mc;
}

// A operand in TMEM (tcgen05.mma ... [d], [a_tmem], b_desc): 128 rows x 512 K bf16 = 256 TMEM
// columns written once with tcgen05.st; B (N x 512) in SW128 smem; whole warp 0 issues with
// elect.sync. mode 0: SS (A in smem) issued the same way, for comparison.
__global__ void __launch_bounds__(128, 1) k_ts(int N, int reps, unsigned long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* A = sm;                 // 8 x 16 KB (mode 0)
  uint8_t* B = sm + 8 * 16384;     // 8 x N*128
  for (int i = threadIdx.x; i < (8 * 16384 + 8 * N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a_tmem = tmem + 128;  // columns 128..383 hold A
  {  // every warp writes its lane quarter of A: 256 columns of 0x3c003c00
    const uint32_t lane_base = (uint32_t)((threadIdx.x >> 5) * 32) << 16;
    for (int c = 0; c < 256; c += 8) {
      const uint32_t v = 0x3c003c00u;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                       a_tmem + lane_base + c),
                   "r"(v), "r"(v), "r"(v), "r"(v), "r"(v), "r"(v), "r"(v), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_make(1, false, false, 128, N);
    const uint64_t ad0 = sdesc_sw128(smem_u32(A), 16, 1024), bd0 = sdesc_sw128(smem_u32(B), 16, 1024);
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int kb = 0; kb < 8; ++kb) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = desc_add(bd0, kb * N * 128 + kk * 32);
          if (mode == 0) {
            umma_bf16_warp(tmem, desc_add(ad0, kb * 16384 + kk * 32), bd, idesc, 1u);
          } else {
            asm volatile(
                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(tmem),
                "r"(a_tmem + (kb * 4 + kk) * 8), "l"(bd), "r"(idesc));
          }
        }
      }
    }
    const long long c1 = clock64();
    umma_commit_warp(&bar);
    mbar_wait(&bar, 0);
    const long long c2 = clock64();
    if (threadIdx.x == 0) {
      out[blockIdx.x * 2 + 0] = c1 - c0;
      out[blockIdx.x * 2 + 1] = c2 - c0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Plain-load ingress: nthr threads each fetch 64 KB / nthr with LDG.128 (all in flight), then
// store to smem; mode 1 uses cp.async (LDGSTS) instead.
__global__ void __launch_bounds__(512, 1) k_ldg(const uint4* __restrict__ src, int reps, unsigned long long* out,
                                                int mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint4* sm = reinterpret_cast<uint4*>(sm_raw);
  const int per = 4096 / blockDim.x;  // uint4 per thread (64 KB = 4096 uint4)
  const long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const uint4* s0 = src + (size_t)(r % 64) * 4096;
    if (mode == 0) {
      uint4 v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < per) v[i] = __ldcg(s0 + i * blockDim.x + threadIdx.x);
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < per) sm[i * blockDim.x + threadIdx.x] = v[i];
    } else {
      for (int i = 0; i < per; ++i)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + i * blockDim.x + threadIdx.x)),
                     "l"(s0 + i * blockDim.x + threadIdx.x) : "memory");
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
  }
  const long long c1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = c1 - c0;
    out[blockIdx.x * 2 + 1] = c1 - c0;
  }
}

__global__ void __launch_bounds__(128, 1) k_mma(int N, int kblocks, int reps, unsigned long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* A = sm;                          // kblocks x 16 KB
  uint8_t* B = sm + kblocks * 16384;        // kblocks x N*128
  for (int i = threadIdx.x; i < (kblocks * 16384 + kblocks * N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, mode == 6 ? 2 : mode == 7 ? 4 : 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (mode >= 6 && (threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < (mode == 6 ? 2 : 4)) {
    const int nw = mode == 6 ? 2 : 4, w = threadIdx.x >> 5;
    const uint32_t idesc = idesc_make(1, false, false, 128, N);
    const uint64_t ad0 = sdesc_sw128(smem_u32(A), 16, 1024), bd0 = sdesc_sw128(smem_u32(B), 16, 1024);
    const long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int kb = w; kb < kblocks; kb += nw) {
        const uint64_t ad = ad0 + (uint64_t)((kb * 16384) >> 4), bd = bd0 + (uint64_t)((kb * N * 128) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma<false>(tmem + w * N, ad + 2 * kk, bd + 2 * kk, idesc, (r | (kb != w) | kk) ? 1u : 0u);
      }
    }
    const long long c1 = clock64();
    umma_commit(&bar);
    if (w == 0) {
      mbar_wait(&bar, 0);
    }
    const long long c2 = clock64();
    if (w == 0) {
      out[blockIdx.x * 2 + 0] = c1 - c0;
      out[blockIdx.x * 2 + 1] = c2 - c0;
    }
  } else if (mode < 6 && threadIdx.x == 0) {
    const uint32_t idesc = idesc_make(1, false, false, 128, N);
    const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
    const long long c0 = clock64();
    if (mode == 10 || mode == 11) {
      // the recurrent kernels' loop: per k-block wait a (complete) full barrier, fence, 4 MMAs,
      // commit to an empty barrier (mode 11: and a globaltimer stamp per k-block)
      __shared__ uint64_t fullb, emptyb;
      mbar_init(&fullb, 1);
      mbar_init(&emptyb, 1);
      fence_barrier_init();
      mbar_arrive(&fullb);  // phase 0 complete
      const uint64_t ad0 = sdesc_sw128(a0, 16, 1024), bd0 = sdesc_sw128(b0, 16, 1024);
      unsigned long long sink = 0;
      for (int r = 0; r < reps; ++r) {
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&fullb, 0);
          tc_fence_after();
          if (mode == 11) sink += globaltimer();
          const uint64_t ad = desc_add(ad0, kb * 16384), bd = desc_add(bd0, kb * N * 128);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma<false>(tmem, desc_add(ad, kk * 32), desc_add(bd, kk * 32), idesc, 1u);
          umma_commit(&emptyb);
        }
      }
      if (sink == 1) out[0] = 0;
    } else if (mode == 5) {
      // descriptors advanced by plain 64-bit adds: start address field is addr>>4 in bits 0..13
      const uint64_t ad0 = sdesc_sw128(a0, 16, 1024), bd0 = sdesc_sw128(b0, 16, 1024);
      for (int r = 0; r < reps; ++r) {
        uint64_t ad = ad0, bd = bd0;
        for (int kb = 0; kb < kblocks; ++kb) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma<false>(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (r | kb | kk) ? 1u : 0u);
          ad += 16384 >> 4;
          bd += (uint64_t)(N * 128) >> 4;
        }
      }
    } else
    for (int r = 0; r < reps; ++r) {
      for (int kb = 0; kb < kblocks; ++kb) {
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = sdesc_sw128(a0 + kb * 16384 + kk * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(b0 + kb * N * 128 + kk * 32, 16, 1024);
          // mode 2/3: round-robin over 2/4 independent accumulators (N columns apart) per MMA
          const int nacc = mode == 2 ? 2 : mode == 3 ? 4 : 1;
          const int ai = ((kb * 4 + kk) % nacc);
          umma<false>(tmem + ai * N, ad, bd, idesc, (r | kb | (kk >= nacc ? 1 : 0) | (kk % nacc != ai)) ? 1u : 0u);
        }
        if (mode == 1) umma_commit(&bar);  // a commit per k-block like the kernels
      }
    }
    const long long c1 = clock64();
    umma_commit(&bar);
    // wait for all: the last commit's phase
    const int commits = (mode == 1 ? reps * kblocks : 0) + 1;
    mbar_wait(&bar, (commits - 1) & 1);
    const long long c2 = clock64();
    out[blockIdx.x * 2 + 0] = c1 - c0;
    out[blockIdx.x * 2 + 1] = c2 - c0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  unsigned long long h[4096];
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int mode : {5})
    for (int N : {64})
      for (int grid : {148}) {
        const int kblocks = N == 256 ? 4 : 8;
        const int reps = 200;
        const size_t smem = 1024 + kblocks * 16384 + kblocks * N * 128;
        k_mma<<<grid, 128, smem>>>(N, kblocks, reps, d, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, grid * 16, cudaMemcpyDeviceToHost);
        const double n_mma = (double)reps * kblocks * 4;
        double worst = 0;
        for (int b = 0; b < grid; ++b) worst = worst > h[2 * b + 1] ? worst : h[2 * b + 1];
        const double cyc = worst / n_mma;
        const double flop = 2.0 * 128 * N * 16;
        printf("mode=%d N=%3d grid=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma -> %.0f FLOP/cyc/SM (peak ~8192)\n",
               mode, N, grid, h[0] / n_mma, cyc, flop / cyc);
      }
  uint8_t* src;
  cudaMalloc(&src, 64ull * 8 * 64 * 128);
  cudaMemset(src, 0, 64ull * 8 * 64 * 128);
  cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_load, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mc : {1}) for (int csz : {16384}) for (int grid : {128}) {
    const int N = 64, kblocks = 8, reps = 200;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(128);
    lc.dynamicSmemBytes = 1024 + kblocks * N * 128 + 100 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, k_load, N, kblocks, reps, (const uint8_t*)src, d, csz, mc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, grid * 16, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int b = 0; b < grid; ++b) worst = worst > h[2 * b] ? worst : h[2 * b];
    printf("load mc=%d csz=%5d grid=%3d: %.0f cyc per 64 KB step -> %.1f B/cyc/SM\n", mc, csz, grid, worst / reps,
           65536.0 * reps / worst);
  }
  cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode : {1}) for (int thr : {128}) {
    const int grid = 128, reps = 200;
    k_ldg<<<grid, thr, 200 * 1024>>>((const uint4*)src, reps, d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, grid * 16, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int b = 0; b < grid; ++b) worst = worst > h[2 * b] ? worst : h[2 * b];
    printf("ldg mode=%d threads=%d: %.0f cyc per 64 KB -> %.1f B/cyc/SM\n", mode, thr, worst / reps, 65536.0 * reps / worst);
  }
  cudaFuncSetAttribute(k_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int mode : {0, 1}) for (int N : {32, 64, 128}) {
    const int grid = 148, reps = 200;
    k_ts<<<grid, 128, 1024 + 8 * 16384 + 8 * N * 128>>>(N, reps, d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, grid * 16, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int b = 0; b < grid; ++b) worst = worst > h[2 * b + 1] ? worst : h[2 * b + 1];
    printf("%s N=%d: %.1f cyc/mma (warp-elect issue)\n", mode ? "TS (A in TMEM)" : "SS (A in smem)", N, worst / (reps * 32.0));
  }
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}
