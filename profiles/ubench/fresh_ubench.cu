// fresh_ubench.cu -- is an L2 bulk load of data that other SMs JUST wrote slower than one of
// static data? The recurrent kernels' per-step load (rec_cluster.cuh cl_load_b) reads h_{t-1} /
// dG_{t+1} microseconds after 16 producer CTAs stored it. P producer CTAs write 128 KB per step
// (each an 8 KB slice; 16-byte or 2-byte stores), release a gpu-scope flag; C consumer CTAs
// acquire it and bulk-load the 128 KB (4 x 32 KB cp.async.bulk) -- of the freshly written buffer
// or of a static one (mode). Reported: consumer time from flag observed to load complete.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fresh_ubench.bin fresh_ubench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kBytes = 128 * 1024, kSteps = 200, kP = 16;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_rlx(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_pc(uint8_t* buf, const uint8_t* stat, uint32_t* flags, uint32_t* done, int C, int mode, int narrow,
                     unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  uint8_t* sb = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const bool prod = blockIdx.x < kP;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar)));
  __syncthreads();
  unsigned long long tot = 0;
  for (int t = 0; t < kSteps; ++t) {
    uint8_t* b = buf + (size_t)(t & 1) * kBytes;
    if (prod) {
      if (t >= 2 && threadIdx.x == 0)
        while (ld_acq(done + t - 2) < (uint32_t)C) {
        }
      __syncthreads();
      uint8_t* sl = b + blockIdx.x * (kBytes / kP);
      if (narrow) {  // 2-byte stores, 32 per thread (the epilogue's pattern)
        for (int i = threadIdx.x; i < kBytes / kP / 2; i += blockDim.x)
          reinterpret_cast<uint16_t*>(sl)[i] = (uint16_t)(t + i);
      } else {
        for (int i = threadIdx.x; i < kBytes / kP / 16; i += blockDim.x)
          reinterpret_cast<uint4*>(sl)[i] = make_uint4(t, i, 0, 0);
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flags + t), "r"(1u) : "memory");
    } else if (threadIdx.x == 0) {
      while (ld_rlx(flags + t) < (uint32_t)kP) {
      }
      (void)ld_acq(flags + t);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const uint64_t t0 = gtime();
      const uint8_t* src = mode ? stat : b;
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(kBytes) : "memory");
      for (int i = 0; i < 4; ++i)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(sb + i * 32768)),
                     "l"(src + i * 32768), "r"(32768), "r"(su32(&bar))
                     : "memory");
      asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                       su32(&bar)),
                   "r"(t & 1)
                   : "memory");
      tot += gtime() - t0;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(done + t), "r"(1u) : "memory");
    }
  }
  if (!prod && threadIdx.x == 0) out[blockIdx.x - kP] = tot / kSteps;
}

int main() {
  uint8_t *buf, *stat;
  uint32_t *flags, *done;
  unsigned long long* out;
  cudaMalloc(&buf, 2 * kBytes);
  cudaMalloc(&stat, kBytes);
  cudaMemset(stat, 3, kBytes);
  cudaMalloc(&flags, kSteps * 4);
  cudaMalloc(&done, kSteps * 4);
  cudaMalloc(&out, 256 * 8);
  const int smem = kBytes + 2048;
  cudaFuncSetAttribute(k_pc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("P=%d producers x 8 KB, consumers bulk-load 128 KB (4 x 32 KB) after the flag; %d steps\n", kP, kSteps);
  for (int C : {1, 16, 64, 112})
    for (int narrow : {0, 1})
      for (int mode : {0, 1}) {
        cudaMemset(flags, 0, kSteps * 4);
        cudaMemset(done, 0, kSteps * 4);
        k_pc<<<kP + C, 256, smem>>>(buf, stat, flags, done, C, mode, narrow, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        std::vector<unsigned long long> h(C);
        cudaMemcpy(h.data(), out, C * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        printf("C=%3d %s stores, load of %s data: median %6llu ns  (min %llu, max %llu)\n", C, narrow ? "2-byte " : "16-byte",
               mode ? "static" : "fresh ", h[C / 2], h[0], h[C - 1]);
      }
  return 0;
}
