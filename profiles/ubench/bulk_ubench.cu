// bulk_ubench.cu -- per-SM ingress of an L2-resident 128 KB operand block into shared memory,
// the recurrent kernels' per-step "load" phase (rec_cluster.cuh cl_load_b: 1-D cp.async.bulk of
// 32 KB k-block pairs). Variants: chunk size of the 1-D bulk copies (all issued at once by one
// thread, or spread over the 32 lanes of a warp), and 2-D tensor TMA (cp.async.bulk.tensor) of
// the same bytes in 128 B x 256-row boxes. G CTAs (one per SM) load concurrently, each rep
// timed with %globaltimer from issue to the mbarrier's completion; the source is written once
// and re-read every rep (L2 hits).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_ubench.bin bulk_ubench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kBytes = 128 * 1024;
constexpr int kReps = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// mode 0: 1-D chunks by thread 0; mode 1: 1-D chunks spread over a warp; mode 2: 2-D TMA boxes
__global__ void k_load(const uint8_t* src, int distinct, int chunk, int mode, const __grid_constant__ CUtensorMap map,
                       unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const uint8_t* s = src + (distinct ? (size_t)blockIdx.x * kBytes : 0);
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  unsigned long long tot = 0;
  for (int r = 0; r < kReps; ++r) {
    uint64_t t0 = 0;
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) {
        t0 = gtime();
        mbar_expect(&bar, kBytes);
      }
      __syncwarp();
      const int n = kBytes / chunk;
      if (mode == 0) {
        if (threadIdx.x == 0)
          for (int i = 0; i < n; ++i) bulk(buf + i * chunk, s + (size_t)i * chunk, chunk, &bar);
      } else if (mode == 1) {
        for (int i = threadIdx.x; i < n; i += 32) bulk(buf + i * chunk, s + (size_t)i * chunk, chunk, &bar);
      } else if (threadIdx.x == 0) {
        // boxes of 64 bf16 (128 B) x 256 rows = 32 KB
        for (int i = 0; i < kBytes / (256 * 128); ++i)
          tma2d(buf + i * 256 * 128, &map, 0, (distinct ? blockIdx.x * (kBytes / 128) : 0) + i * 256, &bar);
      }
      if (threadIdx.x == 0) {
        mbar_wait(&bar, r & 1);
        tot += gtime() - t0;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tot / kReps;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int maxG = 148;
  uint8_t* src;
  cudaMalloc(&src, (size_t)maxG * kBytes);
  cudaMemset(src, 1, (size_t)maxG * kBytes);
  unsigned long long* out;
  cudaMalloc(&out, maxG * 8);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {64, (cuuint64_t)maxG * kBytes / 128};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 256}, es[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) printf("tensor map encode failed %d\n", (int)cr);
  const int smem = kBytes + 2048;
  cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("B200 SMs=%d, %d KB per CTA per rep, %d reps; ns = mean issue->complete per CTA (median over CTAs)\n", sms,
         kBytes / 1024, kReps);
  const char* mname[3] = {"1d-thread0", "1d-warp", "2d-tma"};
  for (int G : {1, 16, 64, 128, 148})
    for (int distinct : {0, 1})
      for (int mode = 0; mode < 3; ++mode)
        for (int chunk : {4096, 16384, 32768, 131072}) {
          if (mode == 2 && chunk != 32768) continue;
          if (mode == 1 && chunk > 16384) continue;
          k_load<<<G, 128, smem>>>(src, distinct, chunk, mode, map, out);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          std::vector<unsigned long long> h(G);
          cudaMemcpy(h.data(), out, G * 8, cudaMemcpyDeviceToHost);
          std::vector<unsigned long long> srt = h;
          std::sort(srt.begin(), srt.end());
          const double ns = (double)srt[G / 2];
          printf("G=%3d %-8s %-10s chunk=%6d: %7.0f ns  %6.1f GB/s per SM\n", G, distinct ? "distinct" : "shared",
                 mname[mode], mode == 2 ? 32768 : chunk, ns, kBytes / ns);
        }
  return 0;
}
