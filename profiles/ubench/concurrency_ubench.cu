// concurrency_ubench.cu -- can two persistent kernels on two streams of one process run at the
// same time on B200? Kernel A (launched first) spins until kernel B (launched second) sets a
// flag. Variants: plain launch / cluster launch (dims 1, 2), small / large dynamic smem.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ int g_tmem_mode;
__device__ __forceinline__ unsigned tmem_alloc32(unsigned* slot) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((unsigned)__cvta_generic_to_shared(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  return *slot;
}
__device__ __forceinline__ void tmem_free32(unsigned a) {
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(a));
}
__global__ void k_wait(volatile unsigned* f, unsigned long long* t, int blocks_needed) {
  extern __shared__ char sm[];
  __shared__ unsigned slot;
  unsigned ta = g_tmem_mode ? tmem_alloc32(&slot) : 0;
  if (threadIdx.x == 0) {
    unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (f[0] == 0) {
      unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 2000000000ULL) { f[1] = 1; break; }  // 2 s: give up
    }
  }
  sm[threadIdx.x] = 0;
  if (g_tmem_mode) tmem_free32(ta);
}
__global__ void k_set(volatile unsigned* f) {
  extern __shared__ char sm[];
  __shared__ unsigned slot;
  unsigned ta = g_tmem_mode ? tmem_alloc32(&slot) : 0;
  if (threadIdx.x == 0 && blockIdx.x == 0) f[0] = 1;
  sm[threadIdx.x] = 0;
  if (g_tmem_mode) tmem_free32(ta);
}

int launch(void* k, void** args, int grid, int smem, int cluster, cudaStream_t s) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid); lc.blockDim = dim3(128); lc.dynamicSmemBytes = smem; lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  lc.attrs = at; lc.numAttrs = cluster ? 1 : 0;
  return cudaLaunchKernelExC(&lc, k, args);
}

int main() {
  unsigned* f; cudaMalloc(&f, 16);
  unsigned long long* t; cudaMalloc(&t, 16);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaFuncSetAttribute(k_wait, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_set, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int tm : {0, 1})
  for (int cl : {0, 1, 2})
    for (int smem : {120 * 1024})
      for (int grid : {8, 64}) {
        cudaMemcpyToSymbol(g_tmem_mode, &tm, sizeof tm);
        cudaMemset(f, 0, 16);
        cudaDeviceSynchronize();
        int n = grid;
        void* aa[] = {&f, &t, &n};
        void* bb[] = {&f};
        int e1 = launch((void*)k_wait, aa, grid, smem, cl, a);
        int e2 = launch((void*)k_set, bb, cl == 2 ? 2 : 1, smem, cl, b);
        cudaDeviceSynchronize();
        unsigned h[2]; cudaMemcpy(h, f, 8, cudaMemcpyDeviceToHost);
        printf("tmem=%d cluster=%d smem=%6d grid=%2d: %s (launch %d %d)\n", tm, cl, smem, grid,
               h[1] ? "NOT concurrent (A timed out)" : "concurrent", e1, e2);
      }
  return 0;
}
