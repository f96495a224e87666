// tmem_probe.cu -- allocate all 512 TMEM columns on every SM (one 200 KB-smem CTA per SM) and
// free them; hangs if some SM's TMEM is still held (leaked) by an earlier kernel. Run under an
// outer `timeout`. Build: nvcc -gencode arch=compute_100a,code=sm_100a tmem_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  __shared__ unsigned slot;
  extern __shared__ char pad[];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  if (threadIdx.x == 0) out[blockIdx.x] = 1 + (pad[0] & 0);
}
int main() {
  int* d;
  cudaMalloc(&d, 148 * 4 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int r = 0; r < 4; ++r) k<<<148 * 2, 64, 200 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("tmem probe: %s\n", cudaGetErrorString(e));
  return 0;
}
