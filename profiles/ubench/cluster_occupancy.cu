#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 12, 16}) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cs * 16); lc.blockDim = dim3(384); lc.dynamicSmemBytes = 220 * 1024;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &lc);
    printf("cluster %2d: max active clusters %d (%s) -> %d CTAs\n", cs, n, cudaGetErrorString(e), n * cs);
  }
}
