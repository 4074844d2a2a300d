// How many clusters of size C fit on this GPU with the sweep's footprint
// (608 threads, ~230 KB dynamic smem per CTA)?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int* p) { if (p) p[blockIdx.x] = 0; }
int main() {
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 230096);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148 * 4);
    cfg.blockDim = dim3(608);
    cfg.dynamicSmemBytes = 230096;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    printf("cluster %2d: max active clusters %d (= %d CTAs) %s\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
