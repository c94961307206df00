// Max co-resident clusters (cudaOccupancyMaxActiveClusters) for GEMM-like
// CTAs (320 threads, given dynamic smem) at split-K cluster sizes 1..16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_occ cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(320, 2) k(int* p) {
  extern __shared__ int s[];
  if (p) p[threadIdx.x] = s[threadIdx.x];
}

int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int smems[] = {50 * 1024, 82 * 1024, 98 * 1024, 112 * 1024, 130 * 1024, 200 * 1024};
  for (int sm : smems) {
    printf("smem %3d KB:", sm / 1024);
    for (int cs : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(1, 1, cs * 64);
      cfg.blockDim = dim3(320);
      cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = 1;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = cs;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("  cs%-2d %4d clusters = %4d CTAs%s", cs, n, n * cs, e ? "(err)" : "");
    }
    printf("\n");
  }
  return 0;
}
