// Max co-resident thread-block clusters per cluster size at a given dynamic
// shared memory and block size (cudaOccupancyMaxActiveClusters), to size the
// fused column + diagonal pass's clusters.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_probe(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}

int main(int argc, char** argv) {
  const int threads = argc > 1 ? atoi(argv[1]) : 320;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int kb[] = {100, 120, 160, 170, 200, 214};
  for (int s : kb) {
    const size_t smem = (size_t)s * 1024;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    printf("smem %3d KB:", s);
    for (int cs = 1; cs <= 16; ++cs) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_probe, &cfg);
      printf(" %d:%d", cs, e == cudaSuccess ? n : -1);
    }
    printf("\n");
  }
  return 0;
}
