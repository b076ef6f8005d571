// Cluster occupancy probe: how many clusters of size CS (256 threads/CTA,
// given dynamic shared memory) can be co-resident on this GPU, via
// cudaOccupancyMaxActiveClusters. Usage: cluster_occ <smem_bytes> <cs>...
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void probe_kernel(int* p) {
  extern __shared__ int s[];
  if (p) p[0] = s[0];
}

int main(int argc, char** argv) {
  const int smem = argc > 1 ? atoi(argv[1]) : 180 * 1024;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  printf("SMs %d, smem/SM %zu, smem/block optin %zu\n", prop.multiProcessorCount, prop.sharedMemPerMultiprocessor,
         prop.sharedMemPerBlockOptin);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int a = 2; a < argc || a == 2; ++a) {
    const int cs = argc > a ? atoi(argv[a]) : 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, probe_kernel, &cfg);
    printf("smem %d cs %2d -> max active clusters %d (%d CTAs) %s\n", smem, cs, ncl, ncl * cs,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
