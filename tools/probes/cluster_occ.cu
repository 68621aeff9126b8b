// Probe: how many thread-block clusters of a given size fit on this B200 at
// once (cudaOccupancyMaxActiveClusters), for CTA shapes like the attention
// kernel's (160 threads, ~70 KB or ~141 KB of shared memory).
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_occ tools/probes/cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dummy(int* p) {
  extern __shared__ int s[];
  if (p) p[blockIdx.x] = s[threadIdx.x];
}

int main() {
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"sms\": %d}\n", sms);
  const int smem_kb[] = {70, 88, 105, 141, 180};
  const int sizes[] = {1, 2, 4, 8, 16};
  for (int kb : smem_kb)
    for (int cs : sizes) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs * 16);
      cfg.blockDim = dim3(160);
      cfg.dynamicSmemBytes = kb * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
      printf("{\"smem_kb\": %d, \"cluster\": %d, \"max_active_clusters\": %d, \"ctas\": %d, \"err\": \"%s\"}\n", kb, cs,
             n, n * cs, cudaGetErrorString(e));
    }
  return 0;
}
