// Occupancy of thread-block clusters on this GPU: how many clusters of size C
// (1 .. 16) with a given block size / dynamic shared memory can be resident.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cp tools/cluster_probe.cu && /tmp/cp
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_probe(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("sms %d\n", sms);
  const int threads[] = {288, 544};
  const int smem_kb[] = {60, 70, 100, 110, 200};
  for (int th : threads)
    for (int kb : smem_kb)
      for (int c : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c * 64);
        cfg.blockDim = dim3(th);
        cfg.dynamicSmemBytes = kb * 1024;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = c;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_probe, &cfg);
        printf("threads %d smem %3d KB cluster %2d: %4d clusters = %4d CTAs (%s)\n", th, kb, c, n,
               n * c, cudaGetErrorString(e));
      }
  return 0;
}
