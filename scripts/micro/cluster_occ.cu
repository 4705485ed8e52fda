// How many 16-CTA (and 8-CTA) clusters of a field-sized CTA (512 threads,
// ~185 KiB shared memory, 1 CTA/SM) can be co-resident on this B200?
#include <cstdio>
__global__ void __launch_bounds__(512, 1) dummy(double* x) {
  extern __shared__ double s[];
  s[threadIdx.x] = x[threadIdx.x];
  __syncthreads();
  x[threadIdx.x] = s[511 - threadIdx.x];
}
int main() {
  const int smem = 189 * 1024;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 8);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    printf("SMs %d, cluster %2d: max active clusters %d (%d CTAs) [%s]\n", sms, cs, n, n * cs,
           cudaGetErrorString(e));
  }
  return 0;
}
