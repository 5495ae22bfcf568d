#include <cstdio>
#include <cuda_runtime.h>
#include <set>
__global__ void k(int* smid, long long spin) {
  extern __shared__ char s[];
  unsigned id; asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
  if (threadIdx.x == 0) smid[blockIdx.x] = id;
  long long t0 = clock64(); while (clock64() - t0 < spin) {}
  s[threadIdx.x] = 1;
}
int main() {
  int *d; cudaMalloc(&d, 4096 * 4);
  size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(148 * 2 / c * c); cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int ncl = 0; cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    cfg.gridDim = dim3(ncl * c);
    cudaMemset(d, 0xff, 4096 * 4);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, d, 200000000LL);
    cudaDeviceSynchronize();
    int h[4096]; cudaMemcpy(h, d, 4096 * 4, cudaMemcpyDeviceToHost);
    std::set<int> s; for (int i = 0; i < ncl * c; ++i) s.insert(h[i]);
    printf("cluster %d: max active clusters %d -> %d CTAs, distinct SMs %zu (%s)\n", c, ncl, ncl * c, s.size(), cudaGetErrorString(e));
  }
}
