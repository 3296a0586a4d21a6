// Can the persistent decode kernel run as clusters?  Max co-resident clusters
// for a 1-CTA-per-SM kernel with ~226 KB of shared memory, and whether a
// cooperative launch accepts a cluster dimension.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(384, 1) k(int* out) {
  extern __shared__ char smem[];
  smem[threadIdx.x] = 1;
  if (threadIdx.x == 0) atomicAdd(out, 1);
}

int main() {
  const int smem = 226 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int* out;
  cudaMalloc(&out, 4);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148 / cs * cs);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d (%d CTAs) [%s]\n", cs, n, n * cs, cudaGetErrorString(e));
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.numAttrs = 2;
    cfg.gridDim = dim3(n > 0 ? n * cs : cs);
    cudaMemset(out, 0, 4);
    e = cudaLaunchKernelEx(&cfg, k, out);
    cudaError_t e2 = cudaDeviceSynchronize();
    int h = 0;
    cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
    printf("   cooperative + cluster launch of %d CTAs: %s / %s, ran %d\n", cfg.gridDim.x,
           cudaGetErrorString(e), cudaGetErrorString(e2), h);
    cudaGetLastError();
  }
  return 0;
}
