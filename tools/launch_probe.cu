// Launch-overhead probe: device time (CUDA events, back-to-back launches) of
// an empty kernel for combinations of cluster size, dynamic shared memory and
// block size -- what a decode step pays before / after its CTAs run.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* p) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0 && p[0] == 12345) sm[0] = 1, p[1] = sm[0];
}

int main() {
  int* d;
  cudaMalloc(&d, 64);
  cudaMemset(d, 0, 64);
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg { int grid, block, cluster; size_t smem; };
  Cfg cfgs[] = {{128, 384, 1, 0}, {128, 384, 4, 0}, {128, 384, 1, 220 * 1024}, {128, 384, 4, 220 * 1024},
                {296, 160, 1, 108 * 1024}, {148, 384, 1, 220 * 1024}, {128, 384, 2, 220 * 1024},
                {128, 384, 8, 220 * 1024}, {128, 128, 4, 220 * 1024}, {256, 160, 8, 100 * 1024}};
  for (const Cfg& c : cfgs) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(c.grid);
    lc.blockDim = dim3(c.block);
    lc.dynamicSmemBytes = c.smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    for (int w = 0; w < 20; ++w) cudaLaunchKernelEx(&lc, empty_kernel, d);
    const int n = 200;
    cudaEventRecord(a);
    for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&lc, empty_kernel, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    // single launch bracketed by events (includes the event overhead)
    float one = 0, best = 1e9;
    for (int r = 0; r < 20; ++r) {
      cudaEventRecord(a);
      cudaLaunchKernelEx(&lc, empty_kernel, d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&one, a, b);
      if (one < best) best = one;
    }
    printf("grid %4d block %3d cluster %2d smem %6zu: back-to-back %.2f us/launch, single %.2f us (%s)\n", c.grid,
           c.block, c.cluster, c.smem, 1e3 * ms / n, 1e3 * best, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
