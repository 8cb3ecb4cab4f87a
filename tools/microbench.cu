// Primitive latency / throughput on sm_100a (one warp per measurement unless
// noted): mma.sync m16n8k16 f16->f32 (dependent chain vs independent),
// ldmatrix.x4, ex2.approx, shfl.xor, and LDS.128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ void mma(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int CHAINS>
__global__ void k_mma(float* out, long long* cyc, int iters) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u};
  float c[CHAINS][4] = {};
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) mma(c[k], a, a[0] + i, a[1] + k);
  }
  long long t1 = clock64();
  float s = 0;
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ex2(float* out, long long* cyc, int iters) {
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[k]));
  long long t1 = clock64();
  float s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_shfl(float* out, long long* cyc, int iters) {
  float x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 + (i & 7));
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ldsm(float* out, long long* cyc, int iters) {
  __shared__ __align__(128) unsigned char sm[16384];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = i;
  __syncthreads();
  uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const int lane = threadIdx.x & 31;
  uint32_t addr = base + ((lane & 7) * 256) + (((lane >> 3) ^ (lane & 7)) << 4);
  uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr + ((r0 & 1) << 9)));  // dependent chain
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = r0 + r1 + r2 + r3;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 1 << 16);
  long long h[4096];
  const int iters = 4096;
  auto rep = [&](const char* name, int blocks, int threads, double ops_per_iter_per_warp) {
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < blocks; ++i) mean += h[i];
    mean /= blocks;
    printf("%-44s blocks %4d thr %4d: %8.2f cycles per op per warp\n", name, blocks, threads,
           mean / (iters * ops_per_iter_per_warp));
  };
  // latency: 1 warp, 1 chain
  k_mma<1><<<1, 32>>>(out, cyc, iters); rep("mma latency (1 warp, 1 chain)", 1, 32, 1);
  k_mma<8><<<1, 32>>>(out, cyc, iters); rep("mma 1 warp, 8 chains", 1, 32, 8);
  k_mma<8><<<1, 128>>>(out, cyc, iters); rep("mma 4 warps/SM, 8 chains", 1, 128, 8);
  k_mma<8><<<1, 256>>>(out, cyc, iters); rep("mma 8 warps/SM, 8 chains", 1, 256, 8);
  k_mma<8><<<148, 512>>>(out, cyc, iters); rep("mma 16 warps/SM x148, 8 chains", 148, 512, 8);
  k_ex2<<<1, 32>>>(out, cyc, iters); rep("ex2 1 warp, 8 indep", 1, 32, 8);
  k_ex2<<<1, 256>>>(out, cyc, iters); rep("ex2 8 warps, 8 indep", 1, 256, 8);
  k_shfl<<<1, 32>>>(out, cyc, iters); rep("shfl latency (dependent)", 1, 32, 1);
  k_ldsm<<<1, 32>>>(out, cyc, iters); rep("ldmatrix.x4 latency (dependent)", 1, 32, 1);
  k_ldsm<<<1, 256>>>(out, cyc, iters); rep("ldmatrix.x4 8 warps (dependent each)", 1, 256, 1);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sm clock attr %d kHz\n", clk);
  return 0;
}
