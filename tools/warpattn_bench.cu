// Latency of the WarpAttn::chunk routine (mma_attn.cuh) in isolation: one CTA
// of W warps, K/V tile resident in shared memory, each warp calls chunk<> on
// the tile `iters` times (16 query rows per warp); prints cycles per call.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2402_15220_b200/csrc/kernels \
//        -o tools/warpattn_bench tools/warpattn_bench.cu
#include <cstdio>

#include "mma_attn.cuh"

using namespace pakv::dev;

template <int NTOK, bool MASK>
__global__ void k_chunk(float* out, long long* cyc, int iters, int c) {
  extern __shared__ __align__(128) unsigned char sm[];
  using WA = WarpAttn<__half, 128, 16>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2 * c * 128; i += blockDim.x)
    reinterpret_cast<__half*>(sm)[i] = __float2half(0.01f * (i % 97));
  __syncthreads();
  uint32_t qa[WA::KS][4];
  for (int ks = 0; ks < WA::KS; ++ks)
    for (int j = 0; j < 4; ++j) qa[ks][j] = 0x3c003c00u ^ (lane * 7 + ks + j);
  WA wa;
  wa.reset();
  const uint32_t k_u32 = smem_u32(sm), v_u32 = k_u32 + c * 128 * 2;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    for (int t = 0; t < c; t += NTOK) wa.template chunk<MASK, NTOK>(qa, k_u32, v_u32, t, c, 0.1f, lane);
  long long t1 = clock64();
  wa.finish();
  float s = wa.n_lo + wa.m_hi;
  for (int i = 0; i < WA::DT; ++i) s += wa.o[i][0] + wa.o[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
}

template <int NTOK, bool MASK>
void run(const char* name, int warps, int ctas, int c) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4 * ctas * warps * 32);
  cudaMalloc(&cyc, 8 * ctas * 32);
  const int smem = 2 * c * 128 * 2;
  cudaFuncSetAttribute(k_chunk<NTOK, MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 200;
  k_chunk<NTOK, MASK><<<ctas, warps * 32, smem>>>(out, cyc, 10, c);
  k_chunk<NTOK, MASK><<<ctas, warps * 32, smem>>>(out, cyc, iters, c);
  cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cyc, 8 * 32, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
  const double calls = (double)iters * (c / NTOK);
  printf("%-34s warps/CTA %d CTAs %4d: %7.1f cycles per call (%d tokens x 16 rows), %6.1f cycles per 64-token chunk\n",
         name, warps, ctas, mx / calls, NTOK, mx / calls * (64 / NTOK));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<16, false>("chunk<false,16>", 1, 1, 64);
  run<32, false>("chunk<false,32>", 1, 1, 64);
  run<64, false>("chunk<false,64>", 1, 1, 64);
  run<16, true>("chunk<true,16> (seq-first)", 1, 1, 64);
  run<16, false>("chunk<false,16>", 4, 1, 64);
  run<32, false>("chunk<false,32>", 4, 1, 64);
  run<32, false>("chunk<false,32>", 4, 148, 64);
  run<32, false>("chunk<false,32> 2 CTA/SM", 4, 296, 64);
  run<32, false>("chunk<false,32>", 8, 148, 64);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
