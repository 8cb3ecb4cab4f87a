// DSMEM probe on the pool's B200: latency of one ld.shared::cluster (local
// and remote rank), cluster barrier round trip, and st.async push bandwidth
// of 16 KB per CTA into the next rank (clusters of 4, one CTA per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ float ldc(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__global__ void __cluster_dims__(4, 1, 1) probe(long long* out) {
  __shared__ __align__(16) float buf[8192];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t me = rank();
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = (float)(i + me);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  csync();
  long long t0, t1;
  float acc = 0;
  if (threadIdx.x == 0) {
    // local-rank and remote-rank dependent-load chains
    uint32_t a = smem_u32(buf);
    t0 = clock64();
    for (int i = 0; i < 64; ++i) acc += ldc(mapa(a + ((int)acc & 4) , me));
    t1 = clock64();
    out[blockIdx.x * 8 + 0] = (t1 - t0) / 64;
    t0 = clock64();
    for (int i = 0; i < 64; ++i) acc += ldc(mapa(a + ((int)acc & 4), (me + 1) & 3));
    t1 = clock64();
    out[blockIdx.x * 8 + 1] = (t1 - t0) / 64;
  }
  __syncthreads();
  // cluster barrier round trip
  t0 = clock64();
  for (int i = 0; i < 16; ++i) csync();
  t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x * 8 + 2] = (t1 - t0) / 16;
  // st.async push: 16 KB (1024 x 16 B) into rank+1's buf, completion on its bar
  const uint32_t dst = (me + 1) & 3;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(16384));
  }
  csync();
  t0 = clock64();
  const uint32_t rb = mapa(smem_u32(buf + 4096), dst), rbar = mapa(smem_u32(&bar), dst);
  for (int v = threadIdx.x; v < 1024; v += blockDim.x) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     rb + v * 16),
                 "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f), "r"(rbar)
                 : "memory");
  }
  // wait for my own incoming 16 KB
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar))
      : "memory");
  t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x * 8 + 3] = t1 - t0;
  long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  if (threadIdx.x == 0) out[blockIdx.x * 8 + 4] = (long long)acc;
  csync();
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 8 * 128);
  probe<<<128, 256>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8 * 128];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  for (int b = 0; b < 8; ++b)
    printf("cta %d: local ld %lld cyc, remote ld %lld cyc, cluster barrier %lld cyc, 16 KB st.async push+recv %lld cyc\n",
           b, h[b * 8], h[b * 8 + 1], h[b * 8 + 2], h[b * 8 + 3]);
  return 0;
}
