// Bandwidth of a bulk-copy (cp.async.bulk) shared-memory ring on sm_100a:
// each CTA streams `units` pairs of `tile` bytes (K and V tiles) from
// scattered 16 KiB-aligned pool positions through an NST-stage ring; a warp
// producer issues, 4 consumer warps spin `delay` cycles per unit and release.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ringbench tools/ringbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   su32(b)),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}

__global__ void ring(const char* pool, const int* perm, int units, int tile, int nst, int delay, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t full[16], empty[16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int base = blockIdx.x * units;
  if (warp == 0) {
    if (lane == 0)
      for (int u = 0; u < units; ++u) {
        const int s = u % nst;
        if (u >= nst) mbar_wait(&empty[s], ((u / nst) - 1) & 1);
        const long long idx = perm[base + u];
        mbar_expect(&full[s], 2 * tile);
        bulk(sm + (size_t)s * 2 * tile, pool + idx * 2 * tile, tile, &full[s]);
        bulk(sm + (size_t)s * 2 * tile + tile, pool + idx * 2 * tile + tile, tile, &full[s]);
      }
    return;
  }
  unsigned long long acc = 0;
  for (int u = 0; u < units; ++u) {
    const int s = u % nst;
    mbar_wait(&full[s], (u / nst) & 1);
    acc += sm[(size_t)s * 2 * tile + tid * 16];
    const long long t0 = clock64();
    while (clock64() - t0 < delay) {
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 12345) sink[0] = acc;
}

int main() {
  const int tile = 16384;
  const long long n_tiles = 16384;  // 16384 x 32 KiB = 512 MiB pool
  char* pool;
  cudaMalloc(&pool, n_tiles * 2 * tile);
  cudaMemset(pool, 1, n_tiles * 2 * tile);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  char* flush;
  cudaMalloc(&flush, 512 << 20);
  int* perm;
  std::vector<int> hp(n_tiles);
  for (long long i = 0; i < n_tiles; ++i) hp[i] = (int)((i * 7919) % n_tiles);
  cudaMalloc(&perm, n_tiles * 4);
  cudaMemcpy(perm, hp.data(), n_tiles * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("%-8s %-6s %-6s %-6s %10s\n", "ctas/sm", "nst", "delay", "units", "GB/s");
  for (int cps : {1, 2, 3}) {
    for (int nst : {2, 3, 4, 6, 8}) {
      const size_t smem = (size_t)nst * 2 * tile;
      if (smem * cps > 220 * 1024) continue;
      cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int delay : {0, 1500}) {
        const int ctas = 148 * cps;
        const int units = (int)(n_tiles / ctas);
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemsetAsync(flush, rep, 512 << 20);
          cudaEventRecord(a);
          ring<<<ctas, 160, smem>>>(pool, perm, units, tile, nst, delay, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          best = ms < best ? ms : best;
        }
        const double bytes = (double)ctas * units * 2 * tile;
        printf("%-8d %-6d %-6d %-6d %10.1f\n", cps, nst, delay, units, bytes / (best * 1e-3) / 1e9);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
