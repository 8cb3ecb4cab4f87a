// Pure-read HBM bandwidth on sm_100a: what ceiling can a streaming kernel
// that only READS reach (the measured copy peak counts read + write bytes)?
//   (a) LDG.128 grid-stride read (sum into a register, one store per thread)
//   (b) cp.async.bulk ring: CTAs x stages x (pieces per 32 KiB stage), each
//       CTA streaming contiguous 32 KiB units at scattered positions
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/readbench tools/readbench.cu
#include <cstdint>
#include <cstdio>
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
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok)
               : "r"(su32(b)), "r"(ph)
               : "memory");
  return ok;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  while (!mbar_try(b, ph)) {
  }
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}

__global__ void ldg_read(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride),
                d = __ldcs(p + i + 3 * stride);
    acc ^= a.x ^ a.w ^ b.y ^ b.z ^ c.x ^ c.w ^ d.y ^ d.z;
  }
  for (; i < n; i += stride) acc ^= __ldcs(p + i).x;
  if (acc == 0x12345678u) sink[0] = acc;
}

// units of 32 KiB at scattered positions perm[], `pieces` bulk copies each
// split != 0: the unit's two 16 KiB halves come from two pools 2 GiB apart (K and V)
__global__ void ring(const char* pool, const int* perm, int units, int nst, int pieces, unsigned* sink, int split = 0) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t full[16], empty[16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kUnit = 32768;
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
    for (int u = 0; u < units; ++u) {
      const int s = u % nst;
      if (u >= nst) mbar_wait(&empty[s], ((u / nst) - 1) & 1);
      if (lane == 0) {
        const long long idx = perm[base + u];
        mbar_expect(&full[s], kUnit);
        const uint32_t piece = kUnit / pieces;
        if (split) {
          const size_t half = (size_t)1 << 31;
          bulk(sm + (size_t)s * kUnit, pool + (idx % (half / 16384)) * 16384, 16384, &full[s]);
          bulk(sm + (size_t)s * kUnit + 16384, pool + half + (idx % (half / 16384)) * 16384, 16384, &full[s]);
        } else {
          for (int k = 0; k < pieces; ++k)
            bulk(sm + (size_t)s * kUnit + k * piece, pool + idx * kUnit + k * piece, piece, &full[s]);
        }
      }
      __syncwarp();
    }
    return;
  }
  uint32_t acc = 0;
  for (int u = 0; u < units; ++u) {
    const int s = u % nst;
    mbar_wait(&full[s], (u / nst) & 1);
    acc ^= reinterpret_cast<const uint32_t*>(sm + (size_t)s * kUnit)[tid];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const size_t bytes = (size_t)4 << 30;
  char* pool;
  unsigned* sink;
  cudaMalloc(&pool, bytes);
  cudaMalloc(&sink, 64);
  cudaMemset(pool, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto best_of = [&](auto&& launch, int reps) {
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    return best;
  };
  printf("kind        ctas/sm nst pieces  GB/s\n");
  for (int cps : {4, 8, 16}) {
    const size_t n = bytes / 16;
    const float ms = best_of([&] { ldg_read<<<sms * cps, 256>>>((const uint4*)pool, n, sink); }, 5);
    printf("ldg.128     %-7d -   -       %.1f\n", cps, bytes / (ms * 1e-3) / 1e9);
  }
  const int total_units = (int)(bytes / 32768);
  std::vector<int> perm(total_units);
  uint32_t x = 12345;
  for (int i = 0; i < total_units; ++i) perm[i] = i;
  for (int i = total_units - 1; i > 0; --i) {  // scattered unit order
    x = x * 1664525u + 1013904223u;
    std::swap(perm[i], perm[x % (i + 1)]);
  }
  int* dperm;
  cudaMalloc(&dperm, perm.size() * 4);
  cudaMemcpy(dperm, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice);
  for (int cps : {1, 2, 3, 4, 6}) {
    for (int nst : {2, 3, 4, 6}) {
      const size_t smem = (size_t)nst * 32768;
      if (smem * cps > 220 * 1024 || smem > 227 * 1024) continue;
      cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int pieces : {1, 2, 8}) {
        const int ctas = sms * cps;
        const int units = total_units / ctas;
        const float ms =
            best_of([&] { ring<<<ctas, 160, smem>>>(pool, dperm, units, nst, pieces, sink); }, 5);
        printf("bulk ring   %-7d %-3d %-7d %.1f\n", cps, nst, pieces, (double)units * ctas * 32768 / (ms * 1e-3) / 1e9);
      }
    }
  }
  for (int cps : {1, 2}) {
    for (int nst : {2, 3, 4}) {
      const size_t smem = (size_t)nst * 32768;
      if (smem * cps > 220 * 1024) continue;
      cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int ctas = sms * cps;
      const int units = total_units / ctas / 2;
      const float ms = best_of([&] { ring<<<ctas, 160, smem>>>(pool, dperm, units, nst, 2, sink, 1); }, 5);
      printf("split K/V   %-7d %-3d 2x16K   %.1f\n", cps, nst, (double)units * ctas * 32768 / (ms * 1e-3) / 1e9);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
