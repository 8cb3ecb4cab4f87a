// Probe: tcgen05.mma with the A operand in TMEM (M = 64, kind::f16), and the
// .16x128b TMEM store layout -- what keeping P (and Q) in tensor memory needs.
//   O[64][128] = P[64][64] . V[64][128]: A = P in TMEM (row r in the M = 64 lane
//   of D, lane (r / 16) * 32 + r % 16; 32-bit column c = tokens 2c, 2c + 1),
//   B = V MN-major SW128 in shared memory (as the chunk-first kernels use it).
// Prints the max error vs a CPU matmul, then the (lane, column) that every
// register of a .16x128b.x2 store lands in.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_tmema_probe tools/umma_tmema_probe.cu
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int C = 64, D = 128, M = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n, bool b_mn_major) {
  return (1u << 4) | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ uint32_t sw_off(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }

__global__ void probe(const __half* p, const __half* vt, float* o_out, int* map_out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sV = sm;  // 2 halves x C x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < C * 16; i += blockDim.x) {
    const int t = i / 16, gp = i % 16, h = gp / 8;
    *reinterpret_cast<uint4*>(sV + h * C * 128 + t * 128 + (gp % 8) * 16) = reinterpret_cast<const uint4*>(vt + t * D)[gp];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tP = tmem_base, tO = tmem_base + 64, tX = tmem_base + 192;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  {  // P into TMEM, 32x32b: thread (warp, lane < 16) = row 16 warp + lane
    uint32_t r[32];
    const int row = warp * 16 + (lane & 15);
    for (int c = 0; c < 32; ++c) {
      __half2 h2 = __halves2half2(p[row * C + 2 * c], p[row * C + 2 * c + 1]);
      r[c] = lane < 16 ? *reinterpret_cast<uint32_t*>(&h2) : 0u;
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tP + lane_base),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t va = smem_u32(sV);
    for (int ks = 0; ks < C / 16; ++ks)
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tO),
          "r"(tP + (uint32_t)(ks * 8)), "l"(sdesc(va + ks * 16 * 128, C * 128, 1024)), "r"(idesc_f16(M, D, true)),
          "r"(ks > 0 ? 1 : 0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < D; c0 += 32) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tO + lane_base + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) o_out[(warp * 32 + lane) * D + c0 + i] = __uint_as_float(r[i]);
  }
  // .16x128b.x2 store: every register carries its (thread, register) id; read back with 32x32b
  {
    uint32_t r[4];
    for (int i = 0; i < 4; ++i) r[i] = 0x10000u + (uint32_t)(tid * 16 + i);
    asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1, %2, %3, %4};" ::"r"(tX + lane_base), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t q[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
                 : "r"(tX + lane_base));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) map_out[(warp * 32 + lane) * 8 + i] = (int)q[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
}

int main() {
  std::vector<__half> p(M * C), vp(C * D);
  std::vector<float> pf(M * C), vf(C * D);
  srand(3);
  auto rnd = [] { return (float)((rand() % 2001) - 1000) / 1000.f; };
  for (int i = 0; i < M * C; ++i) { p[i] = __float2half(rnd()); pf[i] = __half2float(p[i]); }
  for (int t = 0; t < C; ++t)
    for (int e = 0; e < D; ++e) {
      vf[t * D + e] = __half2float(__float2half(rnd()));
      const int g = e / 8, pg = g ^ (t & 7);
      vp[t * D + pg * 8 + e % 8] = __float2half(vf[t * D + e]);
    }
  __half *dp, *dv;
  float* dout;
  int* dmap;
  cudaMalloc(&dp, 2 * M * C);
  cudaMalloc(&dv, 2 * C * D);
  cudaMalloc(&dout, 4 * 128 * D);
  cudaMalloc(&dmap, 4 * 128 * 8);
  cudaMemcpy(dp, p.data(), 2 * M * C, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, vp.data(), 2 * C * D, cudaMemcpyHostToDevice);
  const int smem = 2 * C * 128 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dp, dv, dout, dmap);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> o(128 * D);
  std::vector<int> map(128 * 8);
  cudaMemcpy(o.data(), dout, 4 * 128 * D, cudaMemcpyDeviceToHost);
  cudaMemcpy(map.data(), dmap, 4 * 128 * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int r = 0; r < M; ++r) {
    const int L = (r / 16) * 32 + r % 16;
    for (int e2 = 0; e2 < D; ++e2) {
      double a = 0;
      for (int t = 0; t < C; ++t) a += (double)pf[r * C + t] * vf[t * D + e2];
      err = fmax(err, fabs(a - o[L * D + e2]));
    }
  }
  printf("O = P(TMEM) V  max abs err %.3e  (O[0][0] %f)\n", err, o[0]);
  printf(".16x128b.x2 store: (lane, column) <- thread.register\n");
  for (int L : {0, 1, 2, 3, 4, 8, 15, 16, 31, 32}) {
    printf("lane %3d:", L);
    for (int i = 0; i < 8; ++i) {
      const int v = map[L * 8 + i];
      if (v >= 0x10000) printf(" c%d=t%d.r%d", i, (v - 0x10000) / 16, (v - 0x10000) % 16);
      else printf(" c%d=-", i);
    }
    printf("\n");
  }
  printf("%s\n", err < 1e-2 ? "PROBE OK" : "PROBE MISMATCH");
  return 0;
}
