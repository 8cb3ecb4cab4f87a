// Probe of the tcgen05 (UMMA) operand layouts the chunk-first phase would use
// (SURVEY §8 f3), checked against a CPU matmul:
//   S[128][c]   = Q[128][128] . K[c][128]^T     A = Q  K-major SW128 (2 d-halves)
//                                               B = K  K-major SW128 (pool tile halves)
//   O[128][128] = P[128][c] . V[c][128]         A = P  K-major SW128 (one 128-B atom column)
//                                               B = V  MN-major SW128 (LBO = half stride)
// Smem images: a d-half h of a [rows][128 d] 16-bit tile is [rows][64] with
// row r's 16-byte group j at r * 128 + ((j ^ (r & 7)) * 16) -- exactly the
// pool's per-row XOR pre-swizzle applied within each 128-byte half.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_probe tools/umma_probe.cu
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

#ifndef PROBE_M
#define PROBE_M 128
#endif
// M = 64 (-DPROBE_M=64): the accumulator's TMEM lane of every row is found by
// matching each lane's S row against the CPU rows (printed as a lane map)
constexpr int C = 64, D = 128, M = PROBE_M;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n, bool b_mn_major) {
  return (1u << 4)                        // D = f32
         | (0u << 7) | (0u << 10)          // A, B = f16
         | ((b_mn_major ? 1u : 0u) << 16)  // B major
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(ph)
      : "memory");
}
// one 16-byte group of a swizzled half-tile image
__device__ __forceinline__ uint32_t sw_off(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }

__device__ __forceinline__ void tmem_ld32(uint32_t addr, float* v) {  // 32 columns, this thread's lane
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// q [M][D], k, v: pool tile [C][D] (row-swizzled groups: group g of token t at g ^ (t & 7)), p [M][C]
__global__ void probe(const __half* q, const __half* kt, const __half* vt, const __half* p, float* s_out,
                      float* o_out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = sm;                   // 2 halves x M x 128 B = 32 KB
  unsigned char* sK = sQ + 2 * M * 128;     // 2 halves x C x 128 B = 16 KB
  unsigned char* sV = sK + 2 * C * 128;     // 16 KB
  unsigned char* sP = sV + 2 * C * 128;     // M x 128 B = 16 KB (C = 64 tokens)
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // images: Q and P written swizzled from linear rows; K and V taken from the
  // pool tile, whose rows are already XOR-swizzled within each 128-B half
  for (int i = tid; i < M * 16; i += blockDim.x) {
    const int r = i / 16, g = i % 16, h = g / 8, j = g % 8;
    *reinterpret_cast<uint4*>(sQ + h * M * 128 + sw_off(r, j)) = reinterpret_cast<const uint4*>(q + r * D)[g];
  }
  for (int i = tid; i < C * 16; i += blockDim.x) {
    const int t = i / 16, gp = i % 16, h = gp / 8;  // gp = physical group in the pool row
    *reinterpret_cast<uint4*>(sK + h * C * 128 + t * 128 + (gp % 8) * 16) = reinterpret_cast<const uint4*>(kt + t * D)[gp];
    *reinterpret_cast<uint4*>(sV + h * C * 128 + t * 128 + (gp % 8) * 16) = reinterpret_cast<const uint4*>(vt + t * D)[gp];
  }
  for (int i = tid; i < M * 8; i += blockDim.x) {
    const int r = i / 8, j = i % 8;
    *reinterpret_cast<uint4*>(sP + sw_off(r, j)) = reinterpret_cast<const uint4*>(p + r * C)[j];
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
  const uint32_t tS = tmem_base, tO = tmem_base + 64;
  if (tid == 0) {
    const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK), va = smem_u32(sV), pa = smem_u32(sP);
    for (int ks = 0; ks < D / 16; ++ks) {  // S = Q K^T, K = d
      const int h = ks / 4, o = (ks % 4) * 32;
      umma(tS, sdesc(qa + h * M * 128 + o, 16, 1024), sdesc(ka + h * C * 128 + o, 16, 1024), idesc_f16(M, C, false),
           ks > 0);
    }
    for (int ks = 0; ks < C / 16; ++ks)  // O = P V, K = tokens; B MN-major, N = 128 over both d-halves
      umma(tO, sdesc(pa + ks * 32, 16, 1024), sdesc(va + ks * 16 * 128, C * 128, 1024), idesc_f16(M, D, true), ks > 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + (tid & 31);  // TMEM lane (all 128)
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  float v[32];
  for (int c0 = 0; c0 < C; c0 += 32) {
    tmem_ld32(tS + lane_off + c0, v);
    for (int i = 0; i < 32; ++i) s_out[row * C + c0 + i] = v[i];
  }
  for (int c0 = 0; c0 < D; c0 += 32) {
    tmem_ld32(tO + lane_off + c0, v);
    for (int i = 0; i < 32; ++i) o_out[row * D + c0 + i] = v[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
}

int main() {
  std::vector<__half> q(M * D), k(C * D), v(C * D), p(M * C);
  std::vector<float> qf(M * D), kf(C * D), vf(C * D), pf(M * C);
  srand(1);
  auto rnd = [] { return (float)((rand() % 2001) - 1000) / 1000.f; };
  for (int i = 0; i < M * D; ++i) { q[i] = __float2half(rnd()); qf[i] = __half2float(q[i]); }
  for (int i = 0; i < M * C; ++i) { p[i] = __float2half(rnd()); pf[i] = __half2float(p[i]); }
  // pool tile: logical group g of token t stored at physical group g ^ (t & 7)
  std::vector<__half> kp(C * D), vp(C * D);
  for (int t = 0; t < C; ++t)
    for (int e = 0; e < D; ++e) {
      kf[t * D + e] = __half2float(__float2half(rnd()));
      vf[t * D + e] = __half2float(__float2half(rnd()));
      const int g = e / 8, pg = g ^ (t & 7);
      kp[t * D + pg * 8 + e % 8] = __float2half(kf[t * D + e]);
      vp[t * D + pg * 8 + e % 8] = __float2half(vf[t * D + e]);
    }
  __half *dq, *dk, *dv, *dp;
  float *ds, *dout;
  CK(cudaMalloc(&dq, 2 * M * D));
  CK(cudaMalloc(&dk, 2 * C * D));
  CK(cudaMalloc(&dv, 2 * C * D));
  CK(cudaMalloc(&dp, 2 * M * C));
  CK(cudaMalloc(&ds, 4 * 128 * C));
  CK(cudaMalloc(&dout, 4 * 128 * D));
  CK(cudaMemcpy(dq, q.data(), 2 * M * D, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk, kp.data(), 2 * C * D, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, vp.data(), 2 * C * D, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dp, p.data(), 2 * M * C, cudaMemcpyHostToDevice));
  const int smem = 2 * M * 128 + 4 * C * 128 + M * 128 + 1024;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<<<1, 128, smem>>>(dq, dk, dv, dp, ds, dout);
  CK(cudaDeviceSynchronize());
  std::vector<float> s(128 * C), o(128 * D);
  CK(cudaMemcpy(s.data(), ds, 4 * 128 * C, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(o.data(), dout, 4 * 128 * D, cudaMemcpyDeviceToHost));
  std::vector<int> lane_of(M, -1);
  if (M != 128) {  // find each row's lane
    for (int r = 0; r < M; ++r)
      for (int L = 0; L < 128 && lane_of[r] < 0; ++L) {
        double e = 0;
        for (int t = 0; t < C; ++t) {
          double a = 0;
          for (int k = 0; k < D; ++k) a += (double)qf[r * D + k] * kf[t * D + k];
          e = fmax(e, fabs(a - s[L * C + t]));
        }
        if (e < 1e-2) lane_of[r] = L;
      }
    printf("M=%d row -> TMEM lane:", M);
    for (int r = 0; r < M; ++r) printf(" %d:%d", r, lane_of[r]);
    printf("\n");
  } else {
    for (int r = 0; r < M; ++r) lane_of[r] = r;
  }
  double es = 0, eo = 0;
  for (int r = 0; r < M; ++r)
    for (int t = 0; t < C; ++t) {
      double a = 0;
      for (int e = 0; e < D; ++e) a += (double)qf[r * D + e] * kf[t * D + e];
      es = fmax(es, lane_of[r] < 0 ? 1e9 : fabs(a - s[lane_of[r] * C + t]));
    }
  for (int r = 0; r < M; ++r)
    for (int e = 0; e < D; ++e) {
      double a = 0;
      for (int t = 0; t < C; ++t) a += (double)pf[r * C + t] * vf[t * D + e];
      eo = fmax(eo, lane_of[r] < 0 ? 1e9 : fabs(a - o[lane_of[r] * D + e]));
    }
  printf("S = Q K^T  max abs err %.3e  (S[0][0] %f S[5][7] %f)\n", es, s[0], s[5 * C + 7]);
  printf("O = P V    max abs err %.3e  (O[0][0] %f O[9][100] %f)\n", eo, o[0], o[9 * D + 100]);
  printf("%s\n", (es < 1e-2 && eo < 1e-2) ? "PROBE OK" : "PROBE MISMATCH");
  return 0;
}
