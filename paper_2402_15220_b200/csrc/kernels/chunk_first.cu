// K3 chunk-first phase on tensor cores (Alg 1; Eqn 1,
// PAPER.md:95-108; "turn the query from a vector into a matrix, allowing
// efficient matrix multiplications with tensor cores").
//
// One CTA = one tile (head, rows [r0, r1) of a shared run, chunks [k0, k1) of
// that run).  The run's rows are contiguous, so the query tile
// is a plain row gather.  K and V tiles of each (chunk, head) (c x d, 16-bit)
// arrive by TMA (cp.async.bulk.tensor.2d, 128-byte swizzle, 64-column boxes)
// into an NST-stage ring with mbarrier completion; 8 warps = G row groups of
// 16 query rows x L token slices of the chunk; every warp computes
// S = Q K^T (mma.sync m16n8k16, fp32 accumulate), its online softmax
// (exp2, log2(e) folded into the scale; P rounded to the input type and the
// row sum n taken from the rounded P, reading A11) and O += P V, keeping
// (O, m, n) in registers across the tile's chunks (Eqn 2 applied in-CTA,
// PAPER.md:145-158).  The L slices of a row group merge through shared memory
// in fixed order and the tile writes one fp32 partial (O, m, n) per row.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace pakv {

using namespace dev;

cudaError_t launch_chunk_first_simt(const AttnLaunch& a, const DevTables& t, cudaStream_t st);

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxStages = 4;

// byte offset of element (row, col) in a [D/64][C][64] 16-bit tile with the
// 128-byte TMA swizzle (16-byte chunk index XOR row % 8)
CA_DEV uint32_t swz(int row, int col, int C) {
  const int box = col >> 6, c64 = col & 63;
  return (uint32_t)(box * C * 128 + row * 128 + ((((c64 >> 3) ^ (row & 7))) << 4) + (c64 & 7) * 2);
}

template <typename T, int D, int TPW>
__global__ void __launch_bounds__(kThreads, 1)
    cf_mma_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const T* __restrict__ q, float* __restrict__ pO, float2* __restrict__ pMN, DevTables t,
                  int32_t h, int32_t C, int32_t L, int64_t layer_rows, float scale_log2, int32_t nst) {
  constexpr int KS = D / 16;   // k-steps over d
  constexpr int NT = TPW / 8;  // n-tiles of S per warp
  constexpr int DT = D / 8;    // n-tiles of O
  extern __shared__ unsigned char smem_raw[];
  __shared__ uint64_t bars[kMaxStages];
  __shared__ float sm_m[kWarps][16], sm_n[kWarps][16];

  pdl_launch_dependents();  // let the seq-first grid start its private work early

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int head = blockIdx.y;
  const int32_t* tile = t.cf_tile + blockIdx.x * 8;
  const int chunk_off = tile[0], n_chunks = tile[1], row0 = tile[2], row1 = tile[3], slot0 = tile[4];
  const int rows = row1 - row0;
  const int lslice = warp % L, rgroup = warp / L;
  const bool active = rgroup * 16 < rows;

  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  const uint32_t tile_bytes = (uint32_t)C * D * 2;
  const uint32_t stage_bytes = 2 * tile_bytes;

  if (tid == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    for (int s = 0; s < nst; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  auto issue = [&](int k) {
    const int s = k % nst;
    const int cid = t.cf_chunk[chunk_off + k];
    const int32_t rc = (int32_t)(layer_rows + ((int64_t)cid * h + head) * C);
    unsigned char* ks = base + s * stage_bytes;
    unsigned char* vs = ks + tile_bytes;
    mbar_arrive_expect_tx(&bars[s], stage_bytes);
#pragma unroll
    for (int bx = 0; bx < D / 64; ++bx) {
      tma_load_2d(ks + bx * C * 128, &tmK, bx * 64, rc, &bars[s]);
      tma_load_2d(vs + bx * C * 128, &tmV, bx * 64, rc, &bars[s]);
    }
  };
  if (tid == 0)
    for (int k = 0; k < min(nst, n_chunks); ++k) issue(k);

  // Q fragments (A operand, row-major 16 x 16 per k-step), rows gathered by caller index
  uint32_t qa[KS][4];
  {
    const int rlo = row0 + rgroup * 16 + (lane >> 2), rhi = rlo + 8;
    const T* qlo = (active && rlo < row1) ? q + ((size_t)t.row_caller[rlo] * h + head) * D : nullptr;
    const T* qhi = (active && rhi < row1) ? q + ((size_t)t.row_caller[rhi] * h + head) * D : nullptr;
    const int cq = (lane & 3) * 2;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      qa[ks][0] = qlo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16 + cq) : 0u;
      qa[ks][1] = qhi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16 + cq) : 0u;
      qa[ks][2] = qlo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16 + 8 + cq) : 0u;
      qa[ks][3] = qhi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16 + 8 + cq) : 0u;
    }
  }

  float o[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, n_lo = 0.f, n_hi = 0.f;
  const int tok0 = lslice * TPW;
  const int mi = lane >> 3, r8 = lane & 7;

  for (int k = 0; k < n_chunks; ++k) {
    const int s = k % nst;
    mbar_wait(&bars[s], (uint32_t)((k / nst) & 1));
    if (active) {
      const uint32_t ks_u32 = base_u32 + s * stage_bytes;
      const uint32_t vs_u32 = ks_u32 + tile_bytes;
      float sc[NT][4];
#pragma unroll
      for (int i = 0; i < NT; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
      // S = Q K^T
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int np = 0; np < NT / 2; ++np) {
          uint32_t b0, b1, b2, b3;
          const int tok = tok0 + np * 16 + (mi >> 1) * 8 + r8;
          ldmatrix_x4(ks_u32 + swz(tok, ks * 16 + (mi & 1) * 8, C), b0, b1, b2, b3);
          Mma<T>::run(sc[2 * np], qa[ks], b0, b1);
          Mma<T>::run(sc[2 * np + 1], qa[ks], b2, b3);
        }
      }
      // online softmax (two rows per thread: lo = lane/4, hi = lane/4 + 8)
      float mx_lo = -INFINITY, mx_hi = -INFINITY;
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        mx_lo = fmaxf(mx_lo, fmaxf(sc[i][0], sc[i][1]));
        mx_hi = fmaxf(mx_hi, fmaxf(sc[i][2], sc[i][3]));
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, off));
        mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, off));
      }
      const float mn_lo = fmaxf(m_lo, mx_lo * scale_log2);
      const float mn_hi = fmaxf(m_hi, mx_hi * scale_log2);
      const float c_lo = fast_exp2(m_lo - mn_lo), c_hi = fast_exp2(m_hi - mn_hi);
      m_lo = mn_lo;
      m_hi = mn_hi;
      uint32_t pa[NT][2];
      float ps_lo = 0.f, ps_hi = 0.f;
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        pa[i][0] = Mma<T>::pack(fast_exp2(fmaf(sc[i][0], scale_log2, -mn_lo)),
                                fast_exp2(fmaf(sc[i][1], scale_log2, -mn_lo)));
        pa[i][1] = Mma<T>::pack(fast_exp2(fmaf(sc[i][2], scale_log2, -mn_hi)),
                                fast_exp2(fmaf(sc[i][3], scale_log2, -mn_hi)));
        const float2 fl = Mma<T>::unpack(pa[i][0]), fh = Mma<T>::unpack(pa[i][1]);
        ps_lo += fl.x + fl.y;
        ps_hi += fh.x + fh.y;
      }
      n_lo = n_lo * c_lo + ps_lo;
      n_hi = n_hi * c_hi + ps_hi;
#pragma unroll
      for (int i = 0; i < DT; ++i) {
        o[i][0] *= c_lo;
        o[i][1] *= c_lo;
        o[i][2] *= c_hi;
        o[i][3] *= c_hi;
      }
      // O += P V
#pragma unroll
      for (int kk = 0; kk < TPW / 16; ++kk) {
        const uint32_t a[4] = {pa[2 * kk][0], pa[2 * kk][1], pa[2 * kk + 1][0], pa[2 * kk + 1][1]};
#pragma unroll
        for (int dp = 0; dp < DT / 2; ++dp) {
          uint32_t b0, b1, b2, b3;
          const int tok = tok0 + kk * 16 + (mi & 1) * 8 + r8;
          ldmatrix_x4_trans(vs_u32 + swz(tok, dp * 16 + (mi >> 1) * 8, C), b0, b1, b2, b3);
          Mma<T>::run(o[2 * dp], a, b0, b1);
          Mma<T>::run(o[2 * dp + 1], a, b2, b3);
        }
      }
    }
    __syncthreads();  // stage s fully consumed
    if (tid == 0 && k + nst < n_chunks) issue(k + nst);
  }

  // ---- merge the L token slices of each row group (fixed order) -> partial
  n_lo += __shfl_xor_sync(0xffffffffu, n_lo, 1);
  n_lo += __shfl_xor_sync(0xffffffffu, n_lo, 2);
  n_hi += __shfl_xor_sync(0xffffffffu, n_hi, 1);
  n_hi += __shfl_xor_sync(0xffffffffu, n_hi, 2);
  float* smO = reinterpret_cast<float*>(base);  // [8 warps][16 rows][D]; stages are drained
  if (active) {
    const int rl = lane >> 2, cq = (lane & 3) * 2;
    if ((lane & 3) == 0) {
      sm_m[warp][rl] = m_lo;
      sm_n[warp][rl] = n_lo;
      sm_m[warp][rl + 8] = m_hi;
      sm_n[warp][rl + 8] = n_hi;
    }
#pragma unroll
    for (int i = 0; i < DT; ++i) {
      float* lo = smO + ((size_t)warp * 16 + rl) * D + i * 8 + cq;
      float* hi = lo + 8 * D;
      *reinterpret_cast<float2*>(lo) = make_float2(o[i][0], o[i][1]);
      *reinterpret_cast<float2*>(hi) = make_float2(o[i][2], o[i][3]);
    }
  }
  __syncthreads();
  for (int idx = tid; idx < rows * D; idx += kThreads) {
    const int rloc = idx / D, x = idx - rloc * D;
    const int g = rloc >> 4, r16 = rloc & 15;
    float ao = 0.f, am = -INFINITY, an = 0.f;
    for (int l = 0; l < L; ++l) {
      const int w = g * L + l;
      const float mc = sm_m[w][r16], nc = sm_n[w][r16], oc = smO[((size_t)w * 16 + r16) * D + x];
      const float mx = fmaxf(am, mc);
      const float xa = fast_exp2(mc - mx), ya = fast_exp2(am - mx);
      ao = xa * oc + ya * ao;
      an = xa * nc + ya * an;
      am = mx;
    }
    float* prow = pO + ((size_t)(slot0 + rloc) * h + head) * (D + 4);  // [o | m n pad pad]
    prow[x] = ao;
    if (x == 0) *reinterpret_cast<float4*>(prow + D) = make_float4(am, an, 0.f, 0.f);
  }
}

template <typename T, int D, int TPW>
cudaError_t launch_mma(const AttnLaunch& a, const DevTables& t, int L, cudaStream_t st) {
  const PoolGeom& p = a.pool;
  const size_t stage = (size_t)2 * p.c * D * 2;
  int nst = (int)std::min<size_t>(kMaxStages, (size_t)(192 * 1024) / stage);
  nst = std::max(1, nst);
  const size_t epi = (size_t)kWarps * 16 * D * 4;
  const size_t smem = 1024 + std::max(nst * stage, epi);
  auto kern = cf_mma_kernel<T, D, TPW>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t layer_rows = (int64_t)a.layer * p.max_chunks * p.h * p.c;
  kern<<<dim3(t.n_cf_tiles, p.h), kThreads, smem, st>>>(*a.tmap_k, *a.tmap_v, (const T*)a.q, a.pO, a.pMN, t, p.h,
                                                          p.c, L, layer_rows, a.scale_log2, nst);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_mma(const AttnLaunch& a, const DevTables& t, int tpw, int L, cudaStream_t st) {
  const int d = a.pool.d;
#define CA_CASE(DD, TT) \
  if (d == DD && tpw == TT) return launch_mma<T, DD, TT>(a, t, L, st);
  CA_CASE(64, 16) CA_CASE(64, 32) CA_CASE(64, 64) CA_CASE(128, 16) CA_CASE(128, 32) CA_CASE(128, 64)
#undef CA_CASE
  return cudaErrorInvalidValue;
}

}  // namespace

bool cf_mma_supported(const PoolGeom& p) {
  return (p.dtype == DT_F16 || p.dtype == DT_BF16) && (p.d == 64 || p.d == 128) && p.c % 16 == 0 && p.c >= 16 &&
         p.c <= 256;
}

// token slices per chunk L (warps per row group) and tokens per warp TPW for a launch
static bool pick_slices(int c, int max_rows, int* L, int* tpw) {
  const int groups = std::max(1, (max_rows + 15) / 16);  // <= 8
  int l = std::min(8 / groups, c / 16);
  while (l > 1 && (8 % l != 0 || c % l != 0 || (c / l) % 16 != 0)) --l;
  const int tp = c / l;
  if (tp > 64 || groups * l > 8) return false;
  *L = l;
  *tpw = tp;
  return true;
}

cudaError_t launch_chunk_first(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (t.n_cf_tiles == 0) return cudaSuccess;
  int L = 1, tpw = 16;
  if (!a.cf_tensor_cores || !cf_mma_supported(a.pool) || !pick_slices(a.pool.c, t.max_tile_rows, &L, &tpw))
    return launch_chunk_first_simt(a, t, st);
  if (a.pool.dtype == DT_F16) return dispatch_mma<__half>(a, t, tpw, L, st);
  return dispatch_mma<__nv_bfloat16>(a, t, tpw, L, st);
}

bool make_pool_tmaps(const PoolGeom& p, CUtensorMap* tk, CUtensorMap* tv) {
  if (!cf_mma_supported(p)) return false;
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn)
      return false;
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t rows = (cuuint64_t)p.num_layers * p.max_chunks * p.h * p.c;
  const cuuint64_t dims[2] = {(cuuint64_t)p.d, rows};
  const cuuint64_t strides[1] = {(cuuint64_t)p.d * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)p.c};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt =
      p.dtype == DT_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  for (int which = 0; which < 2; ++which) {
    CUresult r = encode(which ? tv : tk, dt, 2, which ? p.v : p.k, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
  }
  return true;
}

}  // namespace pakv
