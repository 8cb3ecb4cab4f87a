// K3 chunk-first phase on tensor cores (Alg 1; Eqn 1,
// PAPER.md:95-108; "turn the query from a vector into a matrix, allowing
// efficient matrix multiplications with tensor cores").
//
// One CTA = one tile (head, rows [r0, r1) of a shared run, chunks [k0, k1) of
// that run).  The run's rows are contiguous, so the query tile
// is a plain row gather.  The K and V tile of each (chunk, head) (c x d,
// 16-bit, contiguous and pre-swizzled in the pool) arrives by one 1-D bulk
// async copy each (cp.async.bulk, TMA engine) into an NST-stage ring with
// mbarrier completion; 8 warps = G row groups of 16 query rows x L token
// slices of the chunk, each running WarpAttn (mma.sync m16n8k16, fp32
// accumulate, online softmax) across the tile's chunks.  The L slices of a
// row group merge through shared memory in a fixed order and the tile writes
// one fp32 partial row (o | m n) per (row, head).
#include <algorithm>

#include "../host/schedule.h"
#include "common.cuh"
#include "kernels.h"
#include "mma_attn.cuh"

namespace pakv {

using namespace dev;

cudaError_t launch_chunk_first_simt(const AttnLaunch& a, const DevTables& t, cudaStream_t st);

namespace {

constexpr int kMaxStages = 8;

// kWarps consumer warps = G row groups x L chunk lanes, + 1 producer warp.
// Warp (g, l) owns query rows [16 g, 16 g + 16) of the tile and the chunks
// k = l, l + L, ... -- whole chunks, TPW tokens per MMA pass -- so L chunks
// are attended concurrently with no CTA-wide sync per chunk.  The producer
// warp refills a stage as soon as its G consumers release it.  kWarps = 4 (for
// tiles of <= 64 rows) keeps the CTA small enough for a seq-first CTA to run
// beside it on the same SM (PDL overlap of the two phases).
template <typename T, int D, int TPW, int kWarps>
__global__ void __launch_bounds__((kWarps + 1) * 32, 1)
    cf_mma_kernel(const T* __restrict__ kpool, const T* __restrict__ vpool, const T* __restrict__ q,
                  float* __restrict__ pO, DevTables t, int32_t h, int32_t C, int32_t L, float scale_log2,
                  int32_t nst, uint64_t* __restrict__ trace) {
  constexpr int kThreads = (kWarps + 1) * 32;
  using WA = WarpAttn<T, D, TPW>;
  constexpr int PR = D + 4;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages];
  __shared__ float sm_m[kWarps][16], sm_n[kWarps][16];
  __shared__ float sm_w[kWarps * 16][kWarps];  // per-row lane weights (epilogue)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int head = blockIdx.y;
  const int32_t* tile = t.cf_tile + blockIdx.x * kCfTileInts;
  const int chunk_off = tile[CF_CHUNK_OFF], n_chunks = tile[CF_NCHUNK], row0 = tile[CF_ROW0], row1 = tile[CF_ROW1];
  const int slot0 = tile[CF_SLOT];
  const int rows = row1 - row0;
  const int G = kWarps / L;  // row groups
  const int lslice = warp % L, rgroup = warp / L;
  const bool consumer = warp < kWarps;
  const bool active = consumer && rgroup * 16 < rows;
  const uint32_t tile_bytes = (uint32_t)C * D * 2;
  const uint32_t stage_bytes = 2 * tile_bytes;
  const uint32_t base_u32 = smem_u32(smem_raw);
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  uint64_t* tr = trace && cta < kTraceCtas ? trace + (size_t)cta * kTraceStride : nullptr;
  if (tr && tid == 0) tr[0] = globaltimer_ns();
  pdl_launch_dependents();  // seq-first may start streaming unchanged private chunks

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], G);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kWarps) {
    // ------------------------------------------------------------ producer
    // The whole warp walks the ring (warp-uniform waits, no lane spinning
    // while its siblings sit at the CTA barrier); lane 0 issues the copies.
    for (int k = 0; k < n_chunks; ++k) {
      const int s = k % nst;
      if (k >= nst) mbar_wait(&empty_bar[s], (uint32_t)(((k / nst) - 1) & 1));
      if (lane == 0) {
        const size_t off = ((size_t)t.cf_chunk[chunk_off + k] * h + head) * C * D;
        unsigned char* ks = smem_raw + s * stage_bytes;
        mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
        bulk_g2s(ks, kpool + off, tile_bytes, &full_bar[s]);
        bulk_g2s(ks + tile_bytes, vpool + off, tile_bytes, &full_bar[s]);
        if (tr && k < kTraceUnits) {
          tr[3 + 4 * k] = globaltimer_ns();
          tr[6 + 4 * k] = stage_bytes;
        }
      }
      __syncwarp();
    }
  }

  // Q fragments (A operand, row-major 16 x 16 per k-step), rows gathered by caller index
  uint32_t qa[WA::KS][4];
  WA wa;
  wa.reset();
  if (active) {
    const int rlo = row0 + rgroup * 16 + (lane >> 2), rhi = rlo + 8;
    const T* qlo = (active && rlo < row1) ? q + ((size_t)t.row_caller[rlo] * h + head) * D : nullptr;
    const T* qhi = (active && rhi < row1) ? q + ((size_t)t.row_caller[rhi] * h + head) * D : nullptr;
    const int cq = (lane & 3) * 2;
#pragma unroll
    for (int ks = 0; ks < WA::KS; ++ks) {
      qa[ks][0] = qlo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16 + cq) : 0u;
      qa[ks][1] = qhi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16 + cq) : 0u;
      qa[ks][2] = qlo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16 + 8 + cq) : 0u;
      qa[ks][3] = qhi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16 + 8 + cq) : 0u;
    }
  }
  if (consumer) {
    for (int k = lslice; k < n_chunks; k += L) {
      const int s = k % nst;
      mbar_wait(&full_bar[s], (uint32_t)((k / nst) & 1));
      if (tr && lane == 0 && rgroup == 0 && k < kTraceUnits) tr[4 + 4 * k] = globaltimer_ns();
      if (active) {
        const uint32_t ks_u32 = base_u32 + s * stage_bytes;
        for (int t0 = 0; t0 < C; t0 += TPW)
          wa.template chunk<false>(qa, ks_u32, ks_u32 + tile_bytes, t0, C, scale_log2, lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty_bar[s]);
      if (tr && lane == 0 && rgroup == 0 && k < kTraceUnits) tr[5 + 4 * k] = globaltimer_ns();
    }
  }
  wa.finish();
  __syncthreads();  // every stage drained (the epilogue reuses the ring)

  // ---- merge the L token slices of each row group (fixed order) -> partial
  float* smO = reinterpret_cast<float*>(smem_raw);  // [8 warps][16 rows][D]; stages are drained
  if (active) {
    const int rl = lane >> 2, cq = (lane & 3) * 2;
    if ((lane & 3) == 0) {
      sm_m[warp][rl] = wa.m_lo;
      sm_n[warp][rl] = wa.n_lo;
      sm_m[warp][rl + 8] = wa.m_hi;
      sm_n[warp][rl + 8] = wa.n_hi;
    }
#pragma unroll
    for (int i = 0; i < WA::DT; ++i) {
      float* lo = smO + ((size_t)warp * 16 + rl) * D + i * 8 + cq;
      *reinterpret_cast<float2*>(lo) = make_float2(wa.o[i][0], wa.o[i][1]);
      *reinterpret_cast<float2*>(lo + 8 * D) = make_float2(wa.o[i][2], wa.o[i][3]);
    }
  }
  __syncthreads();
  if (tid < rows) {  // per-row rebase weights of the L slices (n-ary Eqn 2), once per row
    const int g = tid >> 4, r16 = tid & 15;
    float M = -INFINITY;
    for (int l = 0; l < L; ++l) M = fmaxf(M, sm_m[g * L + l][r16]);
    float ns = 0.f;
    for (int l = 0; l < L; ++l) {
      const float w = fast_exp2(sm_m[g * L + l][r16] - M);
      sm_w[tid][l] = w;
      ns = fmaf(w, sm_n[g * L + l][r16], ns);
    }
    float* prow = pO + ((size_t)(slot0 + tid) * h + head) * PR;
    *reinterpret_cast<float4*>(prow + D) = make_float4(M, ns, 0.f, 0.f);
  }
  __syncthreads();
  for (int idx = tid; idx < rows * (D / 4); idx += kThreads) {
    const int rloc = idx / (D / 4), x4 = (idx - rloc * (D / 4)) * 4;
    const int g = rloc >> 4, r16 = rloc & 15;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int l = 0; l < L; ++l) {
      const float w = sm_w[rloc][l];
      const float4 v = *reinterpret_cast<const float4*>(smO + ((size_t)(g * L + l) * 16 + r16) * D + x4);
      acc.x = fmaf(w, v.x, acc.x);
      acc.y = fmaf(w, v.y, acc.y);
      acc.z = fmaf(w, v.z, acc.z);
      acc.w = fmaf(w, v.w, acc.w);
    }
    *reinterpret_cast<float4*>(pO + ((size_t)(slot0 + rloc) * h + head) * PR + x4) = acc;
  }
  if (tr && tid == 0) {
    tr[1] = tr[2] = globaltimer_ns();
  }
  // PDL chain append -> chunk-first -> seq-first: this grid started before the
  // append finished; do not complete before it, so seq-first's single wait
  // covers both predecessors.
  pdl_wait();
}

template <typename T, int D, int TPW, int W>
cudaError_t launch_mma(const AttnLaunch& a, const DevTables& t, int L, size_t budget, cudaStream_t st) {
  const PoolGeom& p = a.pool;
  const size_t stage = (size_t)2 * p.c * D * 2;
  int nst = (int)std::min<size_t>(kMaxStages, budget / stage);
  nst = std::max(2, nst);
  const size_t epi = (size_t)W * 16 * D * 4;
  const size_t smem = std::max(nst * stage, epi);
  auto kern = cf_mma_kernel<T, D, TPW, W>;
  // max shared-memory carveout: a seq-first CTA can fit beside this one (PDL overlap)
  cudaError_t e = set_smem_once((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  const T* kp = (const T*)p.k + (size_t)a.layer * p.layer_stride;
  const T* vp = (const T*)p.v + (size_t)a.layer * p.layer_stride;
  return launch_ex(kern, dim3(t.n_cf_tiles, p.h), dim3((W + 1) * 32), smem, st, a.use_pdl, kp, vp, (const T*)a.q,
                   a.pO, t, (int32_t)p.h, (int32_t)p.c, (int32_t)L, a.scale_log2, (int32_t)nst,
                   a.trace_cf ? a.trace : (uint64_t*)nullptr);
}

template <typename T, int W>
cudaError_t dispatch_mma(const AttnLaunch& a, const DevTables& t, int tpw, int L, size_t budget, cudaStream_t st) {
  const int d = a.pool.d;
#define CA_CASE(DD, TT) \
  if (d == DD && tpw == TT) return launch_mma<T, DD, TT, W>(a, t, L, budget, st);
  CA_CASE(64, 16) CA_CASE(64, 32) CA_CASE(64, 64) CA_CASE(128, 16) CA_CASE(128, 32) CA_CASE(128, 64)
#undef CA_CASE
  return cudaErrorInvalidValue;
}

// chunk lanes L (= warps per row group; G = W / L row groups of 16 rows) and
// tokens per MMA pass TPW (a warp walks its whole chunk in TPW-token passes)
bool pick_slices(int c, int max_rows, int warps, int* L, int* tpw) {
  int groups = 1;
  while (groups * 16 < max_rows) groups *= 2;
  if (groups > warps) return false;
  *L = warps / groups;
  *tpw = c % 64 == 0 ? 64 : (c % 32 == 0 ? 32 : 16);
  return true;
}

}  // namespace

bool cf_mma_supported(const PoolGeom& p) {
  return (p.dtype == DT_F16 || p.dtype == DT_BF16) && (p.d == 64 || p.d == 128) && p.c % 16 == 0 && p.c >= 16 &&
         p.c <= 256;
}

cudaError_t launch_chunk_first(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (t.n_cf_tiles == 0) return cudaSuccess;
  int L = 1, tpw = 16;
  // small CTA (4 consumer warps, ~100 KB ring) when the tiles allow it, so a
  // seq-first CTA fits beside it; 8 warps for tiles of up to 128 rows
  if (a.cf_tensor_cores && a.cf_umma && cf_umma_supported(a.pool, t.max_tile_rows))
    return launch_chunk_first_umma(a, t, st);
  const bool small = a.cf_small && t.max_tile_rows <= 64;
  const int warps = small ? 4 : 8;
  if (!a.cf_tensor_cores || !cf_mma_supported(a.pool) || !pick_slices(a.pool.c, t.max_tile_rows, warps, &L, &tpw))
    return launch_chunk_first_simt(a, t, st);
  if (a.pool.d == 128 && tpw == 64) tpw = 32;  // keeps the d = 128 warp state under the register cap
  const size_t budget = small ? (size_t)100 * 1024 : (size_t)200 * 1024;
  if (small) {
    if (a.pool.dtype == DT_F16) return dispatch_mma<__half, 4>(a, t, tpw, L, budget, st);
    return dispatch_mma<__nv_bfloat16, 4>(a, t, tpw, L, budget, st);
  }
  if (a.pool.dtype == DT_F16) return dispatch_mma<__half, 8>(a, t, tpw, L, budget, st);
  return dispatch_mma<__nv_bfloat16, 8>(a, t, tpw, L, budget, st);
}

}  // namespace pakv
