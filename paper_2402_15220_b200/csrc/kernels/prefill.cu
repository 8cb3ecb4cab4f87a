// Prefill attention with prefix lookup (§3.1:
// "prefix lookup to avoid repeated computation of KV projection").  After
// chunkattn_add_sequence has matched the longest cached prefix and written the
// K/V of the unmatched suffix into the pool, every suffix query attends
// causally over its sequence's whole context in the pool -- the matched
// (shared) chunks plus the new ones:  out_p = softmax(s q_p K[0..p]^T) V[0..p]
// for each query position p (the per-row definition of PAPER.md:344 with the
// causal mask of prefill).
//
// CTA = (tile of <= 64 consecutive query positions of one sequence, head):
// 4 warps x 16 query rows on mma.sync (WarpAttn, causal mask on the chunks
// that straddle the tile's positions), the sequence's chunks streamed through
// a 2-stage shared-memory ring by 1-D bulk copies (pool tiles are pre-swizzled,
// one copy per K / V tile), online softmax across chunks (Eqn 2), O / n in the
// epilogue.  Chunks past the tile's last position are not read.
#include "common.cuh"
#include "kernels.h"
#include "mma_attn.cuh"

namespace pakv {

using namespace dev;

namespace {

constexpr int kPfWarps = 4;
constexpr int kPfRows = 16 * kPfWarps;
constexpr int kPfStages = 2;

template <typename T, typename TO, int D>
__global__ void __launch_bounds__(kPfWarps * 32) prefill_kernel(const T* __restrict__ kpool,
                                                               const T* __restrict__ vpool,
                                                               const T* __restrict__ q, TO* __restrict__ out,
                                                               const int32_t* __restrict__ tiles,
                                                               const int32_t* __restrict__ chunks, int32_t h,
                                                               int32_t c, float scale_log2) {
  using WA = WarpAttn<T, D, 16>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kPfStages];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int head = blockIdx.y;
  const int4 tr = *reinterpret_cast<const int4*>(tiles + (size_t)blockIdx.x * kPfTileInts);
  const int chunk_off = tr.x, q_row0 = tr.y, nq = tr.z, pos0 = tr.w;
  const int seq_len = tiles[(size_t)blockIdx.x * kPfTileInts + 4];
  const int last_pos = pos0 + nq - 1;
  const int n_chunks = last_pos / c + 1;  // chunks holding positions 0..last_pos
  const size_t tile_bytes = (size_t)c * D * sizeof(T);
  if (tid == 0) {
    for (int s = 0; s < kPfStages; ++s) mbar_init(&full_bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int k) {  // thread 0: K and V tile of chunk k into stage k % 2
    const int s = k % kPfStages;
    const int nt = min(c, seq_len - k * c);  // valid tokens of the chunk (partial last chunk)
    const uint32_t bytes = (uint32_t)(nt * D * (int)sizeof(T));
    const size_t off = ((size_t)chunks[chunk_off + k] * h + head) * c * D;
    unsigned char* st = smem_raw + (size_t)s * 2 * tile_bytes;
    mbar_arrive_expect_tx(&full_bar[s], 2 * bytes);
    bulk_g2s(st, kpool + off, bytes, &full_bar[s]);
    bulk_g2s(st + tile_bytes, vpool + off, bytes, &full_bar[s]);
  };
  if (tid == 0) {
    for (int k = 0; k < min(kPfStages, n_chunks); ++k) issue(k);
  }
  // Q fragments of the warp's 16 rows (rows past nq are zero and not written)
  uint32_t qa[WA::KS][4];
  const int rlo = warp * 16 + (lane >> 2), rhi = rlo + 8;
  {
    const T* qlo = rlo < nq ? q + ((size_t)(q_row0 + rlo) * h + head) * D : nullptr;
    const T* qhi = rhi < nq ? q + ((size_t)(q_row0 + rhi) * h + head) * D : nullptr;
    const int cq = (lane & 3) * 2;
#pragma unroll
    for (int ks = 0; ks < WA::KS; ++ks) {
      qa[ks][0] = qlo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16 + cq) : 0u;
      qa[ks][1] = qhi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16 + cq) : 0u;
      qa[ks][2] = qlo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16 + 8 + cq) : 0u;
      qa[ks][3] = qhi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16 + 8 + cq) : 0u;
    }
  }
  WA wa;
  wa.reset();
  const int plo = pos0 + rlo, phi = pos0 + rhi;             // query positions of the lane's rows
  const int wlast = min(pos0 + warp * 16 + 15, last_pos);  // last position of the warp's rows
  for (int k = 0; k < n_chunks; ++k) {
    const int s = k % kPfStages;
    mbar_wait(&full_bar[s], (uint32_t)((k / kPfStages) & 1));
    const int cs = k * c;                     // first position of the chunk
    const int nt = min(c, seq_len - cs);      // valid tokens (the V fragments past them are zeroed)
    if (cs <= wlast && warp * 16 < nq) {      // the chunk holds a position some row of the warp sees
      const uint32_t k_u32 = smem_u32(smem_raw + (size_t)s * 2 * tile_bytes);
      const uint32_t v_u32 = k_u32 + (uint32_t)tile_bytes;
      const int lim_lo = plo - cs + 1, lim_hi = phi - cs + 1;  // row sees tokens < lim of this chunk
      const int nvis = min(nt, wlast - cs + 1);                // tokens any row of the warp sees
      int t0 = 0;
      for (; t0 + 32 <= nvis; t0 += 32)
        wa.template chunk<true, 32, true>(qa, k_u32, v_u32, t0, nvis, scale_log2, lane, lim_lo, lim_hi);
      for (; t0 < nvis; t0 += 16)
        wa.template chunk<true, 16, true>(qa, k_u32, v_u32, t0, nvis, scale_log2, lane, lim_lo, lim_hi);
    }
    __syncthreads();  // every warp is done with stage s
    if (tid == 0 && k + kPfStages < n_chunks) {
      fence_proxy_async();
      issue(k + kPfStages);
    }
  }
  wa.finish();
  const int cq = (lane & 3) * 2;
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    const int r = hf ? rhi : rlo;
    if (r < nq) {
      const float inv = 1.f / (hf ? wa.n_hi : wa.n_lo);
      TO* orow = out + ((size_t)(q_row0 + r) * h + head) * D;
#pragma unroll
      for (int i = 0; i < WA::DT; ++i) {
        Elem<TO>::store1(orow + i * 8 + cq, wa.o[i][2 * hf] * inv);
        Elem<TO>::store1(orow + i * 8 + cq + 1, wa.o[i][2 * hf + 1] * inv);
      }
    }
  }
}

template <typename T, typename TO, int D>
cudaError_t launch_t(const PrefillLaunch& a, cudaStream_t st) {
  auto kern = prefill_kernel<T, TO, D>;
  const size_t smem = (size_t)kPfStages * 2 * a.pool.c * D * sizeof(T);
  cudaError_t e = set_smem_once(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const size_t loff = (size_t)a.layer * a.pool.layer_stride;
  dim3 grid(a.n_tiles, a.pool.h);
  kern<<<grid, kPfWarps * 32, smem, st>>>(static_cast<const T*>(a.pool.k) + loff, static_cast<const T*>(a.pool.v) + loff,
                                         static_cast<const T*>(a.q), static_cast<TO*>(a.out), a.tiles, a.chunks,
                                         a.pool.h, a.pool.c, a.scale_log2);
  return cudaGetLastError();
}

template <typename T, int D>
cudaError_t dispatch_out(const PrefillLaunch& a, cudaStream_t st) {
  switch (a.out_dtype) {
    case DT_F16: return launch_t<T, __half, D>(a, st);
    case DT_BF16: return launch_t<T, __nv_bfloat16, D>(a, st);
    case DT_F32: return launch_t<T, float, D>(a, st);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t dispatch_d(const PrefillLaunch& a, cudaStream_t st) {
  if (a.pool.d == 128) return dispatch_out<T, 128>(a, st);
  if (a.pool.d == 64) return dispatch_out<T, 64>(a, st);
  return cudaErrorInvalidValue;
}

}  // namespace

bool prefill_supported(const PoolGeom& pool) {
  return (pool.dtype == DT_F16 || pool.dtype == DT_BF16) && (pool.d == 64 || pool.d == 128) && pool.c % 16 == 0 &&
         (size_t)kPfStages * 2 * pool.c * pool.d * 2 <= 200 * 1024;
}

cudaError_t launch_prefill(const PrefillLaunch& a, cudaStream_t st) {
  if (a.n_tiles == 0) return cudaSuccess;
  if (a.pool.dtype == DT_F16) return dispatch_d<__half>(a, st);
  if (a.pool.dtype == DT_BF16) return dispatch_d<__nv_bfloat16>(a, st);
  return cudaErrorInvalidValue;
}

}  // namespace pakv
