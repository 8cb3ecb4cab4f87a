// K4 seq-first phase (Alg 2) and the SIMT chunk-first
// fallback (Alg 1 for fp32 / shapes the tensor-core kernel does not take).
//
// One CTA per (row, head) [seq-first] or (tile row, head) [chunk-first SIMT].
// The row's chunks are streamed (K and V tile of one (chunk, head): c x d,
// contiguous in the pool) with 1-D bulk async copies into an NST-stage shared
// memory ring; only the valid tokens of the last, partial chunk are copied and
// the rest are masked by select (stale slots never enter the arithmetic).
// 128 threads = G groups of d/VEC threads; a group owns every G-th token of a
// chunk, computes its logits with 16-byte shared loads + FMA + shfl_xor
// reduction and keeps its own online-softmax state (o, m, n) in registers
// (Eqn 1 partial_attn fused with Eqn 2 attn_reduce, PAPER.md:95-108, 145-158;
// m in log2 units, exp2 with log2(e) folded into the scale).  At the end the
// groups merge in a fixed order through shared memory; the seq-first CTA then
// merges the chunk-first partials listed for its row (fixed order, reading A12)
// and writes O / n in the output dtype.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace pakv {

using namespace dev;

namespace {

constexpr int kThreads = 128;
constexpr int kMaxStages = 4;

CA_DEV void merge_state(float& o, float& m, float& n, float oc, float mc, float nc) {
  // Eqn 2 in log2 units; empty partials (m = -inf) skipped (reading A2).
  const float mx = fmaxf(m, mc);
  if (mx == -INFINITY) return;
  const float x = fast_exp2(mc - mx);
  const float y = fast_exp2(m - mx);
  o = x * oc + y * o;
  n = x * nc + y * n;
  m = mx;
}

template <typename T, int D>
struct Geo {
  static constexpr int kVec = Elem<T>::kVec;
  static constexpr int kTpt = D / kVec;            // threads per token row
  static constexpr int kGroups = kThreads / kTpt;  // token groups per CTA
  static_assert(kTpt <= 32 && (32 % kTpt) == 0, "group must sit inside a warp");
};

// One chunk tile in shared memory: nt valid tokens.
template <typename T, int D>
CA_DEV void consume_chunk(const T* __restrict__ Ks, const T* __restrict__ Vs, int nt, const float* qf, float& m,
                          float& n, float* o, int g, int j) {
  using G = Geo<T, D>;
  constexpr int U = 4;  // tokens per group per batch
  const int iters = (nt + G::kGroups * U - 1) / (G::kGroups * U);
  for (int it = 0; it < iters; ++it) {
    float l[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = (it * U + u) * G::kGroups + g;
      float acc = 0.f;
      if (t < nt) {
        const uint4 raw = *reinterpret_cast<const uint4*>(Ks + (size_t)t * D + j * G::kVec);
        float kf[G::kVec];
        Elem<T>::to_float(raw, kf);
#pragma unroll
        for (int v = 0; v < G::kVec; ++v) acc = fmaf(qf[v], kf[v], acc);
      }
#pragma unroll
      for (int off = G::kTpt / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      l[u] = t < nt ? acc : -INFINITY;
    }
    float mx = l[0];
#pragma unroll
    for (int u = 1; u < U; ++u) mx = fmaxf(mx, l[u]);
    const float m_new = fmaxf(m, mx);
    if (m_new == -INFINITY) continue;  // whole batch masked and nothing seen yet
    const float corr = fast_exp2(m - m_new);
    float p[U];
    float psum = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      p[u] = fast_exp2(l[u] - m_new);
      psum += p[u];
    }
    n = n * corr + psum;
#pragma unroll
    for (int v = 0; v < G::kVec; ++v) o[v] *= corr;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = (it * U + u) * G::kGroups + g;
      if (t < nt) {  // select, not multiply: stale slots never enter the sum
        const uint4 raw = *reinterpret_cast<const uint4*>(Vs + (size_t)t * D + j * G::kVec);
        float vf[G::kVec];
        Elem<T>::to_float(raw, vf);
#pragma unroll
        for (int v = 0; v < G::kVec; ++v) o[v] = fmaf(p[u], vf[v], o[v]);
      }
    }
    m = m_new;
  }
}

// MODE 0: seq-first (grid b x h).  MODE 1: chunk-first SIMT (grid tiles x h x rows).
template <typename T, typename TO, int D, int MODE>
__global__ void __launch_bounds__(kThreads) attend_simt_kernel(const T* __restrict__ kpool,
                                                               const T* __restrict__ vpool,
                                                               const T* __restrict__ q, TO* __restrict__ out,
                                                               float* __restrict__ pO, float2* __restrict__ pMN,
                                                               DevTables t, int32_t h, int32_t c, float scale_log2,
                                                               int32_t nst) {
  using G = Geo<T, D>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bars[kMaxStages];
  __shared__ float sm_m[G::kGroups], sm_n[G::kGroups];
  __shared__ float sm_o[G::kGroups][D];

  const int head = blockIdx.y;
  int row, n_chunks, first_pos, len, slot = -1;
  const int32_t* chunks;
  if (MODE == 0) {
    row = blockIdx.x;
    chunks = t.sf_chunk + t.sf_ptr[row];
    n_chunks = t.sf_ptr[row + 1] - t.sf_ptr[row];
    first_pos = t.sf_first[row];
    len = t.seq_len[row];
  } else {
    const int32_t* tile = t.cf_tile + blockIdx.x * 8;
    row = tile[2] + blockIdx.z;
    if (row >= tile[3]) return;
    chunks = t.cf_chunk + tile[0];
    n_chunks = tile[1];
    first_pos = 0;
    len = 0x7fffffff;  // shared chunks are always full (reading T1)
    slot = tile[4] + (int)blockIdx.z;
  }
  const int caller = t.row_caller[row];
  const int tid = threadIdx.x;
  const int g = tid / G::kTpt, j = tid % G::kTpt;

  const size_t tile_elems = (size_t)c * D;
  T* Ks = reinterpret_cast<T*>(smem_raw);
  T* Vs = Ks + (size_t)nst * tile_elems;

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  auto issue = [&](int k) {
    const int s = k % nst;
    const int cid = chunks[k];
    const int nt = min(c, len - (first_pos + k * c));
    const uint32_t bytes = (uint32_t)(nt * D * (int)sizeof(T));
    const size_t off = ((size_t)cid * h + head) * tile_elems;
    mbar_arrive_expect_tx(&bars[s], 2 * bytes);
    bulk_g2s(Ks + s * tile_elems, kpool + off, bytes, &bars[s]);
    bulk_g2s(Vs + s * tile_elems, vpool + off, bytes, &bars[s]);
  };
  if (tid == 0)
    for (int k = 0; k < min(nst, n_chunks); ++k) issue(k);

  float qf[G::kVec];
  {
    const uint4 raw = *reinterpret_cast<const uint4*>(q + ((size_t)caller * h + head) * D + j * G::kVec);
    Elem<T>::to_float(raw, qf);
#pragma unroll
    for (int v = 0; v < G::kVec; ++v) qf[v] *= scale_log2;
  }
  float m = -INFINITY, n = 0.f, o[G::kVec];
#pragma unroll
  for (int v = 0; v < G::kVec; ++v) o[v] = 0.f;

  for (int k = 0; k < n_chunks; ++k) {
    const int s = k % nst;
    mbar_wait(&bars[s], (uint32_t)((k / nst) & 1));
    const int nt = min(c, len - (first_pos + k * c));
    consume_chunk<T, D>(Ks + s * tile_elems, Vs + s * tile_elems, nt, qf, m, n, o, g, j);
    __syncthreads();  // every group is done with stage s
    if (tid == 0 && k + nst < n_chunks) issue(k + nst);
  }

  if (j == 0) {
    sm_m[g] = m;
    sm_n[g] = n;
  }
#pragma unroll
  for (int v = 0; v < G::kVec; ++v) sm_o[g][j * G::kVec + v] = o[v];
  __syncthreads();

  for (int x = tid; x < D; x += kThreads) {
    float ao = 0.f, am = -INFINITY, an = 0.f;
    if (MODE == 0) {
      pdl_wait();  // chunk-first partials are complete (no-op without PDL)
      for (int e = t.mg_ptr[row]; e < t.mg_ptr[row + 1]; ++e) {
        const int sl = t.mg_slot[e];
        const float2 mn = pMN[(size_t)sl * h + head];
        merge_state(ao, am, an, pO[((size_t)sl * h + head) * D + x], mn.x, mn.y);
      }
    }
    for (int gg = 0; gg < G::kGroups; ++gg) merge_state(ao, am, an, sm_o[gg][x], sm_m[gg], sm_n[gg]);
    if (MODE == 0) {
      Elem<TO>::store1(out + ((size_t)caller * h + head) * D + x, ao / an);
    } else {
      pO[((size_t)slot * h + head) * D + x] = ao;
      if (x == 0) pMN[(size_t)slot * h + head] = make_float2(am, an);
    }
  }
}

template <typename T, typename TO, int D, int MODE>
cudaError_t launch_simt(const AttnLaunch& a, const DevTables& t, dim3 grid, cudaStream_t st, bool pdl) {
  const PoolGeom& p = a.pool;
  const size_t stage = (size_t)2 * p.c * D * sizeof(T);
  int nst = (int)std::min<size_t>(3, (size_t)(160 * 1024) / stage);
  nst = std::max(1, nst);
  const size_t smem = nst * stage;
  auto kern = attend_simt_kernel<T, TO, D, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const T* kp = (const T*)p.k + (size_t)a.layer * p.layer_stride;
  const T* vp = (const T*)p.v + (size_t)a.layer * p.layer_stride;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, kp, vp, (const T*)a.q, (TO*)a.out, a.pO, a.pMN, t, p.h, p.c, a.scale_log2,
                            nst);
}

template <typename T, int MODE>
cudaError_t dispatch_d_out(const AttnLaunch& a, const DevTables& t, dim3 grid, cudaStream_t st, bool pdl) {
  const int d = a.pool.d;
  const int od = MODE == 1 ? DT_F32 : a.out_dtype;
#define CA_CASE(DD, TO)                                                           \
  if (d == DD) return launch_simt<T, TO, DD, MODE>(a, t, grid, st, pdl);
  if (od == DT_F32) {
    CA_CASE(64, float) CA_CASE(128, float)
  } else if (od == DT_F16) {
    CA_CASE(64, __half) CA_CASE(128, __half)
  } else {
    CA_CASE(64, __nv_bfloat16) CA_CASE(128, __nv_bfloat16)
  }
#undef CA_CASE
  return cudaErrorInvalidValue;
}

template <int MODE>
cudaError_t dispatch(const AttnLaunch& a, const DevTables& t, dim3 grid, cudaStream_t st, bool pdl) {
  switch (a.pool.dtype) {
    case DT_F32: return dispatch_d_out<float, MODE>(a, t, grid, st, pdl);
    case DT_F16: return dispatch_d_out<__half, MODE>(a, t, grid, st, pdl);
    default: return dispatch_d_out<__nv_bfloat16, MODE>(a, t, grid, st, pdl);
  }
}

}  // namespace

cudaError_t launch_seq_first(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (t.b == 0) return cudaSuccess;
  return dispatch<0>(a, t, dim3(t.b, a.pool.h), st, a.use_pdl && t.n_cf_tiles > 0);
}

cudaError_t launch_chunk_first_simt(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (t.n_cf_tiles == 0) return cudaSuccess;
  return dispatch<1>(a, t, dim3(t.n_cf_tiles, a.pool.h, t.max_tile_rows), st, false);
}

}  // namespace pakv
