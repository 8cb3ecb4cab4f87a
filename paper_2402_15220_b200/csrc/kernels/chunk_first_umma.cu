// K3 chunk-first phase on the 5th-generation tensor cores (tcgen05 / UMMA;
// SURVEY §8 row f3).  Same job and output contract as cf_mma_kernel (Alg 1,
// PAPER.md:72-91; Eqn 1): one CTA = (head, rows [r0, r1) <=
// 128 of a shared run, chunks [k0, k1) of that run) -> one fp32 partial row
// (o | m n, m in log2 units) per (row, head).
//
//   S_k = Q . K_k^T   M = 128 rows, N = c tokens, K = d   (A = Q, B = K: K-major)
//   O  += P_k . V_k   M = 128 rows, N = d, K = c tokens   (A = P: K-major, B = V: MN-major)
// issued by one thread (warp 5), S double-buffered and O in TMEM; the online
// softmax (Eqn 1 + Eqn 2 rescale) runs on 4 warps, thread = row = TMEM lane,
// concurrently with the next chunk's S.  O is rescaled lazily (only when a
// row's max grows by more than 2^8: P <= 256 is exact enough in 16 bits and
// the final O / n does not depend on the reference max).  K / V tiles arrive
// by 2-D TMA (one box per 64-element d-half: the pool rows are already XOR
// pre-swizzled within each 128-byte half, so the boxes land as canonical
// SWIZZLE_128B atoms -- tools/umma_probe.cu validates both operand layouts).
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "../host/schedule.h"
#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace pakv {

using namespace dev;

namespace {

constexpr int kUmRows = 128;   // UMMA M
constexpr int kUmStages = 3;   // K/V ring depth
constexpr int kUmThreads = 224;  // warps 0-3 softmax/epilogue, 4 TMA producer, 5 S issuer, 6 P V issuer
constexpr float kRescaleLog2 = 8.f;  // lazy O rescale threshold (P <= 2^8)


// 32 consecutive fp32 TMEM columns x inv -> 32 output elements, 16-byte stores
template <typename TO>
CA_DEV void store_row32(TO* dst, const uint32_t (&u)[32], float inv) {
  if constexpr (std::is_same<TO, float>::value) {
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4*>(dst + i) = make_float4(__uint_as_float(u[i]) * inv, __uint_as_float(u[i + 1]) * inv,
                                                        __uint_as_float(u[i + 2]) * inv, __uint_as_float(u[i + 3]) * inv);
  } else {
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w[e] = Mma<TO>::pack(__uint_as_float(u[i + 2 * e]) * inv, __uint_as_float(u[i + 2 * e + 1]) * inv);
      *reinterpret_cast<uint4*>(dst + i) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}


// PREFILL (row f1 on tcgen05): CTA = (<= 128 NG consecutive query positions
// of one sequence, head); causal mask per row, stale K/V rows past the
// sequence end masked (K) and zeroed in shared memory before PV (V), output
// O / n in TO (no partials).  NG = 2 softmax groups (two 128-row query tiles
// of the same head) share every K/V stage and ping-pong on the tensor core.
template <typename T, typename TO, int D, int C, bool PREFILL, int NG>
__global__ void __launch_bounds__(NG * 128 + 96, 1)
    cf_umma_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                   const T* __restrict__ q, float* __restrict__ pO, DevTables t, int32_t h, int64_t layer_rows,
                   float scale_log2, TO* __restrict__ out, const int32_t* __restrict__ pf_tiles,
                   const int32_t* __restrict__ pf_chunks) {
  constexpr int NST = NG == 1 ? kUmStages : 2;   // K/V ring depth (shared-memory budget)
  constexpr int HALVES = D / 64;            // 128-byte d-halves of a token row
  constexpr int PATOMS = C / 64;            // 128-byte token atoms of a P row
  constexpr uint32_t kQBytes = HALVES * kUmRows * 128;
  constexpr uint32_t kTileBytes = HALVES * C * 128;  // one K (or V) tile image
  constexpr uint32_t kStageBytes = 2 * kTileBytes;
  constexpr uint32_t kPBytes = PATOMS * kUmRows * 128;
  constexpr uint32_t kGroupCols = 2 * C + D;        // S double buffer + O per group
  constexpr uint32_t kTmemCols = NG * kGroupCols <= 256 ? 256 : 512;
  static_assert(NG * kGroupCols <= 512, "TMEM columns");
  constexpr int PR = D + 4;
  constexpr int kProducer = 4 * NG, kIssuer = 4 * NG + 1, kPvIssuer = 4 * NG + 2;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = sm;                       // [NG][kQBytes]
  unsigned char* sKV = sQ + NG * kQBytes;       // [NST][kStageBytes]
  unsigned char* sP = sKV + NST * kStageBytes;  // [NG][2][kPBytes]
  __shared__ uint64_t kv_full[NST], kv_empty[NST];
  __shared__ uint64_t s_full[NG][2], s_free[NG][2], p_full[NG][2], pv_done[NG][2], q_full[NG];
  __shared__ uint64_t o_ready;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int head = blockIdx.y;
  int chunk_off, n_chunks, row0, rows, slot0 = 0, pos0 = 0, seq_len = 0;
  const int32_t* chunk_list;
  if (PREFILL) {  // {chunk list offset, first query row, queries, first position, sequence length}
    const int32_t* pt = pf_tiles + (size_t)blockIdx.x * kPfTileInts;
    chunk_off = pt[0];
    row0 = pt[1];
    rows = pt[2];
    pos0 = pt[3];
    seq_len = pt[4];
    n_chunks = (pos0 + rows - 1) / C + 1;
    chunk_list = pf_chunks;
  } else {
    const int32_t* tile = t.cf_tile + blockIdx.x * kCfTileInts;
    chunk_off = tile[CF_CHUNK_OFF];
    n_chunks = tile[CF_NCHUNK];
    row0 = tile[CF_ROW0];
    rows = tile[CF_ROW1] - row0;
    slot0 = tile[CF_SLOT];
    chunk_list = t.cf_chunk;
  }
  pdl_launch_dependents();

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int g = 0; g < NG; ++g) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&s_full[g][b], 1);
        mbar_init(&s_free[g][b], 4);
        mbar_init(&p_full[g][b], 4);
        mbar_init(&pv_done[g][b], 1);
      }
      mbar_init(&q_full[g], 4);
    }
    mbar_init(&o_ready, 1);
    fence_barrier_init();
  }
  if (warp == kIssuer) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == kProducer) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      for (int k = 0; k < n_chunks; ++k) {
        const int s = k % NST;
        if (k >= NST) mbar_wait(&kv_empty[s], (uint32_t)(((k / NST) - 1) & 1));
        mbar_arrive_expect_tx(&kv_full[s], kStageBytes);
        const int y = (int)(layer_rows + ((int64_t)chunk_list[chunk_off + k] * h + head) * C);
        unsigned char* st = sKV + s * kStageBytes;
#pragma unroll
        for (int hf = 0; hf < HALVES; ++hf) {
          tma_load_2d(st + hf * C * 128, &tmap_k, hf * 64, y, &kv_full[s]);
          tma_load_2d(st + kTileBytes + hf * C * 128, &tmap_v, hf * 64, y, &kv_full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == kIssuer) {
    // ---------------------------------------------------------- S issuer
    // S_{g,k} = Q_g K_k^T into S buffer k & 1; P V runs on its own issuer
    // (warp kPvIssuer), so S of the next chunk never waits behind it
    if (lane == 0) {
      constexpr uint32_t idS = umma_idesc<T>(C, false);
      const uint32_t qa = smem_u32(sQ), kva = smem_u32(sKV);
      for (int g = 0; g < NG; ++g) mbar_wait(&q_full[g], 0);
      tc_fence_after();
      for (int k = 0; k < n_chunks; ++k) {
        const int s = k % NST, b = k & 1;
        mbar_wait(&kv_full[s], (uint32_t)((k / NST) & 1));
        const uint32_t ka = kva + s * kStageBytes;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          if (k >= 2) mbar_wait(&s_free[g][b], (uint32_t)(((k >> 1) - 1) & 1));
          tc_fence_after();
          const uint32_t qg = qa + g * kQBytes, tS = tmem + g * kGroupCols + b * C;
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {  // S_{g,k} = Q_g K_k^T over d
            const uint32_t o = (ks % 4) * 32;
            umma_f16(tS, umma_sdesc(qg + (ks / 4) * kUmRows * 128 + o, 16, 1024),
                     umma_sdesc(ka + (ks / 4) * C * 128 + o, 16, 1024), idS, ks > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[g][b]);
        }
      }
    }
    __syncwarp();
  } else if (warp == kPvIssuer) {
    // -------------------------------------------------------- P V issuer
    // O_g += P_{g,k} V_k once the softmax has published P_{g,k}; the stage
    // is released after the last group's P V
    if (lane == 0) {
      constexpr uint32_t idO = umma_idesc<T>(D, true);
      const uint32_t kva = smem_u32(sKV), pa = smem_u32(sP);
      for (int k = 0; k < n_chunks; ++k) {
        const int s = k % NST, b = k & 1;
        mbar_wait(&kv_full[s], (uint32_t)((k / NST) & 1));  // V of the stage (the S issuer saw it first)
        const uint32_t va = kva + s * kStageBytes + kTileBytes;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          mbar_wait(&p_full[g][b], (uint32_t)((k >> 1) & 1));
          tc_fence_after();
          const uint32_t pb = pa + (g * 2 + b) * kPBytes, tO = tmem + g * kGroupCols + 2 * C;
#pragma unroll
          for (int ks = 0; ks < C / 16; ++ks)
            umma_f16(tO, umma_sdesc(pb + (ks / 4) * kUmRows * 128 + (ks % 4) * 32, 16, 1024),
                     umma_sdesc(va + ks * 16 * 128, C * 128, 1024), idO, (k > 0 || ks > 0) ? 1u : 0u);
          umma_commit(&pv_done[g][b]);
        }
        umma_commit(&kv_empty[s]);
      }
      umma_commit(&o_ready);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------- softmax / epilogue
    const int g = warp >> 2;            // query group
    const int r = tid & 127;            // row of the group = TMEM lane
    const int grow0 = g * kUmRows;      // first row of the group in the tile
    const int grows = min(kUmRows, rows - grow0);  // valid rows of the group (may be <= 0)
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS0 = tmem + g * kGroupCols, tO = tS0 + 2 * C;
    unsigned char* sQg = sQ + g * kQBytes;
    {  // Q image (SWIZZLE_128B, d-halves), rows past the tile zero
      const T* qrow = r >= grows ? nullptr
                      : PREFILL ? q + ((size_t)(row0 + grow0 + r) * h + head) * D
                                : q + ((size_t)t.row_caller[row0 + grow0 + r] * h + head) * D;
#pragma unroll
      for (int gg = 0; gg < D / 8; ++gg) {
        const uint4 v = qrow ? *reinterpret_cast<const uint4*>(qrow + gg * 8) : make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(sQg + (gg / 8) * kUmRows * 128 + sw128(r, gg % 8)) = v;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&q_full[g]);
    }
    float m_ref = -INFINITY, n = 0.f;
    for (int k = 0; k < n_chunks; ++k) {
      const int b = k & 1;
      mbar_wait(&s_full[g][b], (uint32_t)((k >> 1) & 1));
      tc_fence_after();
      float sv[C];
      {  // all column blocks in flight, one wait
        uint32_t u[C / 32][32];
#pragma unroll
        for (int cb = 0; cb < C / 32; ++cb) tmem_ld32(tS0 + b * C + lane_base + cb * 32, u[cb]);
        tmem_wait_ld();
#pragma unroll
        for (int cb = 0; cb < C / 32; ++cb)
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[cb * 32 + i] = __uint_as_float(u[cb][i]);  // raw logits; scale folded below
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&s_free[g][b]);
      if (PREFILL) {
        // causal: row r (position pos0 + grow0 + r) sees positions <= its own,
        // and nothing past the sequence end (stale pool rows)
        const int nt = seq_len - k * C;
        const int lim = min(pos0 + grow0 + r - k * C, nt - 1);  // last visible token of this chunk
        if (lim < C - 1) {  // only the chunks on the diagonal / at the end are masked
#pragma unroll
          for (int i = 0; i < C; ++i)
            if (i > lim) sv[i] = -INFINITY;
        }
        // zero the stale V rows of the stage before any P . V reads them: group
        // 0's P_k is published after this, and the issuer issues group 0's P.V
        // of chunk k before any other group's
        if (nt < C && g == 0) {
          unsigned char* vt = sKV + (k % NST) * kStageBytes + kTileBytes;
          for (int i = r; i < (C - max(nt, 0)) * HALVES * 8; i += 128) {
            const int row = max(nt, 0) + i / (HALVES * 8), hf = (i / 8) % HALVES, j = i % 8;
            *reinterpret_cast<uint4*>(vt + hf * C * 128 + sw128(row, j)) = make_uint4(0u, 0u, 0u, 0u);
          }
        }
      }
      float mx8[8];  // 8 independent max chains (a 64-deep chain is latency-bound)
#pragma unroll
      for (int e = 0; e < 8; ++e) mx8[e] = sv[e];
#pragma unroll
      for (int i = 8; i < C; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], sv[i]);
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])), fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      mx *= scale_log2;  // scale > 0: the max commutes with it
      // lazy rescale: a new reference max only when this row's max grew by more than 2^8
      const bool need = mx > m_ref + kRescaleLog2;
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? mx : m_ref;
        const float f = (need && m_ref != -INFINITY) ? fast_exp2(m_ref - m_new) : 1.f;
        if (k > 0) {  // O holds chunks 0..k-1: wait for PV_{k-1}, scale it in TMEM
          mbar_wait(&pv_done[g][(k - 1) & 1], (uint32_t)(((k - 1) >> 1) & 1));
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t u[32];
            tmem_ld32(tO + lane_base + c0, u);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * f);
            tmem_st32(tO + lane_base + c0, u);
          }
          tmem_wait_st();
          tc_fence_before();
        }
        n *= f;
        m_ref = m_new;
      }
      // P_k = exp2(s - m_ref) rounded to T (n from the rounded P, reading A11)
      if (k >= 2) mbar_wait(&pv_done[g][b], (uint32_t)(((k >> 1) - 1) & 1));  // PV_{k-2} read this buffer
      unsigned char* pb = sP + (g * 2 + b) * kPBytes;
      float ns[4] = {0.f, 0.f, 0.f, 0.f};  // independent partial sums of the rounded P
#pragma unroll
      for (int gg = 0; gg < C / 8; ++gg) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          w[e] = Mma<T>::pack(fast_exp2(fmaf(sv[gg * 8 + 2 * e], scale_log2, -m_ref)),
                              fast_exp2(fmaf(sv[gg * 8 + 2 * e + 1], scale_log2, -m_ref)));
          const float2 f2 = Mma<T>::unpack(w[e]);
          ns[e] += f2.x + f2.y;
        }
        *reinterpret_cast<uint4*>(pb + (gg / 8) * kUmRows * 128 + sw128(r, gg % 8)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      n += (ns[0] + ns[1]) + (ns[2] + ns[3]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&p_full[g][b]);
    }
    // epilogue
    mbar_wait(&o_ready, 0);
    tc_fence_after();
    if (PREFILL) {  // O / n straight to the output row
      TO* orow = r < grows ? out + ((size_t)(row0 + grow0 + r) * h + head) * D : nullptr;
      const float inv = 1.f / n;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t u[32];
        tmem_ld32(tO + lane_base + c0, u);
        tmem_wait_ld();
        if (orow) store_row32<TO>(orow + c0, u, inv);
      }
    } else {  // O (unnormalised), m (log2 units), n -> the row's partial
      float* prow = r < grows ? pO + ((size_t)(slot0 + grow0 + r) * h + head) * PR : nullptr;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t u[32];
        tmem_ld32(tO + lane_base + c0, u);
        tmem_wait_ld();
        if (prow) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(prow + c0 + i) = make_float4(__uint_as_float(u[i]), __uint_as_float(u[i + 1]),
                                                                   __uint_as_float(u[i + 2]), __uint_as_float(u[i + 3]));
        }
      }
      if (prow) *reinterpret_cast<float2*>(prow + D) = make_float2(m_ref, n);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kIssuer) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  pdl_wait();  // PDL chain append -> chunk-first -> seq-first (see cf_mma_kernel)
}

// 2-D views of the pools for TMA: [layers * chunks * h * c rows][d] 16-bit,
// boxes of 64 elements x c rows (one 128-byte d-half of a (chunk, head) tile)
struct MapKey {
  const void* base;
  int64_t rows;
  int32_t d, c;
  bool operator<(const MapKey& o) const {
    return std::tie(base, rows, d, c) < std::tie(o.base, o.rows, o.d, o.c);
  }
};

bool encode_map(const void* base, int64_t rows, int d, int c, CUtensorMap* out) {
  static std::mutex mu;
  static std::map<MapKey, CUtensorMap> cache;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  std::lock_guard<std::mutex> lk(mu);
  const MapKey key{base, rows, d, c};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  if (!encode) {
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)c};
  const cuuint32_t estr[2] = {1, 1};
  if (encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache[key] = m;
  *out = m;
  return true;
}

template <int D, int C, int NG>
constexpr size_t um_smem() {
  return 1024 + (size_t)NG * (D / 64) * kUmRows * 128 + (size_t)(NG == 1 ? kUmStages : 2) * 2 * (D / 64) * C * 128 +
         (size_t)NG * 2 * (C / 64) * kUmRows * 128;
}
// prefill: 128-query tiles per CTA.  Two groups per CTA sharing the K/V stages
// (NG = 2, 2-deep ring) measured slower (0.78 vs 0.52 ms on bench_prefill's
// lookup case: the issuer runs the groups in lock step and half-empty tiles
// still pay both groups), so one group it is.
constexpr int kPfGroups = 1;

}  // namespace

bool pool_maps(const PoolGeom& p, int D, int C, CUtensorMap* mk, CUtensorMap* mv) {
  const int64_t rows = (int64_t)p.num_layers * p.max_chunks * p.h * p.c;
  return encode_map(p.k, rows, D, C, mk) && encode_map(p.v, rows, D, C, mv);
}

namespace {
// 3-D view of a d = 128 pool: {64 elements, rows (stride d * 2 bytes), 2
// d-halves (stride 128 bytes)}; a box {64, c, 2} lands as [half][row][128 B]
// -- both SWIZZLE_128B images of a (chunk, head) tile in ONE TMA op
bool encode_map3(const void* base, int64_t rows, int c, CUtensorMap* out) {
  static std::mutex mu;
  static std::map<MapKey, CUtensorMap> cache;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  std::lock_guard<std::mutex> lk(mu);
  const MapKey key{base, rows, 128, c};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  if (!encode) {
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CUtensorMap m;
  const cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
  const cuuint64_t strides[2] = {256, 128};
  const cuuint32_t box[3] = {64, (cuuint32_t)c, 2};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache[key] = m;
  *out = m;
  return true;
}
}  // namespace

bool pool_maps3(const PoolGeom& p, int C, CUtensorMap* mk, CUtensorMap* mv) {
  if (p.d != 128) return false;
  const int64_t rows = (int64_t)p.num_layers * p.max_chunks * p.h * p.c;
  return encode_map3(p.k, rows, C, mk) && encode_map3(p.v, rows, C, mv);
}

namespace {

template <typename T, int D, int C>
cudaError_t launch_t(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  const PoolGeom& p = a.pool;
  CUtensorMap mk, mv;
  if (!pool_maps(p, D, C, &mk, &mv)) return cudaErrorNotSupported;
  auto kern = cf_umma_kernel<T, T, D, C, false, 1>;
  cudaError_t e = set_smem_once((const void*)kern, um_smem<D, C, 1>());
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3(t.n_cf_tiles, p.h), dim3(kUmThreads), um_smem<D, C, 1>(), st, a.use_pdl, mk, mv,
                   (const T*)a.q, a.pO, t, (int32_t)p.h, (int64_t)a.layer * p.max_chunks * p.h * p.c, a.scale_log2,
                   (T*)nullptr, (const int32_t*)nullptr, (const int32_t*)nullptr);
}

template <typename T>
cudaError_t dispatch(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (a.pool.d == 128 && a.pool.c == 64) return launch_t<T, 128, 64>(a, t, st);
  if (a.pool.d == 64 && a.pool.c == 64) return launch_t<T, 64, 64>(a, t, st);
  return cudaErrorInvalidValue;
}

template <typename T, typename TO, int D, int C>
cudaError_t launch_pf(const PrefillLaunch& a, cudaStream_t st) {
  const PoolGeom& p = a.pool;
  CUtensorMap mk, mv;
  if (!pool_maps(p, D, C, &mk, &mv)) return cudaErrorNotSupported;
  auto kern = cf_umma_kernel<T, TO, D, C, true, kPfGroups>;
  cudaError_t e = set_smem_once((const void*)kern, um_smem<D, C, kPfGroups>());
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3(a.n_tiles, p.h), dim3(kPfGroups * 128 + 96), um_smem<D, C, kPfGroups>(), st, false, mk,
                   mv, (const T*)a.q,
                   (float*)nullptr, DevTables{}, (int32_t)p.h, (int64_t)a.layer * p.max_chunks * p.h * p.c,
                   a.scale_log2, (TO*)a.out, a.tiles, a.chunks);
}

template <typename T, int D>
cudaError_t dispatch_pf_out(const PrefillLaunch& a, cudaStream_t st) {
  switch (a.out_dtype) {
    case DT_F16: return launch_pf<T, __half, D, 64>(a, st);
    case DT_BF16: return launch_pf<T, __nv_bfloat16, D, 64>(a, st);
    case DT_F32: return launch_pf<T, float, D, 64>(a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool cf_umma_supported(const PoolGeom& p, int max_tile_rows) {
  // c = 128 would need 2 x 32 KB P buffers and 64 KB stages: over the shared-memory budget
  return (p.dtype == DT_F16 || p.dtype == DT_BF16) && (p.d == 64 || p.d == 128) && p.c == 64 &&
         max_tile_rows <= kUmRows;
}

bool prefill_umma_supported(const PoolGeom& p) { return cf_umma_supported(p, kUmRows); }

cudaError_t launch_prefill_umma(const PrefillLaunch& a, cudaStream_t st) {
  if (a.n_tiles == 0) return cudaSuccess;
  if (a.pool.dtype == DT_F16)
    return a.pool.d == 128 ? dispatch_pf_out<__half, 128>(a, st) : dispatch_pf_out<__half, 64>(a, st);
  return a.pool.d == 128 ? dispatch_pf_out<__nv_bfloat16, 128>(a, st) : dispatch_pf_out<__nv_bfloat16, 64>(a, st);
}

cudaError_t launch_chunk_first_umma(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (t.n_cf_tiles == 0) return cudaSuccess;
  if (a.pool.dtype == DT_F16) return dispatch<__half>(a, t, st);
  return dispatch<__nv_bfloat16>(a, t, st);
}

}  // namespace pakv
