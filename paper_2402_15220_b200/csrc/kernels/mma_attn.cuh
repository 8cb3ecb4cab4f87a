// Per-warp tensor-core partial attention over one chunk tile (Eqn 1 fused
// with the Eqn 2 rescale) -- shared by the
// chunk-first kernel (16 query rows per warp) and the seq-first kernel (the
// row's query in row 0 of the 16-row MMA tile).
//
// Tile layout in shared memory = pool layout: [c][D] 16-bit, rows of D*2
// bytes, 16-byte chunk index XOR (token % 8) (common.cuh swz_chunk), so
// ldmatrix of 8 consecutive tokens is bank-conflict free.
//
// mma.sync.m16n8k16 (fp32 accumulate):  S = Q K^T over the warp's token slice
// [tok0, tok0 + NTOK), online softmax in log2 units (P rounded to the input
// type, row sum n from the rounded P: reading A11), O = O * corr + P V.
#pragma once

#include "common.cuh"

namespace pakv {
namespace dev {

template <int D>
CA_DEV uint32_t tile_off(int row, int col) {  // byte offset of (token, element) in a [c][D] 16-bit tile
  return (uint32_t)(row * (D * 2) + ((((col >> 3) ^ (row & 7))) << 4) + (col & 7) * 2);
}

template <typename T, int D, int TPW>
struct WarpAttn {
  static constexpr int KS = D / 16;   // k-steps over d
  static constexpr int DT = D / 8;    // n-tiles of O
  float o[DT][4];
  float m_lo, m_hi, n_lo, n_hi;

  CA_DEV void reset() {
#pragma unroll
    for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    m_lo = m_hi = -INFINITY;
    n_lo = n_hi = 0.f;
  }

  // Tokens [tok0, tok0 + NTOK) of the tile; tokens >= nvalid are masked (MASK).
  // NTOK > 16 gives the mma chains NTOK / 8 independent accumulators (the
  // chunk-first phase is latency-bound at 16 tokens per call).
  // CAUSAL (prefill): additionally, row lo / hi (lane >> 2, + 8) sees only
  // tokens < lim_lo / lim_hi of the tile.
  // sp_tok >= 0: that token's K and V rows are not in the tile but at sp_k /
  // sp_v (row-major, unswizzled) -- the decode step's new row, read straight
  // from where it was staged (each lane addresses its own ldmatrix row).
  template <bool MASK, int NTOK = TPW, bool CAUSAL = false>
  CA_DEV void chunk(const uint32_t (&qa)[KS][4], uint32_t k_u32, uint32_t v_u32, int tok0, int nvalid,
                    float scale_log2, int lane, int lim_lo = 0, int lim_hi = 0, int sp_tok = -1,
                    uint32_t sp_k = 0, uint32_t sp_v = 0) {
    constexpr int NT = NTOK / 8;
    const int mi = lane >> 3, r8 = lane & 7;
    float sc[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
    // K fragments of k-step ks + 1 are loaded before the mma of k-step ks
    // (ldmatrix is ordered asm: without the register double buffer every
    // mma would wait out a full ldmatrix latency)
    uint32_t kb[2][NT / 2][4];
    auto load_k = [&](int ks, uint32_t (&dst)[NT / 2][4]) {
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        const int tok = tok0 + np * 16 + (mi >> 1) * 8 + r8;
        const int col = ks * 16 + (mi & 1) * 8;
        const uint32_t a = tok == sp_tok ? sp_k + col * 2 : k_u32 + tile_off<D>(tok, col);
        ldmatrix_x4(a, dst[np][0], dst[np][1], dst[np][2], dst[np][3]);
      }
    };
    load_k(0, kb[0]);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      if (ks + 1 < KS) load_k(ks + 1, kb[(ks + 1) & 1]);
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        Mma<T>::run(sc[2 * np], qa[ks], kb[ks & 1][np][0], kb[ks & 1][np][1]);
        Mma<T>::run(sc[2 * np + 1], qa[ks], kb[ks & 1][np][2], kb[ks & 1][np][3]);
      }
    }
    if (MASK) {
      const int cb = tok0 + (lane & 3) * 2;
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const int t0 = cb + i * 8;
        if (t0 >= nvalid) sc[i][0] = sc[i][2] = -INFINITY;
        if (t0 + 1 >= nvalid) sc[i][1] = sc[i][3] = -INFINITY;
        if (CAUSAL) {
          if (t0 >= lim_lo) sc[i][0] = -INFINITY;
          if (t0 + 1 >= lim_lo) sc[i][1] = -INFINITY;
          if (t0 >= lim_hi) sc[i][2] = -INFINITY;
          if (t0 + 1 >= lim_hi) sc[i][3] = -INFINITY;
        }
      }
    }
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
    const float b_lo = mn_lo == -INFINITY ? 0.f : mn_lo;  // fully masked row: no NaN
    const float b_hi = mn_hi == -INFINITY ? 0.f : mn_hi;
    const float c_lo = fast_exp2(m_lo - b_lo), c_hi = fast_exp2(m_hi - b_hi);
    m_lo = mn_lo;
    m_hi = mn_hi;
    uint32_t pa[NT][2];
    float ps_lo = 0.f, ps_hi = 0.f;
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      pa[i][0] = Mma<T>::pack(fast_exp2(fmaf(sc[i][0], scale_log2, -b_lo)), fast_exp2(fmaf(sc[i][1], scale_log2, -b_lo)));
      pa[i][1] = Mma<T>::pack(fast_exp2(fmaf(sc[i][2], scale_log2, -b_hi)), fast_exp2(fmaf(sc[i][3], scale_log2, -b_hi)));
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
#pragma unroll
    for (int kk = 0; kk < NTOK / 16; ++kk) {
      const uint32_t a[4] = {pa[2 * kk][0], pa[2 * kk][1], pa[2 * kk + 1][0], pa[2 * kk + 1][1]};
      // masked tokens: P = 0 there, and their V rows (stale shared memory, maybe
      // not finite) are zeroed in the B fragments so 0 * V cannot produce NaN.
      // b0/b2 hold tokens tb, tb + 1 (low, high half); b1/b3 tokens tb + 8, tb + 9.
      uint32_t vm0 = 0xffffffffu, vm1 = 0xffffffffu;
      if (MASK) {
        const int tb = tok0 + kk * 16 + (lane & 3) * 2;
        vm0 = (tb < nvalid ? 0x0000ffffu : 0u) | (tb + 1 < nvalid ? 0xffff0000u : 0u);
        vm1 = (tb + 8 < nvalid ? 0x0000ffffu : 0u) | (tb + 9 < nvalid ? 0xffff0000u : 0u);
      }
      // V fragments one d-pair ahead of the mma (see load_k)
      const int vtok = tok0 + kk * 16 + (mi & 1) * 8 + r8;
      const bool vsp = vtok == sp_tok;
      auto vaddr = [&](int col) { return vsp ? sp_v + col * 2 : v_u32 + tile_off<D>(vtok, col); };
      uint32_t vb[2][4];
      ldmatrix_x4_trans(vaddr((mi >> 1) * 8), vb[0][0], vb[0][1], vb[0][2], vb[0][3]);
#pragma unroll
      for (int dp = 0; dp < DT / 2; ++dp) {
        if (dp + 1 < DT / 2) {
          uint32_t(&nx)[4] = vb[(dp + 1) & 1];
          ldmatrix_x4_trans(vaddr((dp + 1) * 16 + (mi >> 1) * 8), nx[0], nx[1], nx[2], nx[3]);
        }
        uint32_t b0 = vb[dp & 1][0], b1 = vb[dp & 1][1], b2 = vb[dp & 1][2], b3 = vb[dp & 1][3];
        if (MASK) {
          b0 &= vm0;
          b2 &= vm0;
          b1 &= vm1;
          b3 &= vm1;
        }
        Mma<T>::run(o[2 * dp], a, b0, b1);
        Mma<T>::run(o[2 * dp + 1], a, b2, b3);
      }
    }
  }

  // Row sums over the quad (the 4 lanes holding one row).
  CA_DEV void finish() {
    n_lo += __shfl_xor_sync(0xffffffffu, n_lo, 1);
    n_lo += __shfl_xor_sync(0xffffffffu, n_lo, 2);
    n_hi += __shfl_xor_sync(0xffffffffu, n_hi, 1);
    n_hi += __shfl_xor_sync(0xffffffffu, n_hi, 2);
  }
};

}  // namespace dev
}  // namespace pakv
