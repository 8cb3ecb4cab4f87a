// K4 seq-first phase (Alg 2) as a persistent, warp-
// specialised kernel, and the SIMT chunk-first fallback (Alg 1) for fp32 and
// shapes the tensor-core kernel does not take.
//
// Seq-first work = items (row, head); an item's units are its private chunks
// (max(1, n) units so rows without private chunks still merge their partials).
// The host cuts the flattened unit list into one balanced contiguous range per
// CTA (2 per SM).  Warp 0 is the producer: it reads the unit descriptors 32 at
// a time (one lane each), and for every unit waits for a free stage of an
// NST-deep shared-memory ring, publishes the unit's metadata in the stage and
// issues 1-D bulk async copies (cp.async.bulk -> UBLKCP) of the K and V tile
// of that (chunk, head) -- only the valid tokens of a partial last chunk --
// plus the query row at a segment start and the chunk-first partial rows of
// the item at its end, all completing on the stage's mbarrier.  Warps 1-4
// consume: 8 groups of 16 threads (d = 128, fp16) each own every 8th token of
// the chunk, computing logits with 16-byte shared loads + FMA + shfl_xor and
// keeping an online-softmax state (Eqn 1 fused with Eqn 2, PAPER.md:95-108,
// 145-158; m in log2 units).  At the end of an item the groups and the
// chunk-first partials merge in a fixed order (n-ary Eqn 2: rebase to the
// common max, sum in list order) and O / n is written.  An item
// cut by a CTA boundary writes a segment partial and releases its flag; the
// CTA holding the item's last segment merges all segments in CTA order after
// its own units -- deterministic.
// Stale slots past a partial chunk are never read (select, not multiply).
#include <algorithm>

#include "../host/schedule.h"
#include "common.cuh"
#include "kernels.h"
#include "mma_attn.cuh"

namespace pakv {

using namespace dev;

namespace {

constexpr int kMaxStages = 8;

template <typename T, int D>
struct Geo {
  static constexpr int kVec = Elem<T>::kVec;
  static constexpr int kTpt = D / kVec;     // threads per token row
  static constexpr int kGroups = 128 / kTpt;  // token groups per 128 consumer threads
  static_assert(kTpt <= 32 && (32 % kTpt) == 0, "group must sit inside a warp");
};

// One chunk tile in shared memory with nt valid tokens, consumed by 128
// threads (tid in [0,128)): group g owns tokens g, g + G, ...
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
        const uint4 raw = *reinterpret_cast<const uint4*>(Ks + (size_t)t * D + swz_chunk(t, j) * G::kVec);
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
        const uint4 raw = *reinterpret_cast<const uint4*>(Vs + (size_t)t * D + swz_chunk(t, j) * G::kVec);
        float vf[G::kVec];
        Elem<T>::to_float(raw, vf);
#pragma unroll
        for (int v = 0; v < G::kVec; ++v) o[v] = fmaf(p[u], vf[v], o[v]);
      }
    }
    m = m_new;
  }
}

// ============================================================ seq-first ===
constexpr int kProducerWarps = 1;
constexpr int kConsumerWarps = 4;
constexpr int kSfThreads = (kProducerWarps + kConsumerWarps) * 32;
constexpr int kMaxPrefetchSlots = 4;  // chunk-first partial rows staged per item

enum : int { F_FIRST = 1, F_LAST = 2, F_FULL = 4, F_FINISH = 8, F_CF = 16 };

struct StageMeta {
  int item, nt, flags, caller;
  int mg0, mg1, seg, nsegs;
};

CA_DEV void named_sync_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory"); }

CA_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Shared-memory state of one seq-first CTA.
template <int D, int NG>
struct SfShared {
  uint64_t full_bar[kMaxStages], empty_bar[kMaxStages];
  StageMeta meta[kMaxStages];
  float m[NG], n[NG];
  float o[NG][D];
  int pdl_done;
  int fix_pending;
  StageMeta fix;  // split item this CTA finishes after its own units
};

// Stage layout: K tile | V tile | q row | chunk-first partial rows.
template <typename T, int D>
CA_DEV const float* stage_partials(const unsigned char* st, size_t tile_bytes) {
  return reinterpret_cast<const float*>(st + 2 * tile_bytes + D * sizeof(T));
}

// Producer warp: walk the CTA's units 32 at a time (one descriptor per lane),
// then for every unit wait for a free stage, publish its metadata and issue
// the bulk copies (K, V valid rows; q at a segment start; partial rows at the
// end of an item finished here), all completing on the stage's full barrier.
template <typename T, int D, int NG>
CA_DEV void sf_produce(SfShared<D, NG>& S, unsigned char* smem_raw, const T* __restrict__ kpool,
                       const T* __restrict__ vpool, const T* __restrict__ q, const float* __restrict__ pO,
                       const DevTables& t, int h, int c, int nst, uint32_t stage_bytes, int u0, int u1, int lane,
                       uint64_t* __restrict__ tr, int pf, int cf0, int cf1) {
  constexpr int PR = D + 4;
  const size_t tile_bytes = (size_t)c * D * sizeof(T);
  int jj = 0;
  bool waited = false;  // PDL: append (new token, seq_len) and chunk-first (partials) complete
  // Fused chunk-first units first (shared chunks: untouched by this step's
  // append, so no PDL wait): full K and V tiles of (chunk, head).
  for (int base = cf0; base < cf1; base += 32) {
    const int u = base + lane;
    int tile = 0, head = 0, k = 0, uf = 0, chunk = 0;
    if (u < cf1) {
      const int4 d = *reinterpret_cast<const int4*>(t.cf_unit + (size_t)u * kCfUnitInts);
      tile = d.x;
      head = d.y;
      k = d.z;
      uf = d.w;
      chunk = t.cf_chunk[t.cf_tile[tile * kCfTileInts + CF_CHUNK_OFF] + k];
    }
    const int cnt = min(32, cf1 - base);
    for (int i = 0; i < cnt; ++i) {
      const int i_tile = __shfl_sync(0xffffffffu, tile, i);
      const int i_head = __shfl_sync(0xffffffffu, head, i);
      const int i_k = __shfl_sync(0xffffffffu, k, i);
      const int i_uf = __shfl_sync(0xffffffffu, uf, i);
      const int i_chunk = __shfl_sync(0xffffffffu, chunk, i);
      const int s = jj % nst;
      if (jj >= nst) mbar_wait(&S.empty_bar[s], (uint32_t)(((jj / nst) - 1) & 1));
      if (lane == 0) {
        const int fl = F_CF | ((i_uf & 1) ? F_FIRST : 0) | ((i_uf & 2) ? F_LAST : 0);
        S.meta[s] = StageMeta{i_tile, c, fl, i_head, 0, 0, i_k, 0};
        unsigned char* st = smem_raw + (size_t)s * stage_bytes;
        const size_t off = ((size_t)i_chunk * h + i_head) * c * D;
        mbar_arrive_expect_tx(&S.full_bar[s], 2 * (uint32_t)tile_bytes);
        bulk_g2s(st, kpool + off, (uint32_t)tile_bytes, &S.full_bar[s]);
        bulk_g2s(st + tile_bytes, vpool + off, (uint32_t)tile_bytes, &S.full_bar[s]);
      }
      __syncwarp();
      ++jj;
    }
  }
  for (int base = u0; base < u1; base += 32) {
    const int u = base + lane;
    int chunk = -1, item = 0, k = 0, per = 1, nt = 0, caller = 0, mg0 = 0, mg1 = 0, seg = -1, nsegs = 1;
    int flags = 0, slot4[kMaxPrefetchSlots] = {0, 0, 0, 0};
    if (u < u1) {
      const int4 d = *reinterpret_cast<const int4*>(t.sf_unit + (size_t)u * kSfUnitInts);
      chunk = d.x;
      item = d.y;
      k = d.z;
      per = d.w;
      const int row = item / h;
      caller = t.row_caller[row];
      mg0 = t.mg_ptr[row];
      mg1 = t.mg_ptr[row + 1];
      // only an item's last chunk can be partial -- and it is the one this
      // step's append writes: its length is read after the PDL wait
      if (chunk >= 0) nt = k < per - 1 ? c : (waited ? min(c, t.seq_len[row] - (t.sf_first[row] + k * c)) : -1);
      const bool first = (u == u0) || k == 0;
      const bool last = (u == u1 - 1) || k == per - 1;
      const bool full = (u - k >= u0) && (u - k + per <= u1);
      flags = (first ? F_FIRST : 0) | (last ? F_LAST : 0) | (full ? F_FULL : 0);
      if (last && !full) {
        const int4 rec = *reinterpret_cast<const int4*>(t.sf_item + (size_t)item * kSfItemInts);
        nsegs = rec.y;
        // ordinal among the CTAs touching the item: only a continued first item has one > 0
        const int ord = (u - k < u0) ? t.sf_cta[blockIdx.x * kSfCtaInts + 4] : 0;
        seg = rec.x + ord;
        if (ord == nsegs - 1) flags |= F_FINISH;
      }
      if (last && full) {
#pragma unroll
        for (int e = 0; e < kMaxPrefetchSlots; ++e)
          if (mg0 + e < mg1) slot4[e] = t.mg_slot[mg0 + e];
      }
    }
    // L2 prefetch descriptor of unit u + pf (issued by this lane when unit u goes out)
    const T* pf_k = nullptr;
    uint32_t pf_bytes = 0;
    if (pf > 0 && u + pf < u1) {
      const int4 d2 = *reinterpret_cast<const int4*>(t.sf_unit + (size_t)(u + pf) * kSfUnitInts);
      if (d2.x >= 0) {
        const int row2 = d2.y / h;
        const int nt2 = min(c, t.seq_len[row2] - (t.sf_first[row2] + d2.z * c));
        pf_k = kpool + ((size_t)d2.x * h + (d2.y % h)) * c * D;
        pf_bytes = (uint32_t)(nt2 * D * (int)sizeof(T));
      }
    }
    if (base == u0 && lane < pf && u < u1 && chunk >= 0) {  // the first pf units of the CTA
      const size_t off = ((size_t)chunk * h + (item % h)) * c * D;
      bulk_prefetch_l2(kpool + off, (uint32_t)(nt * D * (int)sizeof(T)));
      bulk_prefetch_l2(vpool + off, (uint32_t)(nt * D * (int)sizeof(T)));
    }
    const int cnt = min(32, u1 - base);
    for (int i = 0; i < cnt; ++i) {
      const int i_chunk = __shfl_sync(0xffffffffu, chunk, i);
      const int i_item = __shfl_sync(0xffffffffu, item, i);
      int i_nt = __shfl_sync(0xffffffffu, nt, i);
      const int i_flags0 = __shfl_sync(0xffffffffu, flags, i);
      if (!waited && (i_nt < 0 || ((i_flags0 & F_LAST) && (i_flags0 & F_FULL)))) {
        pdl_wait();  // first unit touching this step's append / chunk-first output
        waited = true;
      }
      if (i_nt < 0) {  // last chunk of an item described before the wait
        const int row = i_item / h;
        const int k_i = __shfl_sync(0xffffffffu, k, i);
        i_nt = min(c, t.seq_len[row] - (t.sf_first[row] + k_i * c));
      }
#ifdef CA_HANG_CHECK
      if (i_chunk >= 0 && (i_nt <= 0 || i_nt > c)) CA_HANG_TRAP("bad token count", i_item, i_nt);
#endif
      const int i_flags = __shfl_sync(0xffffffffu, flags, i);
      const int i_caller = __shfl_sync(0xffffffffu, caller, i);
      const int i_mg0 = __shfl_sync(0xffffffffu, mg0, i);
      const int i_mg1 = __shfl_sync(0xffffffffu, mg1, i);
      const int i_seg = __shfl_sync(0xffffffffu, seg, i);
      const int i_nsegs = __shfl_sync(0xffffffffu, nsegs, i);
      int my_slot = 0;
#pragma unroll
      for (int e = 0; e < kMaxPrefetchSlots; ++e) {
        const int v = __shfl_sync(0xffffffffu, slot4[e], i);
        if (lane == e) my_slot = v;
      }
      const int s = jj % nst;
      const int head = i_item % h;
      const bool want_q = (i_flags & F_FIRST) && i_chunk >= 0;
      const bool want_p = (i_flags & F_LAST) && (i_flags & F_FULL);
      // fused: the partials are produced inside this kernel -> read at finalize, not staged
      const int np = (want_p && !t.fused) ? min(i_mg1 - i_mg0, kMaxPrefetchSlots) : 0;
      if (jj >= nst) mbar_wait(&S.empty_bar[s], (uint32_t)(((jj / nst) - 1) & 1));
      unsigned char* st = smem_raw + (size_t)s * stage_bytes;
      const uint32_t kv_bytes = (uint32_t)(i_nt * D * (int)sizeof(T));
      const uint32_t q_bytes = want_q ? (uint32_t)(D * sizeof(T)) : 0u;
      const uint32_t p_bytes = (uint32_t)(np * PR * 4);
      if (lane == 0) {
        S.meta[s] = StageMeta{i_item, i_nt, i_flags, i_caller, i_mg0, i_mg1, i_seg, i_nsegs};
        mbar_arrive_expect_tx(&S.full_bar[s], 2 * kv_bytes + q_bytes + p_bytes);
        if (kv_bytes) {
          const size_t off = ((size_t)i_chunk * h + head) * c * D;
          bulk_g2s(st, kpool + off, kv_bytes, &S.full_bar[s]);
          bulk_g2s(st + tile_bytes, vpool + off, kv_bytes, &S.full_bar[s]);
        }
        if (q_bytes) bulk_g2s(st + 2 * tile_bytes, q + ((size_t)i_caller * h + head) * D, q_bytes, &S.full_bar[s]);
      }
      __syncwarp();
      if (lane < np) {
        float* pdst = const_cast<float*>(stage_partials<T, D>(st, tile_bytes)) + lane * PR;
        bulk_g2s(pdst, pO + ((size_t)my_slot * h + head) * PR, PR * 4, &S.full_bar[s]);
      }
      if (lane == i && pf_bytes) {
        bulk_prefetch_l2(pf_k, pf_bytes);
        bulk_prefetch_l2(vpool + (pf_k - kpool), pf_bytes);
      }
      if (tr && lane == 0 && jj < kTraceUnits) tr[3 + 3 * jj] = globaltimer_ns();
      ++jj;
    }
  }
}

// End of an item segment: the NG consumer states sit in S.m/S.n/S.o.  A whole
// item merges the chunk-first partials (staged rows first, the rest from
// global) with the states and writes O / n; a segment of a split item writes
// its partial and the last-arriving segment merges all of them in CTA order.
// n-ary Eqn 2: rebase to the common max, sum in the fixed list order.
// Fused kernel: the chunk-first partials of (row, head) come from other CTAs
// of this launch -- wait for their tiles' readiness flags (this launch's tag).
// Deadlock-free: every CTA runs all its chunk-first units before any
// seq-first unit, and chunk-first work never waits.
CA_DEV void wait_cf_ready(const DevTables& t, const uint32_t* __restrict__ cf_flags, uint32_t tag, int mg0, int mg1,
                          int head, int h, int ct) {
  // warp-uniform trip count: every lane of a warp runs the same iterations
  for (int e0 = mg0 + (ct & ~31); e0 < mg1; e0 += kConsumerWarps * 32) {
    const int e = e0 + (ct & 31);
    const bool mine = e < mg1;
    spin_flags_warp(mine ? cf_flags + (size_t)t.mg_tile[e] * h + head : cf_flags, mine, tag, -1 - e0);
  }
  __threadfence();
  named_sync_consumers();
}

template <typename TO, int D, int NG>
CA_DEV void sf_finalize(SfShared<D, NG>& S, const StageMeta& md, const float* pst, const float* __restrict__ pO,
                        float* __restrict__ segO, uint32_t* __restrict__ segflags, uint32_t tag,
                        const uint32_t* __restrict__ cf_flags, TO* __restrict__ out,
                        const DevTables& t, int h, int ct) {
  constexpr int PR = D + 4;
  const int head = md.item % h;
  if (!S.pdl_done) {  // chunk-first partials (and the append) complete -- waited once per CTA
    pdl_wait();
    named_sync_consumers();
    if (ct == 0) S.pdl_done = 1;
  }
  if (md.flags & F_FULL) {
    if (t.fused) wait_cf_ready(t, cf_flags, tag, md.mg0, md.mg1, head, h, ct);
    const int np = t.fused ? 0 : min(md.mg1 - md.mg0, kMaxPrefetchSlots);
    for (int x = ct; x < D; x += kConsumerWarps * 32) {
      float M = -INFINITY;
      for (int e = 0; e < np; ++e) M = fmaxf(M, pst[e * PR + D]);
      for (int e = md.mg0 + np; e < md.mg1; ++e)
        M = fmaxf(M, __ldcg(pO + ((size_t)t.mg_slot[e] * h + head) * PR + D));
      for (int gg = 0; gg < NG; ++gg) M = fmaxf(M, S.m[gg]);
      float ao = 0.f, an = 0.f;
      for (int e = 0; e < np; ++e) {
        const float w = fast_exp2(pst[e * PR + D] - M);
        ao = fmaf(w, pst[e * PR + x], ao);
        an = fmaf(w, pst[e * PR + D + 1], an);
      }
      for (int e = md.mg0 + np; e < md.mg1; ++e) {
        const float* pr = pO + ((size_t)t.mg_slot[e] * h + head) * PR;
        const float w = fast_exp2(__ldcg(pr + D) - M);
        ao = fmaf(w, __ldcg(pr + x), ao);
        an = fmaf(w, __ldcg(pr + D + 1), an);
      }
      for (int gg = 0; gg < NG; ++gg) {
        const float w = fast_exp2(S.m[gg] - M);
        ao = fmaf(w, S.o[gg][x], ao);
        an = fmaf(w, S.n[gg], an);
      }
      Elem<TO>::store1(out + ((size_t)md.caller * h + head) * D + x, ao / an);
    }
    return;
  }
  for (int x = ct; x < D; x += kConsumerWarps * 32) {
    float M = -INFINITY;
    for (int gg = 0; gg < NG; ++gg) M = fmaxf(M, S.m[gg]);
    float ao = 0.f, an = 0.f;
    for (int gg = 0; gg < NG; ++gg) {
      const float w = M == -INFINITY ? 0.f : fast_exp2(S.m[gg] - M);
      ao = fmaf(w, S.o[gg][x], ao);
      an = fmaf(w, S.n[gg], an);
    }
    float* srow = segO + (size_t)md.seg * PR;
    srow[x] = ao;
    if (x == 0) {
      srow[D] = M;
      srow[D + 1] = an;
    }
  }
  __threadfence();  // every writer's part of the segment row visible GPU-wide ...
  named_sync_consumers();
  if (ct == 0) {
    st_release_gpu(segflags + md.seg, tag);  // ... before its flag
    // The CTA holding the item's last segment meets it first in its range (the
    // item continues from the previous CTA): it finishes the item after its
    // own units, so the ring never stalls on the other segments.
    if (md.flags & F_FINISH) {
      S.fix = md;
      S.fix_pending = 1;
    }
  }
}

// Deferred finish of the split item whose last segment this CTA holds: wait for
// the other segments' flags (this launch's tag), then merge the chunk-first
// partials and all segments in CTA order and write O / n.
template <typename TO, int D, int NG>
CA_DEV void sf_fixup(SfShared<D, NG>& S, const float* __restrict__ pO, const float* __restrict__ segO,
                     const uint32_t* __restrict__ segflags, uint32_t tag, const uint32_t* __restrict__ cf_flags,
                     TO* __restrict__ out, const DevTables& t, int h, int ct) {
  constexpr int PR = D + 4;
  named_sync_consumers();
  if (!S.fix_pending) return;
  const StageMeta md = S.fix;
  const int base = md.seg - (md.nsegs - 1);
  const int head = md.item % h;
  if (t.fused) wait_cf_ready(t, cf_flags, tag, md.mg0, md.mg1, head, h, ct);
  for (int e0 = ct & ~31; e0 < md.nsegs - 1; e0 += kConsumerWarps * 32) {  // warp-uniform
    const int e = e0 + (ct & 31);
    spin_flags_warp(segflags + base + e, e < md.nsegs - 1, tag, base + e0);
  }
  __threadfence();
  named_sync_consumers();
  for (int x = ct; x < D; x += kConsumerWarps * 32) {
    float M = -INFINITY;
    for (int e = md.mg0; e < md.mg1; ++e) M = fmaxf(M, __ldcg(pO + ((size_t)t.mg_slot[e] * h + head) * PR + D));
    for (int sg = 0; sg < md.nsegs; ++sg) M = fmaxf(M, __ldcg(segO + (size_t)(base + sg) * PR + D));
    float ao = 0.f, an = 0.f;
    for (int e = md.mg0; e < md.mg1; ++e) {
      const float* pr = pO + ((size_t)t.mg_slot[e] * h + head) * PR;
      const float w = fast_exp2(__ldcg(pr + D) - M);
      ao = fmaf(w, __ldcg(pr + x), ao);
      an = fmaf(w, __ldcg(pr + D + 1), an);
    }
    for (int sg = 0; sg < md.nsegs; ++sg) {
      const float* sr = segO + (size_t)(base + sg) * PR;
      const float w = fast_exp2(__ldcg(sr + D) - M);
      ao = fmaf(w, __ldcg(sr + x), ao);
      an = fmaf(w, __ldcg(sr + D + 1), an);
    }
    Elem<TO>::store1(out + ((size_t)md.caller * h + head) * D + x, ao / an);
  }
}

// MMA: consumers run WarpAttn with the row's query in row 0 of the 16-row
// tile (warp cw owns the token slice [cw TPW, (cw+1) TPW) of each chunk).
// SIMT (fp32 and fallback): 8 groups x 16 threads own every 8th token.
template <typename T, typename TO, int D, bool MMA, int TPW>
__global__ void __launch_bounds__(kSfThreads) sf_persistent_kernel(
    const T* __restrict__ kpool, const T* __restrict__ vpool, const T* __restrict__ q, TO* __restrict__ out,
    float* __restrict__ pO, float* __restrict__ segO, uint32_t* __restrict__ segflags, uint32_t tag,
    uint32_t* __restrict__ cf_flags, DevTables t, int32_t h, int32_t c, float scale_log2, int32_t nst,
    uint32_t stage_bytes, uint64_t* __restrict__ trace, int32_t pf) {
  using G = Geo<T, D>;
  constexpr int NG = MMA ? kConsumerWarps : G::kGroups;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ SfShared<D, NG> S;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* tr = trace && blockIdx.x < kTraceCtas ? trace + (size_t)blockIdx.x * kTraceStride : nullptr;
  if (tr && tid == 0) tr[0] = globaltimer_ns();
  const int u0 = t.sf_cta[blockIdx.x * kSfCtaInts + 0], u1 = t.sf_cta[blockIdx.x * kSfCtaInts + 1];
  const size_t tile_bytes = (size_t)c * D * sizeof(T);

  // stale shared memory must be finite: masked MMA columns multiply P = 0 by it
  for (size_t i = tid * 16; i < (size_t)nst * stage_bytes; i += kSfThreads * 16)
    *reinterpret_cast<uint4*>(smem_raw + i) = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      S.pdl_done = 0;
      S.fix_pending = 0;
      mbar_init(&S.full_bar[s], 1);
      mbar_init(&S.empty_bar[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  fence_proxy_async();  // generic-proxy zero fill before async-proxy bulk writes
  __syncthreads();

  if (warp == 0) {
    const int cf0 = MMA && t.fused ? t.sf_cta[blockIdx.x * kSfCtaInts + 2] : 0;
    const int cf1 = MMA && t.fused ? t.sf_cta[blockIdx.x * kSfCtaInts + 3] : 0;
    sf_produce<T, D, NG>(S, smem_raw, kpool, vpool, q, pO, t, h, c, nst, stage_bytes, u0, u1, lane, tr, pf, cf0,
                         cf1);
    if (tr && lane == 0) tr[1] = globaltimer_ns();
    return;
  }

  const int ct = tid - 32;  // 0..127
  const int cw = warp - 1;  // consumer warp 0..3
  int jj = 0;
  if constexpr (MMA) {
    using WA = WarpAttn<T, D, TPW>;
    constexpr int PR = D + 4;
    const int L = c / TPW;  // token slices per chunk (<= 4)
    uint32_t qa[WA::KS][4];
    WA wa;
    wa.reset();
    // ---- fused chunk-first units (Alg 1): job = (tile, head); warp (g, l)
    // owns rows [16 g, 16 g + 16) of the tile and the job's chunks k with
    // k % L == l; at the job's end every lane writes its own partial rows and
    // the job's readiness flag is released.
    {
      const int cf0 = t.fused ? t.sf_cta[blockIdx.x * kSfCtaInts + 2] : 0;
      const int cf1 = t.fused ? t.sf_cta[blockIdx.x * kSfCtaInts + 3] : 0;
      int cfL = 1, cfg = 0, cfl = 0, crow0 = 0, crows = 0, cslot = 0;
      bool cact = false;
      for (int u = cf0; u < cf1; ++u, ++jj) {
        const int s = jj % nst;
        mbar_wait(&S.full_bar[s], (uint32_t)((jj / nst) & 1));
        const StageMeta md = S.meta[s];
        const int tile = md.item, head = md.caller, k = md.seg;
        if (md.flags & F_FIRST) {
          const int32_t* rec = t.cf_tile + tile * kCfTileInts;
          crow0 = rec[CF_ROW0];
          crows = rec[CF_ROW1] - crow0;
          cslot = rec[CF_SLOT];
          cfL = rec[CF_LANES];
          cfg = cw / cfL;
          cfl = cw % cfL;
          cact = cfg * 16 < crows;
          wa.reset();
          const int rlo = crow0 + cfg * 16 + (lane >> 2), rhi = rlo + 8;
          const T* qlo = (cact && rlo < crow0 + crows) ? q + ((size_t)t.row_caller[rlo] * h + head) * D : nullptr;
          const T* qhi = (cact && rhi < crow0 + crows) ? q + ((size_t)t.row_caller[rhi] * h + head) * D : nullptr;
          const int cq = (lane & 3) * 2;
#pragma unroll
          for (int ks = 0; ks < WA::KS; ++ks) {
            qa[ks][0] = qlo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16 + cq) : 0u;
            qa[ks][1] = qhi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16 + cq) : 0u;
            qa[ks][2] = qlo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16 + 8 + cq) : 0u;
            qa[ks][3] = qhi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16 + 8 + cq) : 0u;
          }
        }
        if (cact && (k % cfL) == cfl) {
          const uint32_t k_u32 = smem_u32(smem_raw + (size_t)s * stage_bytes);
          for (int t0 = 0; t0 < c; t0 += TPW)
            wa.template chunk<false>(qa, k_u32, k_u32 + (uint32_t)tile_bytes, t0, c, scale_log2, lane);
        }
        if (md.flags & F_LAST) {
          wa.finish();
          if (cact) {
            const int rl = lane >> 2, cq = (lane & 3) * 2;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const int rloc = cfg * 16 + rl + 8 * hf;
              if (rloc < crows) {
                float* prow = pO + ((size_t)(cslot + cfl * crows + rloc) * h + head) * PR;
#pragma unroll
                for (int i = 0; i < WA::DT; ++i)
                  *reinterpret_cast<float2*>(prow + i * 8 + cq) =
                      make_float2(wa.o[i][2 * hf], wa.o[i][2 * hf + 1]);
                if ((lane & 3) == 0)
                  *reinterpret_cast<float2*>(prow + D) =
                      hf ? make_float2(wa.m_hi, wa.n_hi) : make_float2(wa.m_lo, wa.n_lo);
              }
            }
          }
          __threadfence();  // every writer's partial rows visible GPU-wide ...
          named_sync_consumers();
          if (ct == 0) st_release_gpu(cf_flags + (size_t)tile * h + head, tag);  // ... before the flag
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty_bar[s]);
      }
      wa.reset();
    }
    for (int u = u0; u < u1; ++u, ++jj) {
      const int s = jj % nst;
      mbar_wait(&S.full_bar[s], (uint32_t)((jj / nst) & 1));
      if (tr && ct == 0 && jj < kTraceUnits) tr[4 + 3 * jj] = globaltimer_ns();
      const StageMeta md = S.meta[s];
      const unsigned char* st = smem_raw + (size_t)s * stage_bytes;
      if (md.flags & F_FIRST) {
        wa.reset();
        if (md.nt > 0) {
          const uint32_t* q32 = reinterpret_cast<const uint32_t*>(st + 2 * tile_bytes);
#pragma unroll
          for (int ks = 0; ks < WA::KS; ++ks) {
            qa[ks][0] = lane < 4 ? q32[ks * 8 + lane] : 0u;
            qa[ks][2] = lane < 4 ? q32[ks * 8 + 4 + lane] : 0u;
            qa[ks][1] = qa[ks][3] = 0u;
          }
        }
      }
      if (cw < L && cw * TPW < md.nt) {
        const uint32_t k_u32 = smem_u32(st);
        wa.template chunk<true>(qa, k_u32, k_u32 + (uint32_t)tile_bytes, cw * TPW, md.nt, scale_log2, lane);
      }
      if (md.flags & F_LAST) {
        wa.finish();
        if (lane < 4) {  // row 0 lives in lanes 0..3 (c0, c1 of every n-tile)
          if (lane == 0) {
            S.m[cw] = wa.m_lo;
            S.n[cw] = wa.n_lo;
          }
#pragma unroll
          for (int i = 0; i < WA::DT; ++i)
            *reinterpret_cast<float2*>(&S.o[cw][i * 8 + lane * 2]) = make_float2(wa.o[i][0], wa.o[i][1]);
        }
        named_sync_consumers();
        sf_finalize<TO, D, NG>(S, md, stage_partials<T, D>(st, tile_bytes), pO, segO, segflags, tag, cf_flags, out,
                               t, h, ct);
        named_sync_consumers();  // S.o / stage reuse
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty_bar[s]);
      if (tr && ct == 0 && jj < kTraceUnits) tr[5 + 3 * jj] = globaltimer_ns();
    }
  } else {
    const int g = ct / G::kTpt, j = ct % G::kTpt;
    float qf[G::kVec];
    float m = -INFINITY, n = 0.f, o[G::kVec];
    for (int u = u0; u < u1; ++u, ++jj) {
      const int s = jj % nst;
      mbar_wait(&S.full_bar[s], (uint32_t)((jj / nst) & 1));
      if (tr && ct == 0 && jj < kTraceUnits) tr[4 + 3 * jj] = globaltimer_ns();
      const StageMeta md = S.meta[s];
      const unsigned char* st = smem_raw + (size_t)s * stage_bytes;
      if (md.flags & F_FIRST) {
        m = -INFINITY;
        n = 0.f;
#pragma unroll
        for (int v = 0; v < G::kVec; ++v) o[v] = 0.f;
        if (md.nt > 0) {
          const uint4 raw = *reinterpret_cast<const uint4*>(st + 2 * tile_bytes + j * 16);
          Elem<T>::to_float(raw, qf);
#pragma unroll
          for (int v = 0; v < G::kVec; ++v) qf[v] *= scale_log2;
        }
      }
      if (md.nt > 0)
        consume_chunk<T, D>(reinterpret_cast<const T*>(st), reinterpret_cast<const T*>(st + tile_bytes), md.nt, qf,
                            m, n, o, g, j);
      if (md.flags & F_LAST) {
        if (j == 0) {
          S.m[g] = m;
          S.n[g] = n;
        }
#pragma unroll
        for (int v = 0; v < G::kVec; ++v) S.o[g][j * G::kVec + v] = o[v];
        named_sync_consumers();
        sf_finalize<TO, D, NG>(S, md, stage_partials<T, D>(st, tile_bytes), pO, segO, segflags, tag, cf_flags, out,
                               t, h, ct);
        named_sync_consumers();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty_bar[s]);
      if (tr && ct == 0 && jj < kTraceUnits) tr[5 + 3 * jj] = globaltimer_ns();
    }
  }
  (void)cw;
  sf_fixup<TO, D, NG>(S, pO, segO, segflags, tag, cf_flags, out, t, h, ct);
  if (tr && ct == 0) tr[2] = globaltimer_ns();
}

template <typename T, int D>
__global__ void __launch_bounds__(128) cf_simt_kernel(const T* __restrict__ kpool, const T* __restrict__ vpool,
                                                      const T* __restrict__ q, float* __restrict__ pO, DevTables t,
                                                      int32_t h, int32_t c, float scale_log2, int32_t nst) {
  using G = Geo<T, D>;
  constexpr int PR = D + 4;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bars[kMaxStages];
  __shared__ float sm_m[G::kGroups], sm_n[G::kGroups];
  __shared__ float sm_o[G::kGroups][D];

  pdl_launch_dependents();
  const int head = blockIdx.y;
  const int32_t* tile = t.cf_tile + blockIdx.x * kCfTileInts;
  const int row = tile[CF_ROW0] + blockIdx.z;
  if (row >= tile[CF_ROW1]) return;
  const int32_t* chunks = t.cf_chunk + tile[CF_CHUNK_OFF];
  const int n_chunks = tile[CF_NCHUNK];
  const int slot = tile[CF_SLOT] + (int)blockIdx.z;
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
    const uint32_t bytes = (uint32_t)(tile_elems * sizeof(T));
    const size_t off = ((size_t)chunks[k] * h + head) * tile_elems;
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
    consume_chunk<T, D>(Ks + s * tile_elems, Vs + s * tile_elems, c, qf, m, n, o, g, j);
    __syncthreads();
    if (tid == 0 && k + nst < n_chunks) issue(k + nst);
  }
  if (j == 0) {
    sm_m[g] = m;
    sm_n[g] = n;
  }
#pragma unroll
  for (int v = 0; v < G::kVec; ++v) sm_o[g][j * G::kVec + v] = o[v];
  __syncthreads();
  for (int x = tid; x < D; x += 128) {
    float M = -INFINITY;
    for (int gg = 0; gg < G::kGroups; ++gg) M = fmaxf(M, sm_m[gg]);
    float ao = 0.f, an = 0.f;
    for (int gg = 0; gg < G::kGroups; ++gg) {
      const float w = fast_exp2(sm_m[gg] - M);
      ao = fmaf(w, sm_o[gg][x], ao);
      an = fmaf(w, sm_n[gg], an);
    }
    float* prow = pO + ((size_t)slot * h + head) * PR;
    prow[x] = ao;
    if (x == 0) *reinterpret_cast<float4*>(prow + D) = make_float4(M, an, 0.f, 0.f);
  }
  pdl_wait();  // PDL chain: complete only after the append (see chunk_first.cu)
}

cudaError_t set_smem(const void* kern, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  return e;
}

template <typename T, typename TO, int D, bool MMA, int TPW>
cudaError_t launch_sf(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  const PoolGeom& p = a.pool;
  const size_t kv = (size_t)2 * p.c * D * sizeof(T);
  const size_t stage = (kv + D * sizeof(T) + (size_t)kMaxPrefetchSlots * (D + 4) * 4 + 127) / 128 * 128;
  const size_t budget = a.sf_ctas_per_sm == 1 ? (size_t)216 * 1024 : (size_t)108 * 1024;  // per CTA
  int nst = (int)std::min<size_t>(kMaxStages, budget / stage);
  nst = std::max(2, nst);
  const size_t smem = nst * stage;
  auto kern = sf_persistent_kernel<T, TO, D, MMA, TPW>;
  cudaError_t e = set_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  const T* kp = (const T*)p.k + (size_t)a.layer * p.layer_stride;
  const T* vp = (const T*)p.v + (size_t)a.layer * p.layer_stride;
  return launch_ex(kern, dim3(t.n_sf_ctas), dim3(kSfThreads), smem, st, a.use_pdl, kp, vp, (const T*)a.q,
                   (TO*)a.out, a.pO, a.segO, a.segflags, a.tag, a.cf_flags, t, (int32_t)p.h, (int32_t)p.c,
                   a.scale_log2,
                   (int32_t)nst, (uint32_t)stage, a.trace_cf ? (uint64_t*)nullptr : a.trace,
                   (int32_t)std::min(a.sf_prefetch, 31));
}

template <typename T, int D>
cudaError_t launch_cf_simt(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  const PoolGeom& p = a.pool;
  const size_t stage = (size_t)2 * p.c * D * sizeof(T);
  int nst = (int)std::min<size_t>(3, (size_t)(160 * 1024) / stage);
  nst = std::max(1, nst);
  const size_t smem = nst * stage;
  auto kern = cf_simt_kernel<T, D>;
  cudaError_t e = set_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  const T* kp = (const T*)p.k + (size_t)a.layer * p.layer_stride;
  const T* vp = (const T*)p.v + (size_t)a.layer * p.layer_stride;
  return launch_ex(kern, dim3(t.n_cf_tiles, p.h, t.max_tile_rows), dim3(128), smem, st, a.use_pdl, kp, vp,
                   (const T*)a.q, a.pO, t, (int32_t)p.h, (int32_t)p.c, a.scale_log2, (int32_t)nst);
}

// tokens per consumer warp of the MMA seq-first kernel (0 = use SIMT)
int sf_tpw(const AttnLaunch& a) {
  if (a.pool.dtype == DT_F32 || !a.sf_tensor_cores) return 0;
  for (int tpw : {16, 32, 64})
    if (a.pool.c % tpw == 0 && a.pool.c / tpw <= kConsumerWarps) return tpw;
  return 0;
}

template <typename T, typename TO, int D>
cudaError_t dispatch_sf_tpw(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if constexpr (std::is_same<T, float>::value) {
    return launch_sf<T, TO, D, false, 16>(a, t, st);
  } else {
    switch (sf_tpw(a)) {
      case 16: return launch_sf<T, TO, D, true, 16>(a, t, st);
      case 32: return launch_sf<T, TO, D, true, 32>(a, t, st);
      case 64: return launch_sf<T, TO, D, true, 64>(a, t, st);
      default: return launch_sf<T, TO, D, false, 16>(a, t, st);
    }
  }
}

template <typename T>
cudaError_t dispatch_sf(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  const int d = a.pool.d;
  const int od = a.out_dtype;
#define CA_CASE(DD, TO) \
  if (d == DD) return dispatch_sf_tpw<T, TO, DD>(a, t, st);
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

template <typename T>
cudaError_t dispatch_cf(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (a.pool.d == 64) return launch_cf_simt<T, 64>(a, t, st);
  if (a.pool.d == 128) return launch_cf_simt<T, 128>(a, t, st);
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_seq_first(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (t.b == 0) return cudaSuccess;
  switch (a.pool.dtype) {
    case DT_F32: return dispatch_sf<float>(a, t, st);
    case DT_F16: return dispatch_sf<__half>(a, t, st);
    default: return dispatch_sf<__nv_bfloat16>(a, t, st);
  }
}

cudaError_t launch_chunk_first_simt(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (t.n_cf_tiles == 0) return cudaSuccess;
  switch (a.pool.dtype) {
    case DT_F32: return dispatch_cf<float>(a, t, st);
    case DT_F16: return dispatch_cf<__half>(a, t, st);
    default: return dispatch_cf<__nv_bfloat16>(a, t, st);
  }
}

}  // namespace pakv
