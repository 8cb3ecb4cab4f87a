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
// Fused chunk-first token slice per warp and call (>= 32 tokens: 16-token
// mma calls are latency-bound).  64-token calls are cheaper in isolation
// (~1650 vs ~2400 cycles per 64 tokens x 16 rows, tools/warpattn_bench.cu) but
// spill in this kernel's 168-register budget and measured slower (49.0 vs
// 45.5 us per cfg2 step).
constexpr int kCfSlice = 32;

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
constexpr int kMaxPend = kMaxPendingMerges;  // merges one CTA may owe (host-checked)

enum : int { F_FIRST = 1, F_LAST = 2, F_FULL = 4, F_CF = 16 };

struct StageMeta {
  int item, nt, flags, caller;
  int mg0, mg1, seg, nsegs;
};

// barrier.sync (not the .aligned bar.sync): lanes of a warp may arrive on
// different paths (compute-sanitizer synccheck flagged bar.sync here).
CA_DEV void named_sync_consumers() {
  asm volatile("barrier.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}

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
  int n_pend;
  int pend[kMaxPend];      // items whose merge this CTA owes (last contributor)
  int n_contrib;
  int2 contrib[kMaxPend];  // (item, weight) counted at the CTA's end
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
  int rs = 0;         // ring slot of unit jj (jj % nst without a division per unit)
  uint32_t rph = 0;   // its phase parity ((jj / nst) & 1)
  auto ring_next = [&] {
    if (++rs == nst) {
      rs = 0;
      rph ^= 1u;
    }
  };
  bool waited = false;  // PDL: append (new token, seq_len) and chunk-first (partials) complete
  // Fused chunk-first units first (shared chunks: untouched by this step's
  // append, so no PDL wait): full K and V tiles of (chunk, head).
  for (int base = cf0; base < cf1; base += 32) {
    const int u = base + lane;
    int4 d = make_int4(0, 0, 0, 0);  // {chunk, tile, head, k << 2 | flags}
    if (u < cf1) d = *reinterpret_cast<const int4*>(t.cf_unit + (size_t)u * kCfUnitInts);
    const int cnt = min(32, cf1 - base);
    for (int i = 0; i < cnt; ++i) {
      const int i_chunk = __shfl_sync(0xffffffffu, d.x, i);
      const int i_tile = __shfl_sync(0xffffffffu, d.y, i);
      const int i_head = __shfl_sync(0xffffffffu, d.z, i);
      const int i_kf = __shfl_sync(0xffffffffu, d.w, i);
      const int s = rs;
      if (jj >= nst) mbar_wait(&S.empty_bar[s], rph ^ 1u);
      if (lane == 0) {
        const int fl = F_CF | ((i_kf & 1) ? F_FIRST : 0) | ((i_kf & 2) ? F_LAST : 0);
        S.meta[s] = StageMeta{i_tile, c, fl, i_head, 0, 0, i_kf >> 2, 0};
        unsigned char* st = smem_raw + (size_t)s * stage_bytes;
        const size_t off = ((size_t)i_chunk * h + i_head) * c * D;
        mbar_arrive_expect_tx(&S.full_bar[s], 2 * (uint32_t)tile_bytes);
        bulk_g2s(st, kpool + off, (uint32_t)tile_bytes, &S.full_bar[s]);
        bulk_g2s(st + tile_bytes, vpool + off, (uint32_t)tile_bytes, &S.full_bar[s]);
        mbar_arrive_cta(&S.full_bar[s]);  // second arrival (the stage barrier counts 2)
        if (tr && jj < kTraceUnits) {
          tr[3 + 4 * jj] = globaltimer_ns();
          tr[6 + 4 * jj] = 2 * tile_bytes;
        }
      }
      __syncwarp();
      ++jj;
      ring_next();
    }
  }
  for (int base = u0; base < u1; base += 32) {
    const int u = base + lane;
    int chunk = -1, item = 0, k = 0, per = 1, nt = 0, caller = 0, mg0 = 0, mg1 = 0, seg = -1, nsegs = 1;
    int flags = 0, slot4[kMaxPrefetchSlots] = {0, 0, 0, 0};
    if (u < u1) {
      const int4 d0 = *reinterpret_cast<const int4*>(t.sf_unit + (size_t)u * kSfUnitInts);
      const int4 d1 = *reinterpret_cast<const int4*>(t.sf_unit + (size_t)u * kSfUnitInts + 4);
      chunk = d0.x;
      item = d0.y;
      k = d0.z;
      per = d0.w;
      mg0 = d1.x;
      mg1 = d1.y;
      seg = d1.z;
      nsegs = d1.w;
      const int row = item / h;
      // only an item's last chunk can be partial -- and it is the one this
      // step's append writes: its length is read after the PDL wait
      if (chunk >= 0) nt = k < per - 1 ? c : (waited ? min(c, t.seq_len[row] - (t.sf_first[row] + k * c)) : -1);
      const bool first = (u == u0) || k == 0;
      const bool last = (u == u1 - 1) || k == per - 1;
      const bool full = (u - k >= u0) && (u - k + per <= u1);
      flags = (first ? F_FIRST : 0) | (last ? F_LAST : 0) | (full ? F_FULL : 0);
      // dependent loads, consumed only after the unit's K/V copies are issued
      caller = t.row_caller[row];
      if (last && seg < 0 && !t.fused) {
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
        // only full non-last chunks: a last chunk's length is written by this
        // step's append (read before the PDL wait it would race)
        if (d2.z < d2.w - 1) {
          pf_k = kpool + ((size_t)d2.x * h + (d2.y % h)) * c * D;
          pf_bytes = (uint32_t)(c * D * (int)sizeof(T));
        }
      }
    }
    if (base == u0 && lane < pf && u < u1 && chunk >= 0 && nt > 0) {  // the first pf units of the CTA (known length)
      const size_t off = ((size_t)chunk * h + (item % h)) * c * D;
      bulk_prefetch_l2(kpool + off, (uint32_t)(nt * D * (int)sizeof(T)));
      bulk_prefetch_l2(vpool + off, (uint32_t)(nt * D * (int)sizeof(T)));
    }
    const int cnt = min(32, u1 - base);
    for (int i = 0; i < cnt; ++i) {
      const int i_chunk = __shfl_sync(0xffffffffu, chunk, i);
      const int i_item = __shfl_sync(0xffffffffu, item, i);
      int i_nt = __shfl_sync(0xffffffffu, nt, i);
      const int i_flags = __shfl_sync(0xffffffffu, flags, i);
      const int i_mg0 = __shfl_sync(0xffffffffu, mg0, i);
      const int i_mg1 = __shfl_sync(0xffffffffu, mg1, i);
      const int i_seg = __shfl_sync(0xffffffffu, seg, i);
      const int i_nsegs = __shfl_sync(0xffffffffu, nsegs, i);
      // partials staged only for an item finished in place (fused: they are
      // produced inside this kernel, so never staged)
      const bool want_p = (i_flags & F_LAST) && i_seg < 0 && !t.fused;
      if (!waited && (i_nt < 0 || want_p)) {
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
      const int s = rs;
      const int head = i_item % h;
      const bool want_q = (i_flags & F_FIRST) && i_chunk >= 0;
      const int np = want_p ? min(i_mg1 - i_mg0, kMaxPrefetchSlots) : 0;
      if (jj >= nst) mbar_wait(&S.empty_bar[s], rph ^ 1u);
      unsigned char* st = smem_raw + (size_t)s * stage_bytes;
      const uint32_t kv_bytes = (uint32_t)(i_nt * D * (int)sizeof(T));
      const uint32_t q_bytes = want_q ? (uint32_t)(D * sizeof(T)) : 0u;
      const uint32_t p_bytes = (uint32_t)(np * PR * 4);
      // arrival 1: arm every byte of the stage and start the K/V copies (they
      // need only the descriptor) ...
      if (lane == 0) {
        mbar_arrive_expect_tx(&S.full_bar[s], 2 * kv_bytes + q_bytes + p_bytes);
        if (kv_bytes) {
          const size_t off = ((size_t)i_chunk * h + head) * c * D;
          bulk_g2s(st, kpool + off, kv_bytes, &S.full_bar[s]);
          bulk_g2s(st + tile_bytes, vpool + off, kv_bytes, &S.full_bar[s]);
        }
      }
      // ... arrival 2 publishes the metadata once the dependent loads (caller,
      // partial slots) are in; then the q row and the partial rows
      const int i_caller = __shfl_sync(0xffffffffu, caller, i);
      int my_slot = 0;
#pragma unroll
      for (int e = 0; e < kMaxPrefetchSlots; ++e) {
        const int v = __shfl_sync(0xffffffffu, slot4[e], i);
        if (lane == e) my_slot = v;
      }
      if (lane == 0) {
        S.meta[s] = StageMeta{i_item, i_nt, i_flags, i_caller, i_mg0, i_mg1, i_seg, i_nsegs};
        mbar_arrive_cta(&S.full_bar[s]);
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
      if (tr && lane == 0 && jj < kTraceUnits) {
        tr[3 + 4 * jj] = globaltimer_ns();
        tr[6 + 4 * jj] = 2 * kv_bytes + q_bytes + p_bytes;
      }
      ++jj;
      ring_next();
    }
  }
}

// Queue an item whose last contribution this CTA made: merged at the CTA's end.
template <int D, int NG>
CA_DEV void push_pending(SfShared<D, NG>& S, int item) {
  const int i = atomicAdd(&S.n_pend, 1);
  if (i < kMaxPend) S.pend[i] = item;
#ifdef CA_HANG_CHECK
  else CA_HANG_TRAP("pending merge list overflow", item, i);
#endif
}

// Record a contribution (its partial rows are written): counted at the CTA's
// end, so the stream never stalls on a GPU-scope fence.
template <int D, int NG>
CA_DEV void record_contribution(SfShared<D, NG>& S, int item, int w) {
  const int i = atomicAdd(&S.n_contrib, 1);
  if (i < kMaxPend) S.contrib[i] = make_int2(item, w);
#ifdef CA_HANG_CHECK
  else CA_HANG_TRAP("contribution list overflow", item, i);
#endif
}

// CTA end: one warp counts the CTA's recorded contributions (segments of items
// merged elsewhere).  The CTA barrier orders every writer's partial rows
// before the warp's release fence (cumulative); the adds are relaxed.
template <int D, int NG>
CA_DEV void settle_contributions(SfShared<D, NG>& S, uint32_t* __restrict__ cnt, int ct) {
  named_sync_consumers();
  const int n = min(S.n_contrib, kMaxPend);
  if (ct < 32 && n > 0) {
    fence_acq_rel_gpu();
    for (int i = ct; i < n; i += 32) {
      const int2 c = S.contrib[i];
      atomicAdd(cnt + c.x, (uint32_t)c.y);
    }
  }
}

// End of an item segment: the NG consumer states sit in S.m/S.n/S.o.  An item
// finished here with no outside contribution (one segment; chunk-first
// partials already complete) merges the chunk-first partials (staged rows
// first, the rest from global) with the states and writes O / n.  Otherwise the
// segment's state goes to its slot in segO and the item's counter is bumped:
// the last contributor (a segment, or in the fused kernel a chunk-first job)
// merges everything in the fixed list order (chunk-first partials in merge-list
// order, then the segments in CTA order): deterministic, and nobody waits.
// n-ary Eqn 2: rebase to the common max, sum in the fixed list order.
template <typename TO, int D, int NG>
CA_DEV void sf_finalize(SfShared<D, NG>& S, const StageMeta& md, const float* pst, const float* __restrict__ pO,
                        float* __restrict__ segO, uint32_t* __restrict__ cnt, TO* __restrict__ out,
                        const DevTables& t, int h, int ct) {
  constexpr int PR = D + 4;
  const int head = md.item % h;
  if (!S.pdl_done) {  // append (and chunk-first partials when not fused) complete -- waited once per CTA
    pdl_wait();
    named_sync_consumers();
    if (ct == 0) S.pdl_done = 1;
  }
  if (md.seg < 0) {
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
  if (ct == 0) {
    if (md.nsegs & kSfMerger)
      push_pending(S, md.item);  // this CTA merges the item at its end
    else
      record_contribution(S, md.item, 1);
  }
}

// The CTA's owed merges (items whose last segment it holds), one warp per
// item -- all five warps once the producer is done -- after all its own units:
// wait until the item's other contributions are counted (chunk-first jobs of
// this launch when fused, the earlier segments), then merge the row's
// chunk-first partials in merge-list order and the item's segments in CTA
// order (n-ary Eqn 2, fixed order).  Lane e holds contribution e's row
// pointer (resolved before the wait) and (m, n); the (m, n) loads and the
// first 8 rows (each lane 4 columns of every row) go out in one round.
// Writes O / n and resets the counter.  Deadlock-free: chunk-first work never
// waits and every CTA counts its own contributions before it waits; the grid
// is one wave (2 CTAs per SM).
constexpr int kMergeWarps = kProducerWarps + kConsumerWarps;
CA_DEV void named_sync_all() {  // non-.aligned barrier: lanes may arrive from different paths
  asm volatile("barrier.sync 2, %0;" ::"n"(kMergeWarps * 32) : "memory");
}

template <typename TO, int D, int NG>
CA_DEV void merge_pending(SfShared<D, NG>& S, const float* __restrict__ pO, const float* __restrict__ segO,
                          uint32_t* __restrict__ cnt, TO* __restrict__ out, const DevTables& t, int h, int mt) {
  constexpr int PR = D + 4;
  constexpr int RB = 8;  // rows per load round
  named_sync_all();
  const int np = min(S.n_pend, kMaxPend);
  const int lane = mt & 31;
  for (int p = mt >> 5; p < np; p += kMergeWarps) {
    const int item = S.pend[p];
    const int row = item / h, head = item % h;
    const int mg0 = t.mg_ptr[row], ncf = t.mg_ptr[row + 1] - mg0;
    const int4 rec = *reinterpret_cast<const int4*>(t.sf_item + (size_t)item * kSfItemInts);
    const int E = ncf + rec.y;
    TO* orow = out + ((size_t)t.row_caller[row] * h + head) * D;
    const uint32_t others = (uint32_t)((t.fused ? ncf : 0) + rec.y - 1);
    const float* pr = nullptr;
    if (E <= 32 && lane < E)
      pr = lane < ncf ? pO + ((size_t)t.mg_slot[mg0 + lane] * h + head) * PR : segO + (size_t)(rec.x + lane - ncf) * PR;
    if (others > 0) spin_flags_warp(cnt + item, lane == 0, others, item);
    __syncwarp();
    if (E <= 32) {
      const uint64_t pu = reinterpret_cast<uint64_t>(pr);
      const bool colv = lane * 4 < D;
      float4 v[RB];
      float me = -INFINITY, ne = 0.f;
      auto load_rows = [&](int e0) {
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const int e = e0 + r;
          const uint64_t pe = (uint64_t)__shfl_sync(0xffffffffu, (uint32_t)pu, e & 31) |
                              ((uint64_t)__shfl_sync(0xffffffffu, (uint32_t)(pu >> 32), e & 31) << 32);
          v[r] = (e < E && colv) ? __ldcg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(pe) + lane * 4))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      if (lane < E) {
        const float2 mn = __ldcg(reinterpret_cast<const float2*>(pr + D));
        me = mn.x;
        ne = mn.y;
      }
      load_rows(0);
      float M = me;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
      const float w = lane < E ? fast_exp2(me - M) : 0.f;
      float nsum = w * ne;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, off);
      float4 ao = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int e0 = 0; e0 < E; e0 += RB) {
        if (e0 > 0) load_rows(e0);
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const float we = __shfl_sync(0xffffffffu, w, (e0 + r) & 31);  // 0 past E
          ao.x = fmaf(we, v[r].x, ao.x);
          ao.y = fmaf(we, v[r].y, ao.y);
          ao.z = fmaf(we, v[r].z, ao.z);
          ao.w = fmaf(we, v[r].w, ao.w);
        }
      }
      if (colv) {
        Elem<TO>::store1(orow + lane * 4 + 0, ao.x / nsum);
        Elem<TO>::store1(orow + lane * 4 + 1, ao.y / nsum);
        Elem<TO>::store1(orow + lane * 4 + 2, ao.z / nsum);
        Elem<TO>::store1(orow + lane * 4 + 3, ao.w / nsum);
      }
    } else {  // many contributions: per-column passes
      for (int x = lane * 4; x < D; x += 128) {
        float M = -INFINITY;
        for (int e = 0; e < ncf; ++e) M = fmaxf(M, __ldcg(pO + ((size_t)t.mg_slot[mg0 + e] * h + head) * PR + D));
        for (int sg = 0; sg < rec.y; ++sg) M = fmaxf(M, __ldcg(segO + (size_t)(rec.x + sg) * PR + D));
        float4 ao = make_float4(0.f, 0.f, 0.f, 0.f);
        float an = 0.f;
        auto add = [&](const float* prr) {
          const float w = fast_exp2(__ldcg(prr + D) - M);
          const float4 v = __ldcg(reinterpret_cast<const float4*>(prr + x));
          ao.x = fmaf(w, v.x, ao.x);
          ao.y = fmaf(w, v.y, ao.y);
          ao.z = fmaf(w, v.z, ao.z);
          ao.w = fmaf(w, v.w, ao.w);
          an = fmaf(w, __ldcg(prr + D + 1), an);
        };
        for (int e = 0; e < ncf; ++e) add(pO + ((size_t)t.mg_slot[mg0 + e] * h + head) * PR);
        for (int sg = 0; sg < rec.y; ++sg) add(segO + (size_t)(rec.x + sg) * PR);
        Elem<TO>::store1(orow + x + 0, ao.x / an);
        Elem<TO>::store1(orow + x + 1, ao.y / an);
        Elem<TO>::store1(orow + x + 2, ao.z / an);
        Elem<TO>::store1(orow + x + 3, ao.w / an);
      }
    }
    if (lane == 0) cnt[item] = 0u;
  }
}

// MMA: consumers run WarpAttn with the row's query in row 0 of the 16-row
// tile (warp cw owns the token slice [cw TPW, (cw+1) TPW) of each chunk).
// SIMT (fp32 and fallback): 8 groups x 16 threads own every 8th token.
template <typename T, typename TO, int D, bool MMA, int TPW>
__global__ void __launch_bounds__(kSfThreads, 2) sf_persistent_kernel(
    const T* __restrict__ kpool, const T* __restrict__ vpool, const T* __restrict__ q, TO* __restrict__ out,
    float* __restrict__ pO, float* __restrict__ segO, uint32_t* __restrict__ cnt, DevTables t, int32_t h, int32_t c, float scale_log2, int32_t nst,
    uint32_t stage_bytes, uint64_t* __restrict__ trace, int32_t pf) {
  using G = Geo<T, D>;
  constexpr int NG = MMA ? kConsumerWarps : G::kGroups;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ SfShared<D, NG> S;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool diag_nocompute = (pf & 256) != 0;  // diagnostic: stream only (outputs wrong)
  pf &= 255;
  uint64_t* tr = trace && blockIdx.x < kTraceCtas ? trace + (size_t)blockIdx.x * kTraceStride : nullptr;
  if (tr && tid == 0) tr[0] = globaltimer_ns();
  const int u0 = t.sf_cta[blockIdx.x * kSfCtaInts + 0], u1 = t.sf_cta[blockIdx.x * kSfCtaInts + 1];
  const size_t tile_bytes = (size_t)c * D * sizeof(T);

  // no zero fill: stale rows past a partial chunk are masked by select (S) and
  // zeroed in the B fragments (V, mma_attn.cuh); the SIMT path never reads them
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      S.pdl_done = 0;
      S.n_pend = 0;
      S.n_contrib = 0;
      mbar_init(&S.full_bar[s], 2);  // producer: arm + copies, then metadata
      mbar_init(&S.empty_bar[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == 0) {
    const int cf0 = MMA && t.fused ? t.sf_cta[blockIdx.x * kSfCtaInts + 2] : 0;
    const int cf1 = MMA && t.fused ? t.sf_cta[blockIdx.x * kSfCtaInts + 3] : 0;
    sf_produce<T, D, NG>(S, smem_raw, kpool, vpool, q, pO, t, h, c, nst, stage_bytes, u0, u1, lane, tr, pf, cf0,
                         cf1);
    if (tr && lane == 0) tr[1] = globaltimer_ns();
    merge_pending<TO, D, NG>(S, pO, segO, cnt, out, t, h, kConsumerWarps * 32 + lane);  // fifth merge warp
    return;
  }

  const int ct = tid - 32;  // 0..127
  const int cw = warp - 1;  // consumer warp 0..3
  int jj = 0;
  int rs = 0;        // ring slot / phase of unit jj, advanced without divisions
  uint32_t rph = 0;
  auto ring_next = [&] {
    if (++rs == nst) {
      rs = 0;
      rph ^= 1u;
    }
  };
  if constexpr (MMA) {
    using WA = WarpAttn<T, D, TPW>;
    constexpr int PR = D + 4;
    const int L = c / TPW;  // token slices per chunk (<= 4)
    uint32_t qa[WA::KS][4];
    WA wa;
    wa.reset();
    // ---- fused chunk-first units (Alg 1): job = (tile, head); warp (g, l)
    // owns rows [16 g, 16 g + 16) of the tile and lane l's token slice of
    // the job's chunks; at the job's end every lane writes its own partial
    // rows and the job's contribution is counted.
    {
      const int cf0 = t.fused ? t.sf_cta[blockIdx.x * kSfCtaInts + 2] : 0;
      const int cf1 = t.fused ? t.sf_cta[blockIdx.x * kSfCtaInts + 3] : 0;
      int cfL = 1, cfP = 1, cfg = 0, cfl = 0, crow0 = 0, crows = 0, cslot = 0;
      int c_altm = 0, c_sel = 0, c_span = c, c_tb = 0;  // this warp's chunk / token slice of the job
      bool cact = false;
      // a job's tile record and Q fragments (dependent global loads): the
      // CTA's first job is begun at kernel start, overlapping the first copies
      auto begin_job = [&](int tile, int head) {
        const int32_t* rec = t.cf_tile + tile * kCfTileInts;
        crow0 = rec[CF_ROW0];
        crows = rec[CF_ROW1] - crow0;
        cslot = rec[CF_SLOT];
        cfL = rec[CF_LANES];
        cfP = rec[CF_PARTS];
        cfg = cw / cfL;
        cfl = cw % cfL;
        cact = cfg * 16 < crows;
        {  // lane l: token slice l % nsl of every alt-th chunk (nsl, alt powers of two)
          int nsl = cfL;  // slices per chunk: divides cfL and c / 16, >= kCfSlice tokens each
          while (nsl > 1 && (nsl * kCfSlice > c || (c / 16) % nsl != 0)) nsl >>= 1;
          c_altm = cfL / nsl - 1;
          c_sel = cfl / nsl;
          c_span = c / nsl;
          c_tb = (cfl % nsl) * c_span;
        }
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
      };
      if (cf0 < cf1) {
        const int4 d0 = *reinterpret_cast<const int4*>(t.cf_unit + (size_t)cf0 * kCfUnitInts);
        begin_job(d0.y, d0.z);
      }
      for (int u = cf0; u < cf1; ++u, ++jj, ring_next()) {
        const int s = rs;
        mbar_wait(&S.full_bar[s], rph);
        if (tr && ct == 0 && jj < kTraceUnits) tr[4 + 4 * jj] = globaltimer_ns();
        const StageMeta md = S.meta[s];
        const int tile = md.item, head = md.caller, k = md.seg;
        if ((md.flags & F_FIRST) && u != cf0) begin_job(tile, head);
        // lane l of the job: token slice l % nsl (>= 32 tokens when the chunk
        // has them) of every alt-th chunk (k % alt == l / nsl): all warps work
        // on each unit, and each mma call covers 32-64 tokens (independent
        // accumulator chains; 16-token calls are latency-bound).  Resolved once
        // per job (begin_job): no integer division per unit.
        if (cact && (k & c_altm) == c_sel && !diag_nocompute) {
          const uint32_t k_u32 = smem_u32(smem_raw + (size_t)s * stage_bytes), v_u32 = k_u32 + (uint32_t)tile_bytes;
          int t0 = c_tb;
          for (; t0 + 32 <= c_tb + c_span; t0 += 32)
            wa.template chunk<false, 32>(qa, k_u32, v_u32, t0, c, scale_log2, lane);
          for (; t0 < c_tb + c_span; t0 += 16) wa.template chunk<false, 16>(qa, k_u32, v_u32, t0, c, scale_log2, lane);
        }
        if (md.flags & F_LAST) {
          wa.finish();
          if (cfP == 1 && cfL > 1) {
            // merge the token lanes of each row group in this stage's K/V
            // tiles (every warp is done with them; the stage is released
            // after): lanes l > 0 store their states, lane 0 folds them in
            // lane order (Eqn 2) and writes the job's single partial row
            constexpr int NR = WA::DT * 4 + 4;
            float* scr = reinterpret_cast<float*>(smem_raw + (size_t)s * stage_bytes);
            named_sync_consumers();
            if (cfl > 0 && cact) {
              float* my = scr + (size_t)(cfg * (cfL - 1) + cfl - 1) * NR * 32 + lane;
#pragma unroll
              for (int i = 0; i < WA::DT; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) my[(i * 4 + j) * 32] = wa.o[i][j];
              my[(NR - 4) * 32] = wa.m_lo;
              my[(NR - 3) * 32] = wa.m_hi;
              my[(NR - 2) * 32] = wa.n_lo;
              my[(NR - 1) * 32] = wa.n_hi;
              fence_proxy_async();  // generic writes before the stage's next bulk copy
            }
            named_sync_consumers();
            if (cfl == 0 && cact) {
              const float* ot = scr + (size_t)cfg * (cfL - 1) * NR * 32 + lane;
              float M_lo = wa.m_lo, M_hi = wa.m_hi;
              for (int l = 1; l < cfL; ++l) {
                M_lo = fmaxf(M_lo, ot[((l - 1) * NR + NR - 4) * 32]);
                M_hi = fmaxf(M_hi, ot[((l - 1) * NR + NR - 3) * 32]);
              }
              const float b_lo = M_lo == -INFINITY ? 0.f : M_lo, b_hi = M_hi == -INFINITY ? 0.f : M_hi;
              const float w_lo = fast_exp2(wa.m_lo - b_lo), w_hi = fast_exp2(wa.m_hi - b_hi);
              wa.n_lo *= w_lo;
              wa.n_hi *= w_hi;
#pragma unroll
              for (int i = 0; i < WA::DT; ++i) {
                wa.o[i][0] *= w_lo;
                wa.o[i][1] *= w_lo;
                wa.o[i][2] *= w_hi;
                wa.o[i][3] *= w_hi;
              }
              for (int l = 1; l < cfL; ++l) {
                const float* ol = ot + (size_t)(l - 1) * NR * 32;
                const float vl = fast_exp2(ol[(NR - 4) * 32] - b_lo), vh = fast_exp2(ol[(NR - 3) * 32] - b_hi);
                wa.n_lo = fmaf(vl, ol[(NR - 2) * 32], wa.n_lo);
                wa.n_hi = fmaf(vh, ol[(NR - 1) * 32], wa.n_hi);
#pragma unroll
                for (int i = 0; i < WA::DT; ++i) {
                  wa.o[i][0] = fmaf(vl, ol[(i * 4 + 0) * 32], wa.o[i][0]);
                  wa.o[i][1] = fmaf(vl, ol[(i * 4 + 1) * 32], wa.o[i][1]);
                  wa.o[i][2] = fmaf(vh, ol[(i * 4 + 2) * 32], wa.o[i][2]);
                  wa.o[i][3] = fmaf(vh, ol[(i * 4 + 3) * 32], wa.o[i][3]);
                }
              }
              wa.m_lo = M_lo;
              wa.m_hi = M_hi;
            }
          }
          if (cact && (cfP > 1 || cfl == 0)) {
            const int rl = lane >> 2, cq = (lane & 3) * 2;
            const int pl = cfP > 1 ? cfl : 0;  // partial index of this lane
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const int rloc = cfg * 16 + rl + 8 * hf;
              if (rloc < crows) {
                float* prow = pO + ((size_t)(cslot + pl * crows + rloc) * h + head) * PR;
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
          // counted now (one fence per job, early in the CTA): each row's
          // merger (the CTA holding its item's last segment) waits for them
          named_sync_consumers();
          if (ct < crows) {
            fence_acq_rel_gpu();
            atomicAdd(cnt + (crow0 + ct) * h + head, (uint32_t)cfP);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty_bar[s]);
        if (tr && ct == 0 && jj < kTraceUnits) tr[5 + 4 * jj] = globaltimer_ns();
      }
      wa.reset();
    }
    for (int u = u0; u < u1; ++u, ++jj, ring_next()) {
      const int s = rs;
      mbar_wait(&S.full_bar[s], rph);
      if (tr && ct == 0 && jj < kTraceUnits) tr[4 + 4 * jj] = globaltimer_ns();
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
      if (cw < L && cw * TPW < md.nt && !diag_nocompute) {
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
        sf_finalize<TO, D, NG>(S, md, stage_partials<T, D>(st, tile_bytes), pO, segO, cnt, out,
                               t, h, ct);
        named_sync_consumers();  // S.o / stage reuse
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty_bar[s]);
      if (tr && ct == 0 && jj < kTraceUnits) tr[5 + 4 * jj] = globaltimer_ns();
    }
  } else {
    const int g = ct / G::kTpt, j = ct % G::kTpt;
    float qf[G::kVec];
    float m = -INFINITY, n = 0.f, o[G::kVec];
    for (int u = u0; u < u1; ++u, ++jj, ring_next()) {
      const int s = rs;
      mbar_wait(&S.full_bar[s], rph);
      if (tr && ct == 0 && jj < kTraceUnits) tr[4 + 4 * jj] = globaltimer_ns();
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
        sf_finalize<TO, D, NG>(S, md, stage_partials<T, D>(st, tile_bytes), pO, segO, cnt, out,
                               t, h, ct);
        named_sync_consumers();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty_bar[s]);
      if (tr && ct == 0 && jj < kTraceUnits) tr[5 + 4 * jj] = globaltimer_ns();
    }
  }
  (void)cw;
  settle_contributions(S, cnt, ct);
  if (tr && ct == 0) tr[kTraceStride - 1] = globaltimer_ns();  // merge phase start
  merge_pending<TO, D, NG>(S, pO, segO, cnt, out, t, h, ct);
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

cudaError_t set_smem(const void* kern, size_t smem) { return set_smem_once(kern, smem); }

size_t sf_stage_bytes(int32_t dtype, int32_t c, int32_t d) {
  const size_t e = (size_t)dtype_bytes(dtype);
  const size_t kv = (size_t)2 * c * d * e;
  return (kv + d * e + (size_t)kMaxPrefetchSlots * (d + 4) * 4 + 127) / 128 * 128;
}

// ring depth for the per-CTA shared-memory budget (>= 2; valid_config
// guarantees two stages fit the opt-in limit)
int sf_stages(int32_t dtype, int32_t c, int32_t d, int sf_ctas_per_sm) {
  const size_t stage = sf_stage_bytes(dtype, c, d);
  const size_t budget = sf_ctas_per_sm == 1 ? (size_t)216 * 1024 : (size_t)108 * 1024;  // per CTA
  int nst = (int)std::min<size_t>(kMaxStages, budget / stage);
  return std::max(2, nst);
}

template <typename T, typename TO, int D, bool MMA, int TPW>
cudaError_t launch_sf(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  const PoolGeom& p = a.pool;
  const size_t stage = sf_stage_bytes(p.dtype, p.c, D);
  const int nst = sf_stages(p.dtype, p.c, D, a.sf_ctas_per_sm);
  const size_t smem = nst * stage;
  auto kern = sf_persistent_kernel<T, TO, D, MMA, TPW>;
  cudaError_t e = set_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  const T* kp = (const T*)p.k + (size_t)a.layer * p.layer_stride;
  const T* vp = (const T*)p.v + (size_t)a.layer * p.layer_stride;
  return launch_ex(kern, dim3(t.n_sf_ctas), dim3(kSfThreads), smem, st, a.use_pdl, kp, vp, (const T*)a.q,
                   (TO*)a.out, a.pO, a.segO, a.counters, t, (int32_t)p.h, (int32_t)p.c,
                   a.scale_log2,
                   (int32_t)nst, (uint32_t)stage, a.trace_cf ? (uint64_t*)nullptr : a.trace,
                   (int32_t)(std::min(a.sf_prefetch & 255, 31) | (a.sf_prefetch & 256)));
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
int sf_tpw(const AttnLaunch& a) { return sf_mma_tpw(a.pool.dtype, a.pool.c, a.sf_tensor_cores); }

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

template <typename T, typename TO, int D>
const void* sf_kernel_tpw(int tpw) {
  if constexpr (std::is_same<T, float>::value) {
    return (const void*)sf_persistent_kernel<T, TO, D, false, 16>;
  } else {
    switch (tpw) {
      case 16: return (const void*)sf_persistent_kernel<T, TO, D, true, 16>;
      case 32: return (const void*)sf_persistent_kernel<T, TO, D, true, 32>;
      case 64: return (const void*)sf_persistent_kernel<T, TO, D, true, 64>;
      default: return (const void*)sf_persistent_kernel<T, TO, D, false, 16>;
    }
  }
}

template <typename T>
const void* sf_kernel_ptr(int d, int od, int tpw) {
#define CA_CASE(DD, TO) \
  if (d == DD) return sf_kernel_tpw<T, TO, DD>(tpw);
  if (od == DT_F32) {
    CA_CASE(64, float) CA_CASE(128, float)
  } else if (od == DT_F16) {
    CA_CASE(64, __half) CA_CASE(128, __half)
  } else {
    CA_CASE(64, __nv_bfloat16) CA_CASE(128, __nv_bfloat16)
  }
#undef CA_CASE
  return nullptr;
}

template <typename T>
cudaError_t dispatch_cf(const AttnLaunch& a, const DevTables& t, cudaStream_t st) {
  if (a.pool.d == 64) return launch_cf_simt<T, 64>(a, t, st);
  if (a.pool.d == 128) return launch_cf_simt<T, 128>(a, t, st);
  return cudaErrorInvalidValue;
}

}  // namespace

size_t seq_first_min_smem(int32_t dtype, int32_t c, int32_t d) { return 2 * sf_stage_bytes(dtype, c, d); }

int seq_first_resident_ctas(const PoolGeom& p, int out_dtype, int sf_ctas_per_sm, bool sf_tensor_cores) {
  const int tpw = sf_mma_tpw(p.dtype, p.c, sf_tensor_cores);
  const void* kern = p.dtype == DT_F32   ? sf_kernel_ptr<float>(p.d, out_dtype, tpw)
                     : p.dtype == DT_F16 ? sf_kernel_ptr<__half>(p.d, out_dtype, tpw)
                                         : sf_kernel_ptr<__nv_bfloat16>(p.d, out_dtype, tpw);
  if (!kern) return 0;
  const size_t smem = (size_t)sf_stages(p.dtype, p.c, p.d, sf_ctas_per_sm) * sf_stage_bytes(p.dtype, p.c, p.d);
  if (set_smem(kern, smem) != cudaSuccess) return 0;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSfThreads, smem) != cudaSuccess)
    return 0;
  return per_sm * sms;
}

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
