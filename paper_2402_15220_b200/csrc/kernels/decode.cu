// K5 cluster decode: one launch per decode step = K1 append (the step's new
// K/V row) + K3 chunk-first (Alg 1, Eqn 1
// :95-108) + K4 seq-first (Alg 2) + the Eqn 2 merge
// + O / n.
//
// Work decomposition (host: schedule.cpp, "dk" tables).  The DFS rows are cut
// into blocks of <= kDkMaxRows rows.  A GROUP = (row block, set of hg heads)
// is computed by one thread-block CLUSTER of cs CTAs, one CTA per SM (the
// host picks hg and cs so that all groups run in one wave and fill the SMs).
// The group's work list -- per head of the set: every shared run clipped to
// the block (chunk-first units: one (chunk, head) K/V tile x all the run's
// rows of the block), then every row's full private chunks (cooperative
// seq-first units) -- is cut into cs contiguous pieces of equal estimated
// cost; every row's last chunk (short in decode) is dealt to the least-loaded
// ranks in packs of up to one row per consumer warp.  Each CTA folds every job
// it runs (a maximal stretch of one run / one row inside its piece) into a
// per-(head, row) online-softmax state (o, m, n) in shared memory, in job
// order (Eqn 2).  At the end the CTAs of the cluster merge the cs states of
// every (head, row) over distributed shared memory in rank order (Eqn 2,
// n-ary form) and write O / n.  No partials in global memory, no counters, no
// cross-CTA waiting outside the cluster barrier: deterministic, any grid is
// safe.
//
// CTA (one per SM, 12 warps) = 1 producer warp (unit descriptors -> 1-D bulk
// copies of the valid tokens of each (chunk, head) K and V tile into an
// NST-deep ring) + 3 idle warps + NC = 8 mma.sync consumer warps
// (mma_attn.cuh WarpAttn):
//   chunk-first job (rows [r0, r0 + nr) <= 64): warp (g, l) = 16 query rows x
//     token slice of every (alt)-th chunk, so consecutive chunks are computed
//     by different warps at once; Q fragments straight from global;
//   cooperative seq-first job (one row, full chunks): warp w = token slice w;
//   PACK (rows' last chunks, 16-token slots): warp w = all of row w's chunk.
// K1 folded in: a row's last chunk reaches the stage as its old tokens (pool)
// plus the new K/V rows copied from the caller's k / v into staging rows of
// the stage (the MMA reads that token's ldmatrix rows from there); the
// consumer warp that attends it writes those rows into the pool slot.
// m is kept in log2 units (scale * log2 e folded into the logits).
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "../host/schedule.h"
#include "common.cuh"
#include "kernels.h"
#include "mma_attn.cuh"
#include "umma.cuh"

namespace pakv {

using namespace dev;

namespace {

// 12 warps in both variants.
//   mma.sync variant (UM = false): warpgroup 0 = the producer warp + 3 idle
//     warps; warpgroups 1-2 = NC = 8 mma.sync consumer warps (every unit).
//   tcgen05 variant (UM = true, c = 64): warp 0 = the seq-first producer
//     (private units and packs, 1-D bulk copies), warp 1 = the chunk-first
//     TMA producer (2-D boxes of the K / V tiles, SWIZZLE_128B images), warp 2
//     = the MMA issuer (one thread: S = Q K^T, O += P V, M = 64, S double
//     buffered and O in TMEM), warp 3 idle; warpgroup 1 = the softmax warps
//     (thread = query row = TMEM lane: the M = 64 layout puts row 16 q + i in
//     lane 32 q + i, so lanes 0-15 of each warp hold rows); warpgroup 2 = NC =
//     4 mma.sync consumer warps for the private units.  The two phases of the
//     paper run concurrently on one SM: tensor cores for the shared chunks,
//     the CUDA-core GEMV ring for the private ones.
// Registers are re-balanced per warpgroup with setmaxnreg.
constexpr int kDkThreads = 12 * 32;
constexpr int kRegsLow = 80, kRegsHigh = 208;            // mma.sync variant: 80 + 2 x 208 <= 3 x 168
constexpr int kRegsLowUm = 80, kRegsSoftmax = 208, kRegsConsumerUm = 216;  // tcgen05 variant: 80 + 208 + 216 = 3 x 168
constexpr int kDkMaxStages = 8;
constexpr int kDkSlice = 32;                     // chunk-first token slice per warp and call (>= 32: latency)
constexpr size_t kDkSmemBudget = 232448 - 3328;  // 227 KB opt-in, minus static shared memory (<= 3 KB, ptxas)
constexpr int kStateRows = kDkMaxRows;           // (head, row) states per CTA: hg * block rows <= 64
constexpr int kMergeWarp0 = 4, kMergeThreads = 256;  // warps 4..11 run the final folds and the cluster merge
// tcgen05 variant
constexpr int kUmC = 64;                 // chunk size of the variant
constexpr int kUmM = 64;                 // UMMA M (rows of a K5 block <= 64)
constexpr int kUmMaxCf = 5;              // K (and V) ring depth cap
constexpr int kCfProducerWarp = 1, kIssuerWarp = 2, kPvIssuerWarp = 3, kSoftmaxWarp0 = 4;
constexpr float kRescaleLog2 = 8.f;      // lazy O rescale threshold (P <= 2^8), as chunk_first_umma.cu

template <bool UM>
struct DkRoles {
  static constexpr int NC = UM ? 4 : 8;  // mma.sync consumer warps
  static constexpr int C0 = UM ? 8 : 4;  // first consumer warp
};

// Stage metadata: a unit (flags, valid tokens, rows, head of the set) or a
// PACK of n rows' last chunks (row, valid tokens, first slot row, head), or END.
struct DkMeta {
  int flags, n, nt, row0, nrows, hh;
  int prow[8], pnt[8], poff[8], phh[8], pchunk[8];
};

template <int NC>
CA_DEV void dk_sync_consumers() {  // bar.sync is .aligned: arrive converged
  __syncwarp();
  asm volatile("bar.sync 1, %0;" ::"n"(NC * 32) : "memory");
}
// warps 4..11 (an mbarrier of 8 warp arrivals, phase `ph`)
CA_DEV void dk_sync_merge(uint64_t* bar, uint32_t ph) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive_cta(bar);
  mbar_wait(bar, ph);
}
template <int N>
CA_DEV void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
CA_DEV void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
CA_DEV void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
CA_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// relaxed: the only writes the other ranks rely on are the mbarrier inits,
// published by fence.mbarrier_init.release.cluster (a .release arrive is a
// GPU-scope MEMBAR in SASS, which waits out every thread's entry loads)
CA_DEV void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
CA_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
// bulk copy of `bytes` from this CTA's shared memory to another CTA's (both
// cluster addresses), completing bytes on that CTA's mbarrier
CA_DEV void bulk_s2cluster(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(bar)
               : "memory");
}
CA_DEV uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

// (head, row) state layout in shared memory: [hg][rows][D + 4] fp32 =
// o[0..D), m (log2 units) at D, n at D + 1.
template <int D>
struct RowState {
  static constexpr int kStride = D + 4;
};

// Eqn 2 weights of a state (ms) and a partial (mj) rebased to their common
// max (either may be -inf: an empty side contributes nothing).
CA_DEV void fold_weights(float ms, float mj, float& M, float& ws, float& wj) {
  M = fmaxf(ms, mj);
  ws = ms == -INFINITY ? 0.f : fast_exp2(ms - M);
  wj = mj == -INFINITY ? 0.f : fast_exp2(mj - M);
}

// Shared-memory layout (bytes from the dynamic base): SF ring [nst][stage] |
// states [scap][SR] | (UM) chunk-first states [scap][SR] | recv area | (UM,
// 1024-aligned at run time) K ring [nk][K image] | V ring [nv][V image].
// TMEM (UM, 512 columns): S [2][64] | O [D] | P [2][32] (16-bit pairs) | Q [D / 2].
struct DkLayout {
  int32_t nst, nk, nv, scap;
  int32_t nocst;  // UM: no chunk-first state set (every CTA folds its one job straight into the states)
  uint32_t stage_bytes, cf_off;
  int32_t bulk1d;  // d = 64: K/V tiles by one 1-D bulk copy (the pool tile is already the SWIZZLE_128B image)
  int32_t map3;        // d = 128: the maps are 3-D (one TMA op per tile)
  int32_t diag_empty;  // DIAGNOSTIC ONLY (no output): every CTA returns at entry -- the launch's own cost
  int32_t diag_nosf;   // DIAGNOSTIC ONLY (wrong output): the private-unit producer issues nothing
  int32_t diag_cf;     // DIAGNOSTIC ONLY (wrong output): bit 0 no UMMA issued, bit 1 no softmax math
};

template <typename T, typename TO, int D, int TPW, bool UM>
__global__ void __launch_bounds__(kDkThreads, 1)
    dk_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v, T* kpool,
              T* vpool, const T* __restrict__ q, TO* __restrict__ out, const T* __restrict__ knew,
              const T* __restrict__ vnew, int32_t* __restrict__ len_out, int32_t mode, DevTables t, int32_t h,
              int32_t c, float scale_log2, DkLayout ly, int64_t layer_rows, int32_t cs, int32_t hg,
              uint64_t* __restrict__ trace) {
  using WA = WarpAttn<T, D, TPW>;
  constexpr int NC = DkRoles<UM>::NC, kConsumer0 = DkRoles<UM>::C0;
  constexpr int SR = RowState<D>::kStride;
  constexpr uint32_t kRowBytes = D * sizeof(T);
  // tcgen05 variant geometry (c = 64)
  constexpr int HALVES = D / 64;                             // 128-byte d-halves of a token row
  constexpr uint32_t kCfTile = HALVES * kUmC * 128;          // one K (or V) SWIZZLE_128B image
  constexpr uint32_t kTmemP = 4 * kUmC;                      // P buffers in TMEM: columns 256 + 32 b (16-bit pairs)
  constexpr uint32_t kTmemQ = kTmemP + kUmC;                // Q in TMEM: D / 2 columns after the two P buffers
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[kDkMaxStages], empty_bar[kDkMaxStages];
  __shared__ DkMeta meta[kDkMaxStages];
  __shared__ uint64_t recv_bar[kDkMaxCluster];  // rank r's copies of this rank's merge states have arrived
  __shared__ uint64_t merge_bar;  // warps 4..11 done with their units (phase 0) / the state folds (phase 1)
  // tcgen05 variant: chunk-first ring, MMA / softmax hand-offs
  __shared__ uint64_t k_full[UM ? kUmMaxCf : 1], k_empty[UM ? kUmMaxCf : 1];
  __shared__ uint64_t v_full[UM ? kUmMaxCf : 1], v_empty[UM ? kUmMaxCf : 1];
  __shared__ int4 cf_meta[UM ? kUmMaxCf : 1];  // K slot's unit {flags, row0, rows, head of the set}
  __shared__ int4 s_meta[2];                   // the unit of S buffer b (issuer -> softmax)
  __shared__ uint64_t s_full[2], s_free[2], s_meta_full[2], p_full[2], pv_done[2], q_full, o_ready, o_free, tm_done;
  __shared__ int pv_flags[2];                  // the unit flags of P buffer b (softmax -> P V issuer)
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t sf_done;  // UM: the private-unit consumers are done with the states
  __shared__ int cf_direct;     // UM: the CTA's one chunk-first job was folded straight into the states

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)(blockIdx.x % (unsigned)cs), grp = (int)(blockIdx.x / (unsigned)cs);
  const int hsets = h / hg;
  const int head0 = (grp % hsets) * hg, blk = grp / hsets;
  // the block's rows (schedule.cpp: balanced blocks of ceil(b / blocks) rows,
  // = the dk_block record) -- arithmetic, no dependent load at entry
  const int bper = (t.b + t.dk_blocks - 1) / t.dk_blocks;
  const int brow0 = blk * bper, brows = min(bper, t.b - brow0);
  // CTA record: units [u0, u1), then the descriptors of its first kDkCtaPre units
  const int32_t* crp = t.dk_cta + (size_t)kDkCtaInts * (blk * cs + rank);
  const int4 crec = *reinterpret_cast<const int4*>(crp);
  const int u0 = crec.x, u1 = crec.y, npre = crec.z;
  const int nst = ly.nst, nk = ly.nk, nv = ly.nv;
  const uint32_t stage_bytes = ly.stage_bytes;
  const uint32_t tile_bytes = (uint32_t)c * kRowBytes;
  float* st = reinterpret_cast<float*>(smem_raw + (size_t)nst * stage_bytes);  // (head, row) states
  float* cst = st + (size_t)ly.scap * SR;                 // UM: chunk-first states (same indexing)
  float* recv = (UM && !ly.nocst ? cst : st) + (size_t)ly.scap * SR;  // [owned state][other rank][SR]: pushed by the other ranks
  unsigned char* cfr = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + ly.cf_off + 1023) & ~uintptr_t(1023));  // UM: chunk-first ring
  auto state_row = [&](int hh, int row) { return st + (size_t)(hh * brows + row - brow0) * SR; };
  // mode bit 0: scatter the step's new K/V row into each row's last chunk
  // (K1 folded in); bit 1: the lengths advance by one in this launch (the
  // step's first layer) and the new lengths go to len_out
  const bool append = (mode & 1) != 0, bump = (mode & 2) != 0;
  // debug timeline (option "trace"): kernel_timeline.py layout (kernels.h)
  uint64_t* tr = trace && blockIdx.x < kTraceCtas ? trace + (size_t)blockIdx.x * kTraceStride : nullptr;
  if (tr && tid == 0) tr[0] = globaltimer_ns();
  if (tr && tid == 32) tr[115] = (uint64_t)(npre + 100 * ly.nk + 10000 * ly.nv);  // layout probe (trace only)
  if (ly.diag_empty) return;

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full_bar[s], 1);  // producer: expected bytes per copy, then one arrive with the metadata
      mbar_init(&empty_bar[s], NC);
    }
    for (int r = 0; r < cs; ++r) mbar_init(&recv_bar[r], 1);
    mbar_init(&merge_bar, kMergeThreads / 32);
    if constexpr (UM) {
      for (int s = 0; s < nk; ++s) {
        mbar_init(&k_full[s], 1);   // K producer: arrive + expected bytes
        mbar_init(&k_empty[s], 1);  // commit after the slot's S
      }
      for (int s = 0; s < nv; ++s) {
        mbar_init(&v_full[s], 1);   // V producer: arrive + expected bytes
        mbar_init(&v_empty[s], 1);  // commit after the slot's P V
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&s_meta_full[b], 1);
        mbar_init(&s_full[b], 1);
        mbar_init(&s_free[b], 4);
        mbar_init(&p_full[b], 4);
        mbar_init(&pv_done[b], 1);
      }
      mbar_init(&q_full, 4);
      mbar_init(&o_ready, 1);
      mbar_init(&o_free, 4);
      mbar_init(&tm_done, 1);
      mbar_init(&sf_done, DkRoles<UM>::NC);
      cf_direct = 0;
    }
    fence_barrier_init();
  }
  if constexpr (UM) {
    if (warp == kIssuerWarp) {  // S double buffer (2 x 64 columns) + O (D columns) <= 256
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
  }
  __syncthreads();
  if constexpr (UM) tc_fence_after();
  // cluster barrier phase: every CTA's recv_bar is initialised before any
  // rank pushes into it (waited for just before the pushes, at the end)
  if (cs > 1) cluster_arrive_relaxed();

  if (warp < 4) {
   if constexpr (UM) regs_dec<kRegsLowUm>(); else regs_dec<kRegsLow>();
   if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Stages: a chunk-first unit (mma.sync variant only), a cooperative
    // seq-first unit, or a PACK of up to NC rows' last chunks (16-token slots,
    // one row per consumer warp), packed greedily in unit order; then an END
    // stage.
    int jj = 0, rs = 0;  // stages published; ring slot / phase of the next one
    uint32_t rph = 0;
    int pk_n = 0, pk_q = 0, pk_s = 0;  // open pack: rows, 16-token slots used, its stage
    uint32_t pk_bytes = 0;
    const int pk_cap = c / 16;  // 16-token slots = rows of a PACK (<= NC: c <= 128); staging rows after V
    auto acquire = [&]() {
      if (jj >= nst) mbar_wait(&empty_bar[rs], rph ^ 1u);
      return rs;
    };
    auto publish = [&](int s, uint32_t bytes) {  // metadata written: complete the stage (lane 0)
      if (lane == 0) {
        mbar_arrive1(&full_bar[s]);
        if (!UM && tr && jj < kTraceUnits) {
          tr[3 + 4 * jj] = globaltimer_ns();
          tr[6 + 4 * jj] = bytes;
        }
      }
      __syncwarp();
      ++jj;
      if (++rs == nst) {
        rs = 0;
        rph ^= 1u;
      }
    };
    // A pack's items are assigned in order (stage, 16-token slot, index) and
    // their copies issued by the lanes holding their descriptors, all at once
    // when the pack closes (packs close at the end of a 32-unit batch).
    int my_pack = -1, my_off = 0, my_idx = 0, pk_id = 0;
    auto close_pack = [&](const int4& d, int caller, int nt, int lenv) {
      if (pk_n == 0) return;
      if (my_pack == pk_id) {
        const int hh = d.w >> 8, head = head0 + hh;
        const size_t toff = ((size_t)d.x * h + head) * c * D;
        const uint32_t kv_bytes = (uint32_t)nt * kRowBytes;
        const bool fresh = append && (d.w & DK_TAIL);  // its last token is this step's
        const uint32_t old = fresh ? kv_bytes - kRowBytes : kv_bytes;
        unsigned char* stg = smem_raw + (size_t)pk_s * stage_bytes;
        const uint32_t off = (uint32_t)my_off * kRowBytes;  // 16-token aligned: the tile swizzle holds
        const size_t src = ((size_t)caller * h + head) * D;
        mbar_expect_tx(&full_bar[pk_s], 2 * kv_bytes + kRowBytes);
        if (old) {
          bulk_g2s(stg + off, kpool + toff, old, &full_bar[pk_s]);
          bulk_g2s(stg + tile_bytes + off, vpool + toff, old, &full_bar[pk_s]);
        }
        bulk_g2s(stg + 2 * tile_bytes + my_idx * kRowBytes, q + src, kRowBytes, &full_bar[pk_s]);
        if (fresh) {  // the new K / V rows, row-major, into the pack's staging rows
          unsigned char* nrow = stg + 2 * tile_bytes + (pk_cap + 2 * my_idx) * kRowBytes;
          bulk_g2s(nrow, knew + src, kRowBytes, &full_bar[pk_s]);
          bulk_g2s(nrow + kRowBytes, vnew + src, kRowBytes, &full_bar[pk_s]);
        }
        if (bump && head == 0) len_out[d.y] = lenv;  // the lengths of the next launch
        meta[pk_s].prow[my_idx] = d.y;
        meta[pk_s].pnt[my_idx] = nt;
        meta[pk_s].poff[my_idx] = my_off;
        meta[pk_s].phh[my_idx] = hh;
        meta[pk_s].pchunk[my_idx] = d.x;
      }
      __syncwarp();
      if (lane == 0) {
        meta[pk_s].flags = DK_PACK;
        meta[pk_s].n = pk_n;
      }
      publish(pk_s, pk_bytes);
      pk_n = pk_q = 0;
      pk_bytes = 0;
      ++pk_id;
    };
    // a chunk-first or cooperative seq-first unit into the next stage
    auto issue_unit = [&](int i_chunk, int i_row0, int i_nrows, int i_flags, int i_hh, int i_caller, int i_nt) {
      const int head = head0 + i_hh;
      const size_t toff = ((size_t)i_chunk * h + head) * c * D;
      const uint32_t kv_bytes = (uint32_t)i_nt * kRowBytes;
      const int s = acquire();
      const bool want_q = (i_flags & DK_PRIV) && (i_flags & DK_FIRST);
      if (lane == 0) {
        unsigned char* stg = smem_raw + (size_t)s * stage_bytes;
        mbar_expect_tx(&full_bar[s], 2 * kv_bytes + (want_q ? kRowBytes : 0u));
        bulk_g2s(stg, kpool + toff, kv_bytes, &full_bar[s]);
        bulk_g2s(stg + tile_bytes, vpool + toff, kv_bytes, &full_bar[s]);
        if (want_q) bulk_g2s(stg + 2 * tile_bytes, q + ((size_t)i_caller * h + head) * D, kRowBytes, &full_bar[s]);
        meta[s].flags = i_flags;
        meta[s].nt = i_nt;
        meta[s].row0 = i_row0;
        meta[s].nrows = i_nrows;
        meta[s].hh = i_hh;
      }
      publish(s, 2 * kv_bytes);
    };
    pdl_wait();  // the pool, q and the lengths may come from the previous kernel (PDL)
    // the leading chunk-first units straight from the CTA record (one
    // dependent load less before the first copy); the tcgen05 variant's
    // chunk-first units belong to the TMA producer (warp 1)
    int upre = u0;
    for (int k = 0; k < npre; ++k) {
      const int4 dd = *reinterpret_cast<const int4*>(crp + 4 + 4 * k);
      if (dd.w & DK_PRIV) break;
      if constexpr (!UM) issue_unit(dd.x, dd.y, dd.z, dd.w & 0xff, dd.w >> 8, 0, c);
      ++upre;
    }
    for (int base = ly.diag_nosf ? u1 : upre; base < u1; base += 32) {
      const int u = base + lane;
      int4 d = make_int4(-1, 0, 0, 0);  // {chunk, row0, rows, flags | hh << 8}
      int caller = 0, nt = c, lenv = 0;
      if (u < u1) d = *reinterpret_cast<const int4*>(t.dk_unit + 4 * (size_t)u);
      // dependent loads of private units (caller row, length): consumed only
      // when their unit comes up, so chunk-first units issue without waiting
      if (u < u1) {
        if (d.w & DK_PRIV) caller = t.row_caller[d.y];
        if (d.w & DK_TAIL) {  // the row's last chunk
          lenv = t.seq_len[d.y] + (bump ? 1 : 0);
          nt = lenv - t.last_start[d.y];
        }
      }
      const int cnt = min(32, u1 - base);
      for (int i = 0; i < cnt; ++i) {
        const int i_chunk = __shfl_sync(0xffffffffu, d.x, i);
        const int i_row0 = __shfl_sync(0xffffffffu, d.y, i);
        const int i_nrows = __shfl_sync(0xffffffffu, d.z, i);
        const int i_word = __shfl_sync(0xffffffffu, d.w, i);
        const int i_flags = i_word & 0xff, i_hh = i_word >> 8;
        if (UM && !(i_flags & DK_PRIV)) continue;  // warp 1's
        int i_caller = 0, i_nt = c;
        if (i_flags & DK_PRIV) {  // warp-uniform
          i_caller = __shfl_sync(0xffffffffu, caller, i);
          i_nt = __shfl_sync(0xffffffffu, nt, i);
        }
        const uint32_t kv_bytes = (uint32_t)i_nt * kRowBytes;
        if (i_flags & DK_PACK) {
          const int slots = (i_nt + 15) >> 4;
          if (pk_n > 0 && (pk_q + slots > pk_cap || pk_n == NC)) close_pack(d, caller, nt, lenv);
          if (pk_n == 0) pk_s = acquire();
          if (lane == i) {
            my_pack = pk_id;
            my_off = pk_q * 16;
            my_idx = pk_n;
          }
          ++pk_n;
          pk_q += slots;
          pk_bytes += 2 * kv_bytes + kRowBytes;
          continue;
        }
        close_pack(d, caller, nt, lenv);
        issue_unit(i_chunk, i_row0, i_nrows, i_flags, i_hh, i_caller, i_nt);
      }
      close_pack(d, caller, nt, lenv);  // packs do not straddle batches (descriptors live in lanes)
    }
    const int s = acquire();
    if (lane == 0) meta[s].flags = DK_END;
    publish(s, 0);
   } else if (UM && warp == kCfProducerWarp) {
    // ----------------------------------- chunk-first TMA producer (K, V)
    // The CTA's chunk-first units (they precede its private ones): per unit
    // its K tile into the K ring (released after S) and its V tile into the V
    // ring (released after P V) -- one 3-D TMA box per tile at d = 128 (2-D
    // boxes of 64 elements x 64 rows per d-half otherwise): the pool rows are
    // XOR pre-swizzled within each 128-byte half, so the boxes land as
    // canonical SWIZZLE_128B atoms.  No chunk-first unit: an END stage.
    if (lane == 0) {
      prefetch_tmap(&tmap_k);
      prefetch_tmap(&tmap_v);
    }
    pdl_wait();
    int k = 0;
    bool done = false;
    auto load_tile = [&](const CUtensorMap* map, T* pool, unsigned char* stg, uint64_t* bar, int chunk, int hh) {
      mbar_arrive_expect_tx(bar, kCfTile);
      const int y = (int)(layer_rows + ((int64_t)chunk * h + head0 + hh) * kUmC);
      if (HALVES == 2 && ly.map3)
        tma_load_3d(stg, map, 0, y, 0, bar);
      else if (HALVES == 1 && ly.bulk1d)
        bulk_g2s(stg, pool + ((size_t)chunk * h + head0 + hh) * kUmC * D, kCfTile, bar);
      else
#pragma unroll
        for (int hf = 0; hf < HALVES; ++hf) tma_load_2d(stg + hf * kUmC * 128, map, hf * 64, y, bar);
    };
    // the first npre units come from the CTA record (loaded at entry), the
    // rest in batches of 32 descriptors, one per lane
    for (int base = u0, first = 1; base < u1 && !done; base += first ? npre : 32, first = 0) {
      if (first && npre == 0) continue;
      const int u = base + lane;
      int4 d = make_int4(-1, 0, 0, DK_PRIV);
      if (first) {
        if (lane < npre) d = *reinterpret_cast<const int4*>(crp + 4 + 4 * lane);
      } else if (u < u1) {
        d = *reinterpret_cast<const int4*>(t.dk_unit + 4 * (size_t)u);
      }
      const int cnt = first ? npre : min(32, u1 - base);
      for (int i = 0; i < cnt; ++i, ++k) {
        const int i_chunk = __shfl_sync(0xffffffffu, d.x, i);
        const int i_row0 = __shfl_sync(0xffffffffu, d.y, i);
        const int i_nrows = __shfl_sync(0xffffffffu, d.z, i);
        const int i_word = __shfl_sync(0xffffffffu, d.w, i);
        if (i_word & DK_PRIV) {
          done = true;
          break;
        }
        const int sk = k % nk, sv = k % nv;
        if (k >= nk) mbar_wait(&k_empty[sk], (uint32_t)(((k / nk) - 1) & 1));
        if (lane == 0) {
          cf_meta[sk] = make_int4(i_word & 0xff, i_row0, i_nrows, i_word >> 8);
          if (tr && k < 16) {  // tcgen05 variant: the timeline traces the chunk-first units
            tr[3 + 4 * k] = globaltimer_ns();
            tr[6 + 4 * k] = 2 * kCfTile;
          }
          load_tile(&tmap_k, kpool, cfr + (size_t)sk * kCfTile, &k_full[sk], i_chunk, i_word >> 8);
        }
        __syncwarp();
        if (k >= nv) mbar_wait(&v_empty[sv], (uint32_t)(((k / nv) - 1) & 1));
        if (lane == 0) {
          if (tr && k < 14) tr[102 + k] = globaltimer_ns();  // V tile k issued
          load_tile(&tmap_v, vpool, cfr + (size_t)(nk + sv) * kCfTile, &v_full[sv], i_chunk, i_word >> 8);
        }
        __syncwarp();
      }
    }
    if (k == 0) {  // no chunk-first unit: an END stage (else the last unit carries DK_FINAL)
      if (lane == 0) {
        cf_meta[0] = make_int4(DK_END, 0, 0, 0);
        mbar_arrive_cta(&k_full[0]);
      }
      __syncwarp();
    }
   } else if (UM && warp == kIssuerWarp) {
    // --------------------------------------------------------- S issuer
    // chunk k: S_{k&1} = Q K_k^T (M = 64, N = 64, K = d; A = Q from TMEM, its
    // K slot released when S completes).  The chunk's metadata goes to the
    // softmax warps through s_meta[k&1] (s_meta_full).  P V runs on its own
    // issuer (warp 3), so S of the next chunks is never held up behind it.
    const uint32_t tmem = tmem_base;
    constexpr uint32_t idS = umma_idesc<T, kUmM>(kUmC, false);
    const uint32_t ka0 = smem_u32(cfr);
    int jobs_q = 0;
    for (int k = 0;; ++k) {
      const int s = k % nk, b = k & 1;
      mbar_wait(&k_full[s], (uint32_t)((k / nk) & 1));
      if (tr && lane == 0 && k < 16) tr[70 + k] = globaltimer_ns();  // K tile k in shared memory (issuer view)
      const int4 mk = cf_meta[s];
      if (k >= 2) mbar_wait(&s_free[b], (uint32_t)(((k >> 1) - 1) & 1));  // S_b and s_meta[b] consumed
      if (lane == 0) {
        s_meta[b] = mk;
        mbar_arrive_cta(&s_meta_full[b]);
      }
      if (mk.x & DK_END) break;
      if (mk.x & DK_FIRST) {
        mbar_wait(&q_full, (uint32_t)(jobs_q & 1));
        ++jobs_q;
      }
      tc_fence_after();
      if (lane == 0) {
        if (tr && k == 3) tr[116] = globaltimer_ns();
        const uint64_t dk = umma_sdesc(ka0 + s * kCfTile, 16, 1024);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {  // S = Q K^T over d
          if (ly.diag_cf & 9) break;
          const uint32_t o = (ks % 4) * 32;
          // A = Q from TMEM (8 columns = 16 elements of d per step), B = K tile
          umma_f16_ta(tmem + b * kUmC, tmem + kTmemQ + (uint32_t)(ks * 8), dk + (uint64_t)(((ks / 4) * kUmC * 128 + o) >> 4),
                      idS, ks > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[b]);
        umma_commit(&k_empty[s]);
        if (tr && k == 3) tr[117] = globaltimer_ns();
        if (tr && k == 0) tr[kTraceStride - 10] = globaltimer_ns();  // first S issued
      }
      __syncwarp();
      if (mk.x & DK_FINAL) break;  // the CTA's last chunk-first unit
    }
    // TMEM is released once the P V issuer reports every job's O read
    mbar_wait(&tm_done, 0);
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
   } else if (UM && warp == kPvIssuerWarp) {
    // -------------------------------------------------------- P V issuer
    // chunk k: O += P_{k&1} V_k (A = P from TMEM, 8 columns = 16 tokens per
    // step; B = V MN-major from the V ring), once the softmax has published
    // P_k (and the chunk's flags) and, at a job's first chunk, read the
    // previous job's O.
    const uint32_t tmem = tmem_base;
    constexpr uint32_t idO = umma_idesc<T, kUmM>(D, true);
    const uint32_t va0 = smem_u32(cfr) + nk * kCfTile;
    int jobs_done = 0;
    for (int k = 0;; ++k) {
      const int b = k & 1, sv = k % nv;
      mbar_wait(&p_full[b], (uint32_t)((k >> 1) & 1));
      const int fj = pv_flags[b];
      if (fj & DK_END) break;
      if (tr && lane == 0 && k < 16) tr[86 + k] = globaltimer_ns();  // P_k in (issuer view)
      mbar_wait(&v_full[sv], (uint32_t)((k / nv) & 1));
      if ((fj & DK_FIRST) && jobs_done > 0) mbar_wait(&o_free, (uint32_t)((jobs_done - 1) & 1));
      tc_fence_after();
      if (lane == 0) {
        const uint64_t db = umma_sdesc(va0 + sv * kCfTile, kUmC * 128, 1024);
        const uint32_t tp = tmem + kTmemP + (uint32_t)(b * (kUmC / 2));
#pragma unroll
        for (int ks = 0; ks < kUmC / 16; ++ks)
          if (!(ly.diag_cf & 5))
            umma_f16_ta(tmem + 2 * kUmC, tp + (uint32_t)(ks * 8), db + (uint64_t)(ks * 16 * 128 >> 4), idO,
                        (!(fj & DK_FIRST) || ks > 0) ? 1u : 0u);
        umma_commit(&pv_done[b]);
        umma_commit(&v_empty[sv]);
        if (fj & DK_LAST) umma_commit(&o_ready);
      }
      __syncwarp();
      if (fj & DK_LAST) ++jobs_done;
      if (fj & DK_FINAL) break;
    }
    if (jobs_done > 0) mbar_wait(&o_free, (uint32_t)((jobs_done - 1) & 1));
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&tm_done);
   }
   if (cs > 1) {
     cluster_wait();            // the cluster barrier phase begun at entry
     cluster_arrive_relaxed();  // phase 2 (the merge warps arrive once their copies are in)
   }
  } else {
    // merge-phase constants, loaded now (the row's caller index is a cold load)
    const int nstate = hg * brows;
    const int mw = warp - kMergeWarp0;
    const int mw0 = rank + cs * mw;
    const int mcaller = mw0 < nstate ? t.row_caller[brow0 + mw0 % brows] : 0;
    if (UM && warp < kSoftmaxWarp0 + 4) {
      regs_inc<kRegsSoftmax>();
      // ------------------------------------------------ softmax (tcgen05)
      // Warp qd reads TMEM lane quadrant qd = M rows 16 qd .. 16 qd + 15 of
      // the M = 64 tile (M row 16 q + i sits in lane 32 q + i) in the
      // .16x256b shape: thread t holds M rows m0 = 16 qd + t / 4 and m0 + 8,
      // columns 8 j + 2 (t % 4) + {0, 1} -- a quad shares a row (max / sum by
      // two shuffles).  Jobs of <= 32 rows are placed 8 per quadrant (job row
      // j at M row 16 (j / 8) + j % 8: all four warps -- all four SM
      // sub-partitions' exp units -- work, on the m0 rows only); larger jobs
      // fill M rows 0..63 in order.  Per chunk: S from TMEM, online softmax
      // with the lazy O rescale, P (16-bit, SWIZZLE_128B) to shared memory;
      // per job: O from TMEM folded into the (head, row) chunk-first states
      // (Eqn 2).
      const int qd = warp - kSoftmaxWarp0;  // TMEM lane quadrant
      const int m0 = qd * 16 + (lane >> 2), c0 = 2 * (lane & 3);
      const uint32_t tmem = tmem_base;
      const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
      const uint32_t tO = tmem + 2 * kUmC;
      const int sct = tid - kSoftmaxWarp0 * 32;
      // job row of M row m (-1: unused row)
      auto job_row = [&](int m, int nrows) {
        const int j = nrows > 32 ? m : ((m & 15) < 8 ? (m >> 4) * 8 + (m & 7) : -1);
        return j < nrows ? j : -1;
      };
      // Q of a job's rows into TMEM, the A operand of S (unused M rows zero):
      // thread t provides, for M rows m0 and m0 + 8, the packed pairs of d =
      // 8 j + 2 (t % 4), + 1 -- the .16x128b store shape puts them at column
      // 4 j + t % 4 of the rows' lanes, the A layout.  The previous job's S
      // MMAs (the only readers) completed before its last S_full.
      constexpr int QJ = D / 8;
      uint32_t qv[2 * QJ];
      // speculative: the CTA's first job usually spans the whole block, so the
      // caller indices of this thread's Q rows are loaded at entry
      const int js0 = job_row(m0, brows), js1 = job_row(m0 + 8, brows);
      const int cs0 = js0 < 0 ? 0 : t.row_identity ? brow0 + js0 : t.row_caller[brow0 + js0];
      const int cs1 = js1 < 0 ? 0 : t.row_identity ? brow0 + js1 : t.row_caller[brow0 + js1];
      auto load_q = [&](int row0, int nrows, int hh) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int j = job_row(m0 + 8 * hf, nrows);
          const int caller = j < 0                                  ? 0
                             : (row0 == brow0 && nrows == brows) ? (hf ? cs1 : cs0)
                             : t.row_identity                    ? row0 + j
                                                                 : t.row_caller[row0 + j];
          const uint32_t* qrow =
              j >= 0 ? reinterpret_cast<const uint32_t*>(q + ((size_t)caller * h + head0 + hh) * D) : nullptr;
#pragma unroll
          for (int jj = 0; jj < QJ; ++jj) qv[2 * jj + hf] = qrow ? qrow[4 * jj + (lane & 3)] : 0u;
        }
      };
      auto store_q = [&]() {
        if constexpr (QJ == 16)
          tmem_st16x128_x16(tmem + kTmemQ + lane_base, qv);
        else
          tmem_st16x128_x8(tmem + kTmemQ + lane_base, qv);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(&q_full);
      };
      pdl_wait();  // q comes from the previous kernel
      // the CTA's first job from its record: its Q loads are in flight while
      // the chunk-first states are initialised and the first K/V tiles load
      load_q(brow0, brows, 0);  // speculative: the whole block, head 0 of the set (the usual first job)
      bool qpre = false;
      if (npre > 0) {
        const int4 d0 = *reinterpret_cast<const int4*>(crp + 4);
        if (!(d0.w & DK_PRIV)) {
          if (d0.y != brow0 || d0.z != brows || (d0.w >> 8) != 0) load_q(d0.y, d0.z, d0.w >> 8);
          qpre = true;
        }
      }
      if (!ly.nocst) {
#pragma unroll 1
        for (int i = sct; i < hg * brows * SR; i += 128) cst[i] = (i % SR) == D ? -INFINITY : 0.f;
      }
      asm volatile("bar.sync 3, 128;" ::: "memory");  // chunk-first states initialised
      if (qpre) {
        store_q();
        if (tr && sct == 0) tr[kTraceStride - 6] = globaltimer_ns();  // first Q in TMEM
      }
      float m_ref[2] = {-INFINITY, -INFINITY}, n[2] = {0.f, 0.f};  // M rows m0, m0 + 8 (n: this thread's columns)
      int crow0 = 0, cnrows = 0, chh = 0, jobs = 0, nh = 2;
      for (int k = 0;; ++k) {
        const int b = k & 1;
        mbar_wait(&s_meta_full[b], (uint32_t)((k >> 1) & 1));
        const int4 mt = s_meta[b];
        if (mt.x & DK_END) {  // no chunk-first unit: tell the P V issuer
          if (lane == 0) {
            if (qd == 0) pv_flags[b] = DK_END;
            mbar_arrive_cta(&p_full[b]);
          }
          break;
        }
        if (mt.x & DK_FIRST) {
          crow0 = mt.y;
          cnrows = mt.z;
          chh = mt.w;
          nh = cnrows > 32 ? 2 : 1;  // M row halves holding job rows (warp-uniform)
          if (!qpre) {
            load_q(crow0, cnrows, chh);
            store_q();
          }
          qpre = false;
          m_ref[0] = m_ref[1] = -INFINITY;
          n[0] = n[1] = 0.f;
        }
        mbar_wait(&s_full[b], (uint32_t)((k >> 1) & 1));
        tc_fence_after();
        if (tr && sct == 0 && k < 16) tr[4 + 4 * k] = globaltimer_ns();
        uint32_t u[32];  // rep j: S[m0][8j + c0 + 0/1] = u[4j], u[4j + 1]; S[m0 + 8][...] = u[4j + 2], u[4j + 3]
        tmem_ld16x256_x8(tmem + b * kUmC + lane_base, u);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(&s_free[b]);
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          if (hf >= nh) break;
          float a0 = __uint_as_float(u[2 * hf]), a1 = __uint_as_float(u[2 * hf + 1]);
#pragma unroll
          for (int j = 1; j < 8; ++j) {
            a0 = fmaxf(a0, __uint_as_float(u[4 * j + 2 * hf]));
            a1 = fmaxf(a1, __uint_as_float(u[4 * j + 2 * hf + 1]));
          }
          float m = fmaxf(a0, a1);
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
          mx[hf] = m * scale_log2;  // scale > 0: the max commutes with it
        }
        // lazy rescale: a new reference max only when a row's max grew by more than 2^8
        const bool need0 = mx[0] > m_ref[0] + kRescaleLog2, need1 = mx[1] > m_ref[1] + kRescaleLog2;
        if (__any_sync(0xffffffffu, need0 || need1)) {
          float f[2];
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            const bool nd = hf ? need1 : need0;
            const float m_new = nd ? mx[hf] : m_ref[hf];
            f[hf] = (nd && m_ref[hf] != -INFINITY) ? fast_exp2(m_ref[hf] - m_new) : 1.f;
            n[hf] *= f[hf];
            m_ref[hf] = m_new;
          }
          if (!(mt.x & DK_FIRST)) {  // O holds this job's chunks so far: wait for the last P V, scale in TMEM
            mbar_wait(&pv_done[(k - 1) & 1], (uint32_t)(((k - 1) >> 1) & 1));
            tc_fence_after();
#pragma unroll 1
            for (int cb = 0; cb < D; cb += 64) {
              uint32_t o[32];
              tmem_ld16x256_x8(tO + lane_base + cb, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f[(i >> 1) & 1]);
              tmem_st16x256_x8(tO + lane_base + cb, o);
            }
            tmem_wait_st();
            tc_fence_before();
          }
        }
        // P = exp2(s - m_ref) rounded to T (n from the rounded P, reading A11)
        if (k >= 2) mbar_wait(&pv_done[b], (uint32_t)(((k >> 1) - 1) & 1));  // P V_{k-2} read this buffer
        // P -> TMEM (the A operand of P V): the .16x128b shape puts this
        // thread's packed pair (row m0 (+8), tokens 8j + c0, +1) at column
        // 4j + t % 4 of its row's lane -- exactly the A layout
        uint32_t pw[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pw[i] = 0u;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          if (hf >= nh || (ly.diag_cf & 2)) break;
          float ns0 = 0.f, ns1 = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t w = Mma<T>::pack(fast_exp2(fmaf(__uint_as_float(u[4 * j + 2 * hf]), scale_log2, -m_ref[hf])),
                                            fast_exp2(fmaf(__uint_as_float(u[4 * j + 2 * hf + 1]), scale_log2, -m_ref[hf])));
            const float2 f2 = Mma<T>::unpack(w);
            if (j & 1) ns1 += f2.x + f2.y; else ns0 += f2.x + f2.y;
            pw[2 * j + hf] = w;
          }
          n[hf] += ns0 + ns1;
        }
        tmem_st16x128_x8(tmem + kTmemP + (uint32_t)(b * (kUmC / 2)) + lane_base, pw);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (qd == 0) pv_flags[b] = mt.x;
          mbar_arrive_cta(&p_full[b]);
        }
        if (tr && sct == 0 && k < 16) tr[5 + 4 * k] = globaltimer_ns();
        if (mt.x & DK_LAST) {
          // job end: O from TMEM folded into the (head, row) chunk-first states
          float nr[2];
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            nr[hf] = n[hf] + __shfl_xor_sync(0xffffffffu, n[hf], 1);
            nr[hf] += __shfl_xor_sync(0xffffffffu, nr[hf], 2);
          }
          // the CTA's only job: straight into the (head, row) states once the
          // private-unit consumers are done with them (the same arithmetic as
          // folding the chunk-first state in at the end: Eqn 2 of two partials)
          const bool direct = (mt.x & DK_SOLO) != 0;
          if (direct) mbar_wait(&sf_done, 0);
          mbar_wait(&o_ready, (uint32_t)(jobs & 1));
          tc_fence_after();
          float* srow[2];
          float ws[2], wj[2], Mn[2];
          bool ok[2];
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            const int j = hf < nh ? job_row(m0 + 8 * hf, cnrows) : -1;
            ok[hf] = j >= 0;
            srow[hf] = (direct ? st : cst) + (size_t)(chh * brows + (ok[hf] ? crow0 + j : brow0) - brow0) * SR;
            ws[hf] = wj[hf] = Mn[hf] = 0.f;
            if (ok[hf]) fold_weights(srow[hf][D], m_ref[hf], Mn[hf], ws[hf], wj[hf]);
          }
          if (direct && sct == 0) cf_direct = 1;
#pragma unroll 1
          for (int cb = 0; cb < D; cb += 64) {
            uint32_t o[32];
            tmem_ld16x256_x8(tO + lane_base + cb, o);
            tmem_wait_ld();
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              if (!ok[hf]) continue;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                float2* p = reinterpret_cast<float2*>(srow[hf] + cb + 8 * j + c0);
                const float2 x = *p;
                *p = make_float2(fmaf(wj[hf], __uint_as_float(o[4 * j + 2 * hf]), x.x * ws[hf]),
                                 fmaf(wj[hf], __uint_as_float(o[4 * j + 2 * hf + 1]), x.y * ws[hf]));
              }
            }
          }
          __syncwarp();  // the quad read m, n before they change
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
            if (ok[hf] && (lane & 3) == 0) {
              srow[hf][D + 1] = fmaf(wj[hf], nr[hf], srow[hf][D + 1] * ws[hf]);
              srow[hf][D] = Mn[hf];
            }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cta(&o_free);
          ++jobs;
          if (tr && sct == 0) tr[kTraceStride - 7] = globaltimer_ns();  // job epilogue done
        }
        if (mt.x & DK_FINAL) break;  // the CTA's last chunk-first unit
      }
    } else {
    // ----------------------------------------------------------- consumers
    if constexpr (UM) regs_inc<kRegsConsumerUm>(); else regs_inc<kRegsHigh>();
    const int ct = tid - kConsumer0 * 32, cw = warp - kConsumer0;
#pragma unroll 1
    for (int i = ct; i < hg * brows * SR; i += NC * 32) st[i] = (i % SR) == D ? -INFINITY : 0.f;
    pdl_wait();  // q comes from the previous kernel
    dk_sync_consumers<NC>();  // states initialised
    WA wa;
    uint32_t qa[WA::KS][4];
    auto q_row0 = [&](const unsigned char* qrow) {  // the query in row 0 of the MMA tile (lanes 0..3)
      const uint32_t* q32 = reinterpret_cast<const uint32_t*>(qrow);
#pragma unroll
      for (int ks = 0; ks < WA::KS; ++ks) {
        qa[ks][0] = lane < 4 ? q32[ks * 8 + lane] : 0u;
        qa[ks][2] = lane < 4 ? q32[ks * 8 + 4 + lane] : 0u;
        qa[ks][1] = qa[ks][3] = 0u;
      }
    };
    // chunk-first job geometry (begin_cf): warp (g, l), G row groups x L lanes
    int cfL = 1, cfg = 0, cfl = 0, crow0 = 0, crows = 0, chh = 0, c_altm = 0, c_sel = 0, c_span = c, c_tb = 0;
    bool cact = false;
    auto begin_cf = [&](int row0, int nrows, int hh) {
      crow0 = row0;
      crows = nrows;
      chh = hh;
      int g = 1;
      while (g * 16 < nrows) g *= 2;
      cfL = NC / g;
      cfg = cw / cfL;
      cfl = cw % cfL;
      cact = cfg * 16 < crows;
      int nsl = cfL;  // token slices per chunk: divides cfL and c / 16, >= kDkSlice tokens each
      while (nsl > 1 && (nsl * kDkSlice > c || (c / 16) % nsl != 0)) nsl >>= 1;
      c_altm = cfL / nsl - 1;  // lane l takes slice l % nsl of every alt-th chunk (k % alt == l / nsl)
      c_sel = cfl / nsl;
      c_span = c / nsl;
      c_tb = (cfl % nsl) * c_span;
      wa.reset();
      const int head = head0 + hh;
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
    // row-0 state (lanes 0..3) of this warp folded into (hh, row)'s state (Eqn 2)
    auto fold_row0 = [&](int hh, int row) {
      if (lane < 4) {
        float* srow = state_row(hh, row);
        const float ms = srow[D], ns = srow[D + 1];
        float M, ws, wj;
        fold_weights(ms, wa.m_lo, M, ws, wj);
#pragma unroll
        for (int i = 0; i < WA::DT; ++i) {
          float2* p = reinterpret_cast<float2*>(srow + i * 8 + lane * 2);
          const float2 o = *p;
          *p = make_float2(fmaf(wj, wa.o[i][0], o.x * ws), fmaf(wj, wa.o[i][1], o.y * ws));
        }
        __syncwarp(0xfu);  // the quad read ms before lane 0 rewrites it
        if (lane == 0) {
          srow[D] = M;
          srow[D + 1] = fmaf(wj, wa.n_lo, ns * ws);
        }
      }
      __syncwarp();
    };
    int kk = 0;  // chunk index inside the current chunk-first job (lane selection)
    int kp = 0;  // chunk index inside the current cooperative seq-first job (team selection)
    // the CTA's first job, if chunk-first: its Q fragments (global loads)
    // overlap the first K/V copies
    bool pre = false;
    if constexpr (!UM) {
      if (npre > 0) {
        const int4 d0 = *reinterpret_cast<const int4*>(crp + 4);
        if (!(d0.w & DK_PRIV)) {
          begin_cf(d0.y, d0.z, d0.w >> 8);
          pre = true;
        }
      }
    }
    int jj = 0, rs = 0;
    uint32_t rph = 0;
    for (;; ++jj) {
      const int s = rs;
      mbar_wait(&full_bar[s], rph);
      if (!UM && tr && ct == 0 && jj < kTraceUnits) tr[4 + 4 * jj] = globaltimer_ns();
      const int flags = meta[s].flags;
      if (flags & DK_END) break;
      const unsigned char* stg = smem_raw + (size_t)s * stage_bytes;
      const uint32_t k_u32 = smem_u32(stg), v_u32 = k_u32 + tile_bytes;
      if (flags & DK_PACK) {
        // ---- seq-first PACK (Alg 2): warp w = the whole last chunk of row w
        if (cw < meta[s].n) {
          const int row = meta[s].prow[cw], ntw = meta[s].pnt[cw], hh = meta[s].phh[cw];
          const uint32_t off = (uint32_t)meta[s].poff[cw] * kRowBytes;
          q_row0(stg + 2 * tile_bytes + cw * kRowBytes);
          // the step's new token (append): its K / V rows are read from the
          // pack's staging rows, not the tile
          const unsigned char* nrow = stg + 2 * tile_bytes + (c / 16 + 2 * cw) * kRowBytes;
          const int sp = append ? ntw - 1 : -1;
          const uint32_t sp_k = smem_u32(nrow), sp_v = sp_k + kRowBytes;
          wa.reset();
          for (int t0 = 0; t0 < ntw; t0 += 16)
            wa.template chunk<true, 16>(qa, k_u32 + off, v_u32 + off, t0, ntw, scale_log2, lane, 0, 0, sp, sp_k, sp_v);
          wa.finish();
          fold_row0(hh, row);
          if (append) {
            // K1: the new K / V row into its pool slot for the next steps
            // (16-byte groups XOR-swizzled by slot % 8; lanes 0-15 K, 16-31 V)
            constexpr int V16 = kRowBytes / 16, E16 = 16 / sizeof(T);
            const int x = lane & 15, slot = ntw - 1;
            if (x < V16) {
              const size_t pofs = ((size_t)meta[s].pchunk[cw] * h + head0 + hh) * c * D + (size_t)slot * D;
              T* to = (lane < 16 ? kpool : vpool) + pofs + (size_t)swz_chunk(slot, x) * E16;
              *reinterpret_cast<uint4*>(to) = *reinterpret_cast<const uint4*>(nrow + (lane < 16 ? 0u : kRowBytes) + x * 16);
            }
          }
        }
      } else if (flags & DK_PRIV) {
        // ---- cooperative seq-first unit (Alg 2): one row; NC / 4 teams of
        // four warps take alternate chunks of the job, warp (team, w) = token
        // slice w
        constexpr int kTeams = NC / 4;
        const int nt = meta[s].nt;
        if (flags & DK_FIRST) {
          wa.reset();
          q_row0(stg + 2 * tile_bytes);
          kp = 0;
        }
        const int team = cw >> 2, tw = cw & 3;
        if ((kp % kTeams) == team && tw * TPW < nt) wa.template chunk<true>(qa, k_u32, v_u32, tw * TPW, nt, scale_log2, lane);
        ++kp;
        if (flags & DK_LAST) {
          // fold the warps' row-0 states into the row's state, warp order
          // (scratch: this stage's K tile -- every warp is done reading it)
          wa.finish();
          float* pw = reinterpret_cast<float*>(const_cast<unsigned char*>(stg));
          dk_sync_consumers<NC>();
          if (lane < 4) {
            if (lane == 0) {
              pw[cw * SR + D] = wa.m_lo;
              pw[cw * SR + D + 1] = wa.n_lo;
            }
#pragma unroll
            for (int i = 0; i < WA::DT; ++i)
              *reinterpret_cast<float2*>(&pw[cw * SR + i * 8 + lane * 2]) = make_float2(wa.o[i][0], wa.o[i][1]);
          }
          dk_sync_consumers<NC>();
          float* srow = state_row(meta[s].hh, meta[s].row0);
          const float ms = srow[D], ns = srow[D + 1];
          float M = ms;
#pragma unroll
          for (int w = 0; w < NC; ++w) M = fmaxf(M, pw[w * SR + D]);
          if (M != -INFINITY) {
            float wgt[NC];
            const float wsf = ms == -INFINITY ? 0.f : fast_exp2(ms - M);
#pragma unroll
            for (int w = 0; w < NC; ++w) {
              const float mw = pw[w * SR + D];
              wgt[w] = mw == -INFINITY ? 0.f : fast_exp2(mw - M);
            }
            for (int x = ct; x < D; x += NC * 32) {
              float a = srow[x] * wsf;
#pragma unroll
              for (int w = 0; w < NC; ++w) a = fmaf(wgt[w], pw[w * SR + x], a);
              srow[x] = a;
            }
            dk_sync_consumers<NC>();  // every thread read ms before it changes
            if (ct == 0) {
              float nn = ns * wsf;
#pragma unroll
              for (int w = 0; w < NC; ++w) nn = fmaf(wgt[w], pw[w * SR + D + 1], nn);
              srow[D] = M;
              srow[D + 1] = nn;
            }
          }
          fence_proxy_async();  // generic writes to the stage before its next bulk copy
          dk_sync_consumers<NC>();  // scratch / row state reuse
        }
      } else if constexpr (!UM) {
        // ---- chunk-first unit (Alg 1): rows [row0, row0 + nrows) of a shared run
        if (flags & DK_FIRST) {
          if (!pre) begin_cf(meta[s].row0, meta[s].nrows, meta[s].hh);
          pre = false;
          kk = 0;
        }
        if (cact && (kk & c_altm) == c_sel) {
          int t0 = c_tb;
          for (; t0 + 32 <= c_tb + c_span; t0 += 32) wa.template chunk<false, 32>(qa, k_u32, v_u32, t0, c, scale_log2, lane);
          for (; t0 < c_tb + c_span; t0 += 16) wa.template chunk<false, 16>(qa, k_u32, v_u32, t0, c, scale_log2, lane);
        }
        ++kk;
        if (flags & DK_LAST) {
          // fold lane l's 16-row partial into the rows' states, lanes in order
          wa.finish();
          for (int l = 0; l < cfL; ++l) {
            dk_sync_consumers<NC>();
            if (cfl == l && cact) {
              const int rl = lane >> 2, cq = (lane & 3) * 2;
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                const int rloc = cfg * 16 + rl + 8 * hf;
                const bool ok = rloc < crows;
                float* srow = state_row(chh, crow0 + (ok ? rloc : 0));
                const float mj = hf ? wa.m_hi : wa.m_lo, nj = hf ? wa.n_hi : wa.n_lo;
                const float ms = ok ? srow[D] : -INFINITY;
                float M, ws, wj;
                fold_weights(ms, mj, M, ws, wj);
                if (ok) {
#pragma unroll
                  for (int i = 0; i < WA::DT; ++i) {
                    float2* p = reinterpret_cast<float2*>(srow + i * 8 + cq);
                    const float2 o = *p;
                    *p = make_float2(fmaf(wj, wa.o[i][2 * hf], o.x * ws), fmaf(wj, wa.o[i][2 * hf + 1], o.y * ws));
                  }
                }
                __syncwarp();  // the quad read ms before lane cq == 0 rewrites it
                if (ok && (lane & 3) == 0) {
                  const float ns = srow[D + 1];
                  srow[D] = M;
                  srow[D + 1] = fmaf(wj, nj, ns * ws);
                }
              }
            }
          }
          dk_sync_consumers<NC>();
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive1(&empty_bar[s]);
      if (!UM && tr && ct == 0 && jj < kTraceUnits) tr[5 + 4 * jj] = globaltimer_ns();
      if (++rs == nst) {
        rs = 0;
        rph ^= 1u;
      }
    }
    if constexpr (UM) {  // the states are the chunk-first epilogue's now
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&sf_done);
    }
    }
    // ------------------------------------------- cluster merge (Eqn 2), O / n
    // Warps 4..11.  (tcgen05 variant: first every chunk-first state is folded
    // into its seq-first state, state i by warp i % 8, chunk-first first.)
    // State i is merged by rank i % cs (merge warp (i / cs) % 8): every
    // other rank pushes its copy of state i into the owner's recv area with
    // st.async (bytes completing on the owner's recv_bar), the owner merges
    // the cs copies in rank order.  No barrier after the pushes; a cluster of
    // one merges nothing.
    constexpr int CPL = D / 32;  // columns per lane (4 for d = 128, 2 for d = 64)
    constexpr int Q4 = SR / 4;   // float4 per state
    const int mth = tid - kMergeWarp0 * 32;
    if (tr && tid == kConsumer0 * 32) tr[1] = globaltimer_ns();  // consumers done with their units
    fence_proxy_async();  // the states' generic writes before the bulk copies read them
    dk_sync_merge(&merge_bar, 0);
    if (tr && tid == kConsumer0 * 32) tr[kTraceStride - 9] = globaltimer_ns();  // merge warps synced  // every warp's last fold is in the states
    if (UM && !cf_direct && !ly.nocst) {
#pragma unroll 1
      for (int i = mw; i < nstate; i += kMergeThreads / 32) {
        float* a = st + (size_t)i * SR;
        const float* b = cst + (size_t)i * SR;
        float M, wa_, wb;
        fold_weights(b[D], a[D], M, wb, wa_);
#pragma unroll
        for (int e = 0; e < CPL; ++e) a[lane * CPL + e] = fmaf(wa_, a[lane * CPL + e], wb * b[lane * CPL + e]);
        __syncwarp();
        if (lane == 0) {
          a[D + 1] = fmaf(wa_, a[D + 1], wb * b[D + 1]);
          a[D] = M;
        }
      }
      fence_proxy_async();
      dk_sync_merge(&merge_bar, 1);
    }
    if (tr && tid == kConsumer0 * 32) tr[kTraceStride - 3] = globaltimer_ns();  // all consumer warps done
    if (cs > 1) {
      cluster_wait();  // the other ranks' recv_bar are initialised
      if (tr && tid == kConsumer0 * 32) tr[kTraceStride - 4] = globaltimer_ns();
      const uint32_t rbase = smem_u32(recv), rbar = smem_u32(&recv_bar[rank]);
      // one bulk shared -> shared copy per state owned by another rank
#pragma unroll 1
      for (int i = mth; i < nstate; i += kMergeThreads) {
        const int grp_i = i / cs, owner = i - grp_i * cs;
        if (owner == rank) continue;
        const int slot = grp_i * (cs - 1) + (rank < owner ? rank : rank - 1);
        bulk_s2cluster(mapa(rbase + (uint32_t)(slot * SR) * 4u, (uint32_t)owner), smem_u32(st + (size_t)i * SR),
                       (uint32_t)(SR * 4), mapa(rbar, (uint32_t)owner));
      }
      if (tr && tid == kConsumer0 * 32) tr[kTraceStride - 5] = globaltimer_ns();  // pushes issued
      if (mth < cs && mth != rank) {  // each other rank's share of copies completes its own barrier
        const int owned = (nstate - rank + cs - 1) / cs;
        mbar_arrive_expect_tx(&recv_bar[mth], (uint32_t)(owned * SR * 4));
      }
    }
    if (tr && tid == kConsumer0 * 32) tr[kTraceStride - 1] = globaltimer_ns();  // merge start (pushes issued)
    // Eqn 2 folds in rank order, each copy as soon as its rank's pushes have
    // landed: after the last arrival only one fold and O / n remain
#pragma unroll 1
    for (int i = mw0; i < nstate; i += cs * (kMergeThreads / 32)) {
      const float* rcv = recv + (size_t)(i / cs) * (cs - 1) * SR;  // the other ranks' copies, rank order
      float acc[CPL], M = -INFINITY, nsum = 0.f;
#pragma unroll
      for (int e = 0; e < CPL; ++e) acc[e] = 0.f;
#pragma unroll 1
      for (int j = 0; j < cs; ++j) {
        const float* r;
        if (j == rank) {
          r = st + (size_t)i * SR;
        } else {
          mbar_wait(&recv_bar[j], 0);
          r = rcv + (size_t)(j < rank ? j : j - 1) * SR;
        }
        const float2 mn = *reinterpret_cast<const float2*>(r + D);
        float Mn, wa, wj;
        fold_weights(M, mn.x, Mn, wa, wj);
        nsum = fmaf(wj, mn.y, nsum * wa);
#pragma unroll
        for (int e = 0; e < CPL; ++e) acc[e] = fmaf(wj, r[lane * CPL + e], acc[e] * wa);
        M = Mn;
      }
      if (tr && tid == kConsumer0 * 32 && i == mw0) tr[kTraceStride - 8] = globaltimer_ns() + (M > 1e30f);
      const int hh = i / brows, row = brow0 + i % brows;
      const float inv = 1.f / nsum;
      const int caller = i == mw0 ? mcaller : t.row_caller[row];
      TO* orow = out + ((size_t)caller * h + head0 + hh) * D + lane * CPL;
      if constexpr (std::is_same<TO, float>::value) {
        if constexpr (CPL == 4)
          *reinterpret_cast<float4*>(orow) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
        else
          *reinterpret_cast<float2*>(orow) = make_float2(acc[0] * inv, acc[1] * inv);
      } else {
        if constexpr (CPL == 4)
          *reinterpret_cast<uint2*>(orow) =
              make_uint2(Mma<TO>::pack(acc[0] * inv, acc[1] * inv), Mma<TO>::pack(acc[2] * inv, acc[3] * inv));
        else
          *reinterpret_cast<uint32_t*>(orow) = Mma<TO>::pack(acc[0] * inv, acc[1] * inv);
      }
    }
    if (tr && tid == kConsumer0 * 32) tr[kTraceStride - 2] = globaltimer_ns();  // merge loop done (rank's states written)
    if (cs > 1) {
      // every copy of ours landed once every rank's recv completed: phase 2
      // of the cluster barrier (waited for at the end) keeps the sources alive
      for (int r = 0; r < cs; ++r)
        if (r != rank) mbar_wait(&recv_bar[r], 0);
      cluster_arrive_relaxed();
    }
  }
  // no CTA leaves while another rank's bulk copy may still read its states
  if (cs > 1) cluster_wait();
  if (tr && tid == 0) tr[2] = globaltimer_ns();
}

template <typename T, typename TO, int D, int TPW>
const void* dk_kernel_ptr() {
  return (const void*)dk_kernel<T, TO, D, TPW, false>;
}

template <typename T, typename TO, int D>
const void* dk_kernel_tpw(int tpw) {
  return tpw == 16 ? dk_kernel_ptr<T, TO, D, 16>() : dk_kernel_ptr<T, TO, D, 32>();
}

template <typename T, typename TO>
const void* dk_kernel_d(int d, int tpw) {
  return d == 128 ? dk_kernel_tpw<T, TO, 128>(tpw) : dk_kernel_tpw<T, TO, 64>(tpw);
}

template <typename T>
const void* dk_kernel_out(int out_dtype, int d, int tpw) {
  if (out_dtype == DT_F32) return dk_kernel_d<T, float>(d, tpw);
  if (out_dtype == DT_F16) return dk_kernel_d<T, __half>(d, tpw);
  return dk_kernel_d<T, __nv_bfloat16>(d, tpw);
}

const void* dk_kernel_for(const PoolGeom& p, int out_dtype) {
  const int tpw = sf_mma_tpw(p.dtype, p.c, true);
  return p.dtype == DT_F16 ? dk_kernel_out<__half>(out_dtype, p.d, tpw)
                           : dk_kernel_out<__nv_bfloat16>(out_dtype, p.d, tpw);
}

// the kernel's shared-memory size, and (once) the non-portable cluster opt-in
cudaError_t dk_prepare(const void* kern, size_t smem) {
  cudaError_t e = set_smem_once(kern, smem);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, bool> done;
  int dev = 0;
  e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({kern, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) done[{kern, dev}] = true;
  return e;
}

size_t state_bytes(int32_t d, int32_t n) { return (size_t)n * (d + 4) * 4; }

// Shared-memory layout of a launch (kernel comment "DkLayout") and its size;
// nk = 0 when the tcgen05 variant does not fit.
DkLayout dk_layout(int32_t dtype, int32_t c, int32_t d, int32_t nstate, int32_t cs, bool um, size_t* smem,
                   int max_slots = 0, int vslots = 0, int sf_stages = 0, bool nocst = false) {
  DkLayout L{};
  L.stage_bytes = (uint32_t)dk_stage_bytes(dtype, c, d);
  if (!um) {
    const size_t recv = dk_recv_bytes(d, nstate, cs);
    L.scap = kStateRows;
    L.nst = dk_stages(dtype, c, d, recv);
    *smem = dk_smem_bytes(dtype, c, d, recv);
    return L;
  }
  L.scap = nstate;
  const size_t tile = (size_t)(d / 64) * kUmC * 128;  // Q and P live in TMEM
  const size_t recv = dk_recv_bytes(d, nstate, cs);
  L.nocst = nocst ? 1 : 0;
  const size_t fixed = (nocst ? 1 : 2) * state_bytes(d, nstate) + recv + 1024 + L.stage_bytes;
  *smem = 0;
  if (fixed + 4 * tile > kDkSmemBudget) return L;
  // a second private-unit stage when 6 K/V slots still fit (the packs of the
  // rows' last chunks then load together instead of one after the other)
  L.nst = sf_stages > 0 ? sf_stages : (fixed + L.stage_bytes + 6 * tile <= kDkSmemBudget ? 2 : 1);
  if (fixed + (L.nst - 1) * L.stage_bytes + 4 * tile > kDkSmemBudget) L.nst = 1;
  int slots = (int)std::min<size_t>(2 * kUmMaxCf, (kDkSmemBudget - fixed - (L.nst - 1) * L.stage_bytes) / tile);
  if (max_slots >= 4) slots = std::min(slots, max_slots);
  L.nv = vslots > 0 ? std::min(vslots, slots - 2) : std::min(3, slots / 2);  // V slots wait for P V: K slots come free sooner
  L.nk = std::min(kUmMaxCf, slots - L.nv);
  L.cf_off = (uint32_t)(L.nst * L.stage_bytes + (nocst ? 1 : 2) * state_bytes(d, nstate) + recv);
  *smem = L.cf_off + 1024 + (L.nk + L.nv) * tile;
  return L;
}

template <typename T, typename TO, int D, int TPW>
cudaError_t launch_dk_t(const AttnLaunch& a, const DevTables& t, const DkAppend& ap, cudaStream_t st) {
  const PoolGeom& p = a.pool;
  const int cs = t.dk_cs;
  bool um = t.dk_um != 0 && dk_umma_supported(p);
  size_t smem = 0;
  DkLayout ly = dk_layout(p.dtype, p.c, D, t.dk_hg * t.dk_max_rows, cs, um, &smem, a.dk_slots & 63, (a.dk_slots >> 15) & 7,
                          (a.dk_slots >> 18) & 3, t.dk_all_solo != 0 && !(a.dk_slots & (1 << 20)));
  if (um && ly.nk < 2) {
    um = false;
    ly = dk_layout(p.dtype, p.c, D, t.dk_hg * t.dk_max_rows, cs, false, &smem);
  }
  ly.bulk1d = (a.dk_slots & 64) ? 0 : 1;
  ly.diag_empty = (a.dk_slots & 128) ? 1 : 0;
  ly.diag_nosf = (a.dk_slots & 256) ? 1 : 0;
  ly.diag_cf = ((a.dk_slots >> 9) & 3) | ((a.dk_slots >> 9) & 12);  // +2048: no P.V UMMA, +4096: no S UMMA
  CUtensorMap mk{}, mv{};
  ly.map3 = 0;
  if (um) {
    if (D == 128 && !(a.dk_slots & 16384) && pool_maps3(p, kUmC, &mk, &mv))
      ly.map3 = 1;
    else if (!pool_maps(p, D, kUmC, &mk, &mv))
      return cudaErrorNotSupported;
  }
  auto kern = um ? dk_kernel<T, TO, D, TPW, true> : dk_kernel<T, TO, D, TPW, false>;
  cudaError_t e = dk_prepare((const void*)kern, kDkSmemBudget);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(t.dk_groups * cs));
  cfg.blockDim = dim3(kDkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = (unsigned)cs;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (a.use_pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  T* kp = (T*)p.k + (size_t)a.layer * p.layer_stride;
  T* vp = (T*)p.v + (size_t)a.layer * p.layer_stride;
  const int64_t layer_rows = (int64_t)a.layer * p.max_chunks * p.h * p.c;
  return cudaLaunchKernelEx(&cfg, kern, mk, mv, kp, vp, (const T*)a.q, (TO*)a.out, (const T*)ap.k, (const T*)ap.v,
                            ap.len_out, (int32_t)ap.mode, t, (int32_t)p.h, (int32_t)p.c, a.scale_log2, ly, layer_rows,
                            (int32_t)cs, (int32_t)t.dk_hg, a.trace);
}

template <typename T, typename TO, int D>
cudaError_t dk_tpw(const AttnLaunch& a, const DevTables& t, const DkAppend& ap, cudaStream_t st) {
  switch (sf_mma_tpw(a.pool.dtype, a.pool.c, true)) {
    case 16: return launch_dk_t<T, TO, D, 16>(a, t, ap, st);
    case 32: return launch_dk_t<T, TO, D, 32>(a, t, ap, st);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T>
cudaError_t dk_dispatch(const AttnLaunch& a, const DevTables& t, const DkAppend& ap, cudaStream_t st) {
  const int d = a.pool.d;
#define CA_CASE(DD, TO) \
  if (d == DD) return dk_tpw<T, TO, DD>(a, t, ap, st);
  if (a.out_dtype == DT_F32) {
    CA_CASE(64, float) CA_CASE(128, float)
  } else if (a.out_dtype == DT_F16) {
    CA_CASE(64, __half) CA_CASE(128, __half)
  } else {
    CA_CASE(64, __nv_bfloat16) CA_CASE(128, __nv_bfloat16)
  }
#undef CA_CASE
  return cudaErrorInvalidValue;
}

}  // namespace

size_t dk_stage_bytes(int32_t dtype, int32_t c, int32_t d) {
  const size_t e = (size_t)dtype_bytes(dtype);
  const size_t pk = (size_t)std::min(8, std::max(1, c / 16));  // rows of one PACK
  // K tile | V tile | pk q rows | pk new (K, V) row pairs (PACK)
  return ((size_t)2 * c * d * e + 3 * pk * d * e + 127) / 128 * 128;
}

size_t dk_state_bytes(int32_t d) { return (size_t)kStateRows * (d + 4) * 4; }

size_t dk_recv_bytes(int32_t d, int32_t nstate, int32_t cs) {
  return cs <= 1 ? 0 : (size_t)((nstate + cs - 1) / cs) * (cs - 1) * (d + 4) * 4;
}

int dk_stages(int32_t dtype, int32_t c, int32_t d, size_t recv) {
  const size_t budget = kDkSmemBudget - dk_state_bytes(d) - recv;
  return (int)std::min<size_t>(kDkMaxStages, budget / dk_stage_bytes(dtype, c, d));
}

size_t dk_smem_bytes(int32_t dtype, int32_t c, int32_t d, size_t recv) {
  return (size_t)dk_stages(dtype, c, d, recv) * dk_stage_bytes(dtype, c, d) + dk_state_bytes(d) + recv;
}

int dk_consumer_warps() { return DkRoles<false>::NC; }

bool dk_supported(const PoolGeom& p) {
  if (p.dtype == DT_F32 || (p.d != 64 && p.d != 128)) return false;
  const int tpw = sf_mma_tpw(p.dtype, p.c, true);
  if (tpw != 16 && tpw != 32) return false;  // c in {16, 32, 48, 64, 96, 128}
  if (p.c % 16 != 0 || p.c / tpw > DkRoles<false>::NC) return false;
  return dk_stages(p.dtype, p.c, p.d, dk_state_bytes(p.d)) >= 3;  // the largest recv area
}

bool dk_umma_supported(const PoolGeom& p) {
  return dk_supported(p) && (p.dtype == DT_F16 || p.dtype == DT_BF16) && p.c == kUmC && (p.d == 64 || p.d == 128) &&
         sf_mma_tpw(p.dtype, p.c, true) * 4 >= p.c;  // one team of four consumer warps covers a chunk
}

bool dk_um_fits(const PoolGeom& p, int nstate, int cs) {
  if (!dk_umma_supported(p)) return false;
  size_t smem = 0;
  return dk_layout(p.dtype, p.c, p.d, nstate, cs, true, &smem).nk >= 2;
}

cudaError_t launch_decode(const AttnLaunch& a, const DevTables& t, const DkAppend& ap, cudaStream_t st) {
  if (t.b == 0 || t.dk_groups == 0) return cudaSuccess;
  switch (a.pool.dtype) {
    case DT_F16: return dk_dispatch<__half>(a, t, ap, st);
    case DT_BF16: return dk_dispatch<__nv_bfloat16>(a, t, ap, st);
    default: return cudaErrorInvalidValue;
  }
}

int dk_max_active_clusters(const PoolGeom& p, int out_dtype, int cs) {
  if (!dk_supported(p)) return 0;
  const void* kern = dk_kernel_for(p, out_dtype);
  const size_t smem = dk_smem_bytes(p.dtype, p.c, p.d, dk_recv_bytes(p.d, kDkMaxRows, cs));
  if (dk_prepare(kern, kDkSmemBudget) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(cs * 64));
  cfg.blockDim = dim3(kDkThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace pakv
