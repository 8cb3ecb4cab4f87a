// C ABI of the ChunkAttention decode library (include/chunkattn.h).
//
// Host side of PAPER.md §3.3: the prefix tree is kept in CPU
// memory, the context (C, i, j) + private lists is generated on the CPU and
// copied to the GPU only when the tree structure changed ("lazy context copy",
// triggers: chunk full, sequence joins, sequence leaves), through a pinned,
// double-buffered staging area and one cudaMemcpyAsync on the caller's stream.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <exception>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/chunkattn.h"
#include "host/schedule.h"
#include "host/tree.h"
#include "kernels/kernels.h"

using namespace pakv;

namespace {

thread_local std::string g_last_error;

chunkattn_status fail(chunkattn_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct WsLayout {
  size_t attend_perm, append_row, tables, pO, segO, counters, prefill, trace, total;
  int64_t table_cap, slot_cap, seg_cap, pf_cap;
};

bool valid_config(const chunkattn_config* c, std::string* why) {
  if (!c) return (*why = "null config", false);
  if (c->num_heads < 1 || c->num_layers < 1) return (*why = "num_heads and num_layers must be >= 1", false);
  if (c->head_dim != 64 && c->head_dim != 128) return (*why = "head_dim must be 64 or 128", false);
  if (c->chunk_size < 1 || c->chunk_size > 256) return (*why = "chunk_size must be in [1, 256]", false);
  if (c->dtype < 0 || c->dtype > 2 || c->out_dtype < 0 || c->out_dtype > 2) return (*why = "bad dtype", false);
  if (c->share_threshold < 2) return (*why = "share_threshold must be >= 2", false);
  if (c->max_chunks < 1 || c->max_chunks > (1LL << 31) - 1) return (*why = "bad max_chunks", false);
  if (c->max_batch < 1 || c->max_batch > (1LL << 24)) return (*why = "bad max_batch", false);
  if (c->max_seq_len < 1 || c->max_seq_len > (1LL << 30)) return (*why = "bad max_seq_len", false);
  if ((int64_t)c->num_layers * c->max_chunks * c->num_heads * c->chunk_size > (1LL << 31) - 1)
    return (*why = "pool too large for 32-bit row coordinates", false);
  // the persistent seq-first kernel double-buffers (chunk, head) K/V tiles in
  // shared memory: two stages must fit the per-CTA opt-in limit
  if (seq_first_min_smem(c->dtype, c->chunk_size, c->head_dim) > kMaxSmemPerCta)
    return (*why = "chunk_size x head_dim too large for this dtype (two K/V tile stages exceed 227 KB of shared "
                   "memory; f32 needs chunk_size * head_dim <= 8192, 16-bit <= 16384)",
            false);
  return true;
}

WsLayout ws_layout(const chunkattn_config* c) {
  WsLayout w{};
  const int64_t B = c->max_batch;
  const int64_t msc = (c->max_seq_len + c->chunk_size - 1) / c->chunk_size;
  w.slot_cap = B * msc;
  const int64_t sfcap = B * msc;
  w.table_cap = 4 * (B + 4) + 2 * (B + 5) + (sfcap + 4) + (w.slot_cap + 4) + (c->max_chunks + 4) +
                kCfTileInts * (w.slot_cap + 1) + kSfCtaInts * kMaxSfCtas + 4 +
                (int64_t)kSfItemInts * B * c->num_heads + 4 +
                (int64_t)kSfUnitInts * c->num_heads * B * (msc + 1) + 4 +
                (w.slot_cap + 4) +                                      // mg_tile
                (int64_t)kCfUnitInts * c->num_heads * w.slot_cap + 4 +  // fused chunk-first units
                (B + 4) +                                                   // second length buffer (K5)
                (int64_t)kDkUnitInts * (std::max<int64_t>(B, kDkMaxRows) * msc + 4) +  // K5 units
                (int64_t)(kDkCtaInts * kDkMaxCluster + kDkBlockInts) * (B / kDkMaxRows + 2) + 8;
  size_t o = 0;
  w.attend_perm = o;
  o = align_up(o + 4 * B, 256);
  w.append_row = o;
  o = align_up(o + 4 * B, 256);
  w.tables = o;
  o = align_up(o + 4 * w.table_cap, 256);
  // chunk-first partials [slot][h][d + 4] fp32: o[0..d), m (log2 units) at d, n at d+1
  w.pO = o;
  o = align_up(o + (size_t)4 * w.slot_cap * c->num_heads * (c->head_dim + 4), 256);
  // seq-first segment partials (items merged by their last contributor: split
  // items, and in the fused kernel items with chunk-first partials), same row
  // format; <= one per item plus one extra per CTA boundary
  w.seg_cap = B * c->num_heads + 2 * kMaxSfCtas;
  w.segO = o;
  o = align_up(o + (size_t)4 * w.seg_cap * (c->head_dim + 4), 256);
  w.counters = o;  // per-item contribution counters [B * h] u32 (zeroed; reset by each merge)
  o = align_up(o + (size_t)4 * B * c->num_heads, 256);
  // prefill tables (chunkattn_prefill_attend): tile records + chunk lists
  w.pf_cap = (int64_t)kPfTileInts * B * ((c->max_seq_len + kPfTileRows - 1) / kPfTileRows + 1) + B * msc + 16;
  w.prefill = o;
  o = align_up(o + (size_t)4 * w.pf_cap, 256);
  w.trace = o;  // debug timeline (option "trace"): the last kTraceCtas*kTraceStride u64 words
  o = align_up(o + (size_t)8 * kTraceCtas * kTraceStride, 256);
  w.total = o;
  return w;
}

}  // namespace

struct chunkattn {
  chunkattn_config cfg{};
  bool host_only = true;
  PrefixTree tree;
  ScheduleOptions sopt;
  Context ctx;
  WsLayout ws{};
  std::string build_err;
  // device
  PoolGeom pool{};
  char* wsp = nullptr;
  bool tma_ok = false;
  bool cf_simt = false;
  bool sf_simt = false;
  // 4-warp chunk-first CTA so a seq-first CTA can share its SM under PDL: off by
  // default -- the co-resident pair faulted intermittently with the SIMT
  // seq-first consumers; costs ~1.5% on cfg2.
  bool cf_small = false;
  bool cf_umma = true;  // tcgen05 chunk-first kernel in the two-kernel path
  // chunk-first units inside the persistent seq-first kernel (one launch per
  // attend; falls back to two kernels when the schedule does not allow it)
  bool fused_opt = true;
  int trace_kernel = 0;    // 1: trace seq-first, 2: trace chunk-first
  int sf_ctas_per_sm = 2;  // persistent seq-first residency (smem budget per CTA)
  int sf_prefetch = 0;     // seq-first L2 prefetch distance (units); measured slower on B200
  int dk_slots = 0;        // K5 tcgen05 variant: cap on K + V ring slots (0 = as many as fit)
  bool perm_identity = false;  // the last attend order equals the DFS row order
  int diag_nocompute = 0;  // DIAGNOSTIC ONLY (wrong outputs): seq-first consumers skip the math
  bool use_pdl = true;
  int num_sms = 148;
  int64_t cf_cpt_forced = 0;
  int dk_opt = 1;             // K5 cluster decode: 0 off, 1 auto (the schedule decides), 2 whenever supported
  int len_parity = 0;         // K5: which of the two device length buffers is current
  int64_t sf_ctas_req = 296;  // requested persistent grid (option sf_ctas / sf_ctas_per_sm)
  int resident_cache = -1;    // occupancy x SMs of the persistent kernel (per residency setting)

  int64_t resident_sf_ctas() {
    if (host_only) return sf_ctas_req;
    if (resident_cache < 0) {
      const int r = seq_first_resident_ctas(pool, cfg.out_dtype, sf_ctas_per_sm, !sf_simt);
      resident_cache = r > 0 ? r : num_sms;  // query failed: one CTA per SM is always resident
    }
    return resident_cache;
  }
  // staging
  int32_t* pinned[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool ev_live[2] = {false, false};
  int next_stage = 0;
  int64_t uploaded_epoch = -1;
  std::vector<int64_t> attend_ids;
  int64_t attend_epoch = -1;
  std::vector<int64_t> append_ids, scratch_ids;
  std::vector<int32_t> append_rows;
  std::vector<AppendItem> append_items;
  int64_t append_epoch = -1;
  // counters
  int64_t n_builds = 0, n_uploads = 0, upload_bytes = 0, n_launches = 0;
  bool failed = false;
  // per-kernel CUDA-event timing ("kernel_events" option)
  enum { K_APPEND = 0, K_CF = 1, K_SF = 2, K_COPY = 3 };
  struct Timed {
    cudaEvent_t a, b;
    int kind;
  };
  bool kernel_events = false;
  std::vector<Timed> timed;
  std::vector<cudaEvent_t> ev_pool;
  double acc_ms[4] = {0, 0, 0, 0};
  int64_t acc_n[4] = {0, 0, 0, 0};

  cudaError_t get_event(cudaEvent_t* e) {
    if (!ev_pool.empty()) {
      *e = ev_pool.back();
      ev_pool.pop_back();
      return cudaSuccess;
    }
    return cudaEventCreate(e);
  }
  cudaError_t flush_times() {
    for (const Timed& t : timed) {
      cudaError_t e = cudaEventSynchronize(t.b);
      if (e != cudaSuccess) return e;
      float ms = 0.f;
      e = cudaEventElapsedTime(&ms, t.a, t.b);
      if (e != cudaSuccess) return e;
      acc_ms[t.kind] += ms;
      acc_n[t.kind] += 1;
      ev_pool.push_back(t.a);
      ev_pool.push_back(t.b);
    }
    timed.clear();
    return cudaSuccess;
  }
  // Launch through f(); when timing, bracket it with events on the same stream.
  template <class F>
  cudaError_t timed_launch(int kind, cudaStream_t st, F f) {
    if (!kernel_events) return f();
    if (timed.size() >= 4096) {
      cudaError_t e = flush_times();
      if (e != cudaSuccess) return e;
    }
    Timed t{nullptr, nullptr, kind};
    cudaError_t e = get_event(&t.a);
    if (e == cudaSuccess) e = get_event(&t.b);
    if (e == cudaSuccess) e = cudaEventRecord(t.a, st);
    if (e != cudaSuccess) return e;
    e = f();
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(t.b, st);
    if (e == cudaSuccess) timed.push_back(t);
    return e;
  }
  ~chunkattn() {
    for (const Timed& t : timed) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
  }

  explicit chunkattn(const chunkattn_config& c)
      : cfg(c), tree(c.chunk_size, c.max_chunks, c.prefix_match != 0) {}

  float scale() const { return cfg.scale > 0.f ? cfg.scale : 1.0f / std::sqrt((float)cfg.head_dim); }

  PoolGeom geom() const {
    PoolGeom g = pool;
    g.h = cfg.num_heads;
    g.c = cfg.chunk_size;
    g.d = cfg.head_dim;
    g.num_layers = cfg.num_layers;
    g.dtype = cfg.dtype;
    return g;
  }
  int32_t* other_len() const {
    int32_t* base = reinterpret_cast<int32_t*>(wsp + ws.tables);
    return base + (len_parity ? ctx.lay.seq_len : ctx.lay.seq_len2);
  }

  // Attend permutation (row -> caller index), uploaded when the ids or the
  // tree changed; validates the ids first.
  chunkattn_status prepare_attend(int64_t n, const int64_t* seq_ids, cudaStream_t st) {
    const bool same = attend_epoch == tree.epoch() && (int64_t)attend_ids.size() == n &&
                      (n == 0 || std::memcmp(attend_ids.data(), seq_ids, n * sizeof(int64_t)) == 0);
    if (!same) {
      for (int64_t i = 0; i < n; ++i)
        if (!tree.find(seq_ids[i])) return fail(CA_ENOSEQ, "unknown seq id " + std::to_string(seq_ids[i]));
    }
    chunkattn_status s = ensure_context(st);
    if (s != CA_OK) return s;
    if (!same) {
      std::vector<int32_t> perm(n, -1);
      for (int64_t i = 0; i < n; ++i) {
        const int32_t r = ctx.row_of.at(seq_ids[i]);
        if (perm[r] >= 0) return fail(CA_ESTATE, "duplicate seq id in attend");
        perm[r] = (int32_t)i;
      }
      if (!host_only) {
        s = upload(wsp + ws.attend_perm, perm.data(), n * 4, st);
        if (s != CA_OK) return s;
      }
      attend_ids.assign(seq_ids, seq_ids + n);
      attend_epoch = ctx.epoch;
      perm_identity = true;  // the caller's order is the DFS row order: kernels may skip the indirection
      for (int64_t r = 0; r < n; ++r) perm_identity = perm_identity && perm[r] == (int32_t)r;
    }
    return CA_OK;
  }

  AttnLaunch attn_launch(int32_t layer, const void* q, void* out) const {
    AttnLaunch a{};
    a.pool = pool;
    a.layer = layer;
    a.q = q;
    a.out = out;
    a.out_dtype = cfg.out_dtype;
    a.pO = reinterpret_cast<float*>(wsp + ws.pO);
    a.segO = reinterpret_cast<float*>(wsp + ws.segO);
    a.counters = reinterpret_cast<uint32_t*>(wsp + ws.counters);
    a.scale_log2 = scale() * 1.4426950408889634f;
    a.cf_tensor_cores = tma_ok && !cf_simt;
    a.sf_tensor_cores = !sf_simt;
    a.cf_small = cf_small;
    a.cf_umma = cf_umma;
    a.trace = trace_kernel ? reinterpret_cast<uint64_t*>(wsp + ws.trace) : nullptr;
    a.trace_cf = trace_kernel == 2;
    a.sf_ctas_per_sm = sf_ctas_per_sm;
    a.sf_prefetch = sf_prefetch | (diag_nocompute ? 256 : 0);
    a.dk_slots = dk_slots;
    a.use_pdl = use_pdl && !kernel_events;
    return a;
  }

  chunkattn_status cuda_fail(cudaError_t e, const char* where) {
    failed = true;
    return fail(CA_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
  }

  chunkattn_status set_device() {
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e == cudaSuccess && cur != cfg.device) e = cudaSetDevice(cfg.device);
    return e == cudaSuccess ? CA_OK : cuda_fail(e, "cudaSetDevice");
  }

  // H2D copy through pinned double-buffered staging (stream ordered).
  chunkattn_status upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return CA_OK;
    const int k = next_stage;
    next_stage ^= 1;
    if (ev_live[k]) {
      cudaError_t e = cudaEventSynchronize(ev[k]);
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
    }
    std::memcpy(pinned[k], src, bytes);
    cudaError_t e = cudaMemcpyAsync(dst, pinned[k], bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync");
    e = cudaEventRecord(ev[k], st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    ev_live[k] = true;
    ++n_uploads;
    upload_bytes += (int64_t)bytes;
    return CA_OK;
  }

  // Rebuild the context if the tree changed; upload it (device mode).
  chunkattn_status ensure_context(cudaStream_t st) {
    if (ctx.epoch == tree.epoch()) return CA_OK;
    sopt.cf_chunks_per_tile = cf_cpt_forced;
    // fused kernel: the MMA seq-first kernel runs the chunk-first units (the
    // SIMT consumers never do), so only shapes that kernel takes
    sopt.fused = fused_opt && !cf_simt && sf_mma_tpw(cfg.dtype, cfg.chunk_size, !sf_simt) != 0;
    // persistent grid: at most one wave (the cross-CTA merges spin on other
    // CTAs' contributions, which must be resident)
    sopt.sf_ctas = std::max<int64_t>(1, std::min<int64_t>(sf_ctas_req, resident_sf_ctas()));
    sopt.dk = dk_opt != 0 && dk_supported(geom());
    sopt.dk_force = dk_opt == 2;
    sopt.dk_umma_ok = sopt.dk && dk_umma_supported(geom());
    Context nc;
    std::string err;
    if (!build_context(tree, sopt, &nc, &err)) return fail(CA_ENOMEM, err);
    // the tcgen05 variant only where its shared-memory layout fits this schedule
    if (nc.dk && nc.dk_um) nc.dk_um = dk_um_fits(geom(), nc.dk_hg * nc.dk_max_rows, nc.dk_cs);
    ctx = std::move(nc);
    ++n_builds;
    if (!host_only) {
      chunkattn_status s = upload(wsp + ws.tables, ctx.blob.data(), ctx.blob.size() * 4, st);
      if (s != CA_OK) return s;
      uploaded_epoch = ctx.epoch;
      len_parity = 0;  // both length buffers now hold the host lengths
    }
    return CA_OK;
  }

  DevTables dev_tables() const {
    DevTables t{};
    const int32_t* base = reinterpret_cast<const int32_t*>(wsp + ws.tables);
    const BlobLayout& L = ctx.lay;
    t.row_caller = reinterpret_cast<const int32_t*>(wsp + ws.attend_perm);
    t.seq_len = const_cast<int32_t*>(base + (len_parity ? L.seq_len2 : L.seq_len));
    t.dk_block = base + L.dk_block;
    t.dk_cta = base + L.dk_cta;
    t.dk_unit = base + L.dk_unit;
    t.dk_cs = ctx.dk_cs;
    t.dk_groups = ctx.dk_groups;
    t.dk_max_rows = ctx.dk_max_rows;
    t.dk_blocks = ctx.dk_blocks;
    t.dk_hg = ctx.dk_hg;
    t.dk_um = ctx.dk_um ? 1 : 0;
    t.row_identity = perm_identity ? 1 : 0;
    t.dk_all_solo = ctx.dk_all_solo ? 1 : 0;
    t.sf_first = base + L.sf_first;
    t.last_chunk = base + L.last_chunk;
    t.last_start = base + L.last_start;
    t.sf_ptr = base + L.sf_ptr;
    t.mg_ptr = base + L.mg_ptr;
    t.sf_chunk = base + L.sf_chunk;
    t.mg_slot = base + L.mg_slot;
    t.cf_chunk = base + L.cf_chunk;
    t.cf_tile = base + L.cf_tile;
    t.b = ctx.b;
    t.n_cf_tiles = ctx.n_cf_tiles;
    t.max_tile_rows = ctx.max_tile_rows;
    t.sf_cta = base + L.sf_cta;
    t.sf_item = base + L.sf_item;
    t.sf_unit = base + L.sf_unit;
    t.mg_tile = base + L.mg_tile;
    t.cf_unit = base + L.cf_unit;
    t.n_cf_units = ctx.n_cf_units;
    t.fused = ctx.fused ? 1 : 0;
    t.n_sf_ctas = ctx.n_sf_ctas;
    return t;
  }
};

namespace {

#define CA_GUARD_BEGIN try {
#define CA_GUARD_END                                              \
  }                                                               \
  catch (const PoolExhausted&) {                                  \
    return fail(CA_ENOMEM, "chunk pool exhausted");               \
  }                                                               \
  catch (const std::bad_alloc&) {                                 \
    return fail(CA_ENOMEM, "host allocation failed");             \
  }                                                               \
  catch (const std::exception& ex) {                              \
    return fail(CA_EINVAL, std::string("internal: ") + ex.what()); \
  }

}  // namespace

extern "C" {

const char* chunkattn_last_error(void) { return g_last_error.c_str(); }

size_t chunkattn_workspace_bytes(const chunkattn_config* cfg) {
  std::string why;
  if (!valid_config(cfg, &why)) return 0;
  return ws_layout(cfg).total;
}

chunkattn_status chunkattn_create(const chunkattn_config* cfg, const chunkattn_buffers* buf, chunkattn_t* out) {
  CA_GUARD_BEGIN
  std::string why;
  if (!out) return fail(CA_EINVAL, "null out");
  *out = nullptr;
  if (!valid_config(cfg, &why)) return fail(CA_EINVAL, why);
  auto* h = new chunkattn(*cfg);
  h->host_only = cfg->device < 0;
  h->ws = ws_layout(cfg);
  h->sopt.share_threshold = cfg->share_threshold;
  h->sopt.num_heads = cfg->num_heads;
  h->sopt.slot_capacity = h->ws.slot_cap;
  h->sopt.table_capacity = h->ws.table_cap;
  h->sopt.seg_capacity = h->ws.seg_cap;
  h->sopt.cf_target_ctas = 148;
  h->sopt.head_dim = cfg->head_dim;
  h->sopt.elem_bytes = (int32_t)dtype_bytes(cfg->dtype);
  if (!h->host_only) {
    if (!buf || !buf->k_pool || !buf->v_pool || !buf->workspace) {
      delete h;
      return fail(CA_EINVAL, "null device buffer");
    }
    if (buf->workspace_bytes < h->ws.total) {
      delete h;
      return fail(CA_EINVAL, "workspace too small: need " + std::to_string(h->ws.total));
    }
    if (((uintptr_t)buf->k_pool | (uintptr_t)buf->v_pool | (uintptr_t)buf->workspace) & 15) {
      delete h;
      return fail(CA_EINVAL, "device buffers must be 16-byte aligned");
    }
    if (h->set_device() != CA_OK) {
      delete h;
      return CA_ECUDA;
    }
    h->wsp = static_cast<char*>(buf->workspace);
    h->pool.k = buf->k_pool;
    h->pool.v = buf->v_pool;
    h->pool.max_chunks = cfg->max_chunks;
    h->pool.layer_stride = cfg->max_chunks * cfg->num_heads * cfg->chunk_size * (int64_t)cfg->head_dim;
    h->pool.h = cfg->num_heads;
    h->pool.c = cfg->chunk_size;
    h->pool.d = cfg->head_dim;
    h->pool.num_layers = cfg->num_layers;
    h->pool.dtype = cfg->dtype;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device) == cudaSuccess && sms > 0)
      h->num_sms = sms;
    h->sopt.cf_target_ctas = h->num_sms;
    h->sf_ctas_req = 2 * h->num_sms;
    h->tma_ok = cf_mma_supported(h->pool);
    if (dk_supported(h->pool))  // co-resident clusters of each size (the K5 cluster-size choice)
      for (int k = 1; k <= kDkMaxCluster; ++k) h->sopt.dk_max_clusters[k] = dk_max_active_clusters(h->pool, cfg->out_dtype, k);
    const size_t pin_bytes = (size_t)4 * (std::max(h->ws.table_cap, h->ws.pf_cap) + 2 * cfg->max_batch + 64);
    for (int k = 0; k < 2; ++k) {
      cudaError_t e = cudaHostAlloc((void**)&h->pinned[k], pin_bytes, cudaHostAllocDefault);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev[k], cudaEventDisableTiming);
      if (e != cudaSuccess) {
        chunkattn_destroy(h);
        return fail(CA_ECUDA, std::string("staging alloc: ") + cudaGetErrorString(e));
      }
    }
  }
  *out = h;
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_destroy(chunkattn_t h) {
  if (!h) return CA_OK;
  for (int k = 0; k < 2; ++k) {
    if (h->ev[k]) {
      cudaEventSynchronize(h->ev[k]);
      cudaEventDestroy(h->ev[k]);
    }
    if (h->pinned[k]) cudaFreeHost(h->pinned[k]);
  }
  delete h;
  return CA_OK;
}

chunkattn_status chunkattn_match_prefix(chunkattn_t h, const int32_t* tokens, int64_t n, int64_t* matched) {
  CA_GUARD_BEGIN
  if (!h || !matched || (n > 0 && !tokens) || n < 0) return fail(CA_EINVAL, "bad argument");
  *matched = (int64_t)h->tree.match(tokens, n).size() * h->cfg.chunk_size;
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_add_sequence(chunkattn_t h, const int32_t* tokens, int64_t n, const void* k,
                                        const void* v, int64_t kv_first_pos, void* stream, int64_t* seq_id,
                                        int64_t* matched) {
  CA_GUARD_BEGIN
  if (!h || !tokens || n < 1 || !seq_id) return fail(CA_EINVAL, "bad argument");
  if (h->failed) return fail(CA_ECUDA, "handle failed on an earlier CUDA error");
  if (n > h->cfg.max_seq_len) return fail(CA_EINVAL, "sequence longer than max_seq_len");
  if (h->tree.live_count() >= h->cfg.max_batch) return fail(CA_ENOMEM, "max_batch live sequences reached");
  const int64_t m = (int64_t)h->tree.match(tokens, n).size() * h->cfg.chunk_size;
  if (kv_first_pos < 0 || kv_first_pos > m) return fail(CA_EINVAL, "kv_first_pos must be in [0, matched]");
  if (!h->host_only && m < n && (!k || !v)) return fail(CA_EINVAL, "null k/v");
  std::vector<int32_t> fresh;
  int64_t mm = 0;
  const int64_t sid = h->tree.add(tokens, n, &fresh, &mm);  // throws PoolExhausted before any change
  if (!h->host_only && !fresh.empty()) {
    if (h->set_device() != CA_OK) return CA_ECUDA;
    const size_t row_bytes = (size_t)h->cfg.num_layers * h->cfg.num_heads * h->cfg.head_dim * dtype_bytes(h->cfg.dtype);
    const size_t skip = (size_t)(mm - kv_first_pos) * row_bytes;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = h->timed_launch(chunkattn::K_COPY, st, [&] {
      return launch_copy_rows(h->pool, fresh.data(), (int32_t)fresh.size(), mm, n - mm,
                              static_cast<const char*>(k) + skip, static_cast<const char*>(v) + skip, st);
    });
    if (e != cudaSuccess) return h->cuda_fail(e, "copy_rows");
    h->n_launches += (n - mm + 256LL * h->cfg.chunk_size - 1) / (256LL * h->cfg.chunk_size);
  }
  *seq_id = sid;
  if (matched) *matched = mm;
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_append_kv(chunkattn_t h, int64_t n, const int64_t* seq_ids, const int32_t* tokens,
                                     const void* k, const void* v, void* stream) {
  CA_GUARD_BEGIN
  if (!h || n < 0 || (n > 0 && (!seq_ids || !tokens))) return fail(CA_EINVAL, "bad argument");
  if (h->failed) return fail(CA_ECUDA, "handle failed on an earlier CUDA error");
  if (n == 0) return CA_OK;
  if (!h->host_only && (!k || !v)) return fail(CA_EINVAL, "null k/v");
  {
    for (int64_t i = 0; i < n; ++i) {
      const Sequence* s = h->tree.find(seq_ids[i]);
      if (!s) return fail(CA_ENOSEQ, "unknown seq id " + std::to_string(seq_ids[i]));
      if (s->len + 1 > h->cfg.max_seq_len) return fail(CA_EINVAL, "sequence would exceed max_seq_len");
    }
    // duplicates: sorted scratch copy (no per-call hashing / allocation)
    h->scratch_ids.assign(seq_ids, seq_ids + n);
    std::sort(h->scratch_ids.begin(), h->scratch_ids.end());
    if (std::adjacent_find(h->scratch_ids.begin(), h->scratch_ids.end()) != h->scratch_ids.end())
      return fail(CA_EINVAL, "duplicate seq id in append");
  }
  const int64_t need = h->tree.append_needs(seq_ids, n);
  if (need > h->tree.pool().available()) return fail(CA_ENOMEM, "chunk pool exhausted");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!h->host_only && h->set_device() != CA_OK) return CA_ECUDA;
  if (need > 0) h->tree.append_grow(seq_ids, n);  // structural: "chunk full" trigger
  chunkattn_status s = h->ensure_context(st);       // tables with pre-step lengths
  if (s != CA_OK) return s;
  if (!h->host_only) {
    // scatter list (row, chunk, slot, new length) travels with the launch
    // parameters: steps that do not change the tree upload no table.
    const bool same = h->append_epoch == h->ctx.epoch && (int64_t)h->append_ids.size() == n &&
                      std::memcmp(h->append_ids.data(), seq_ids, n * sizeof(int64_t)) == 0;
    if (!same) {
      h->append_rows.resize(n);
      for (int64_t i = 0; i < n; ++i) h->append_rows[i] = h->ctx.row_of.at(seq_ids[i]);
      h->append_ids.assign(seq_ids, seq_ids + n);
      h->append_epoch = h->ctx.epoch;
    }
    h->append_items.resize(n);
    for (int64_t i = 0; i < n; ++i) {
      const Sequence* sq = h->tree.find(seq_ids[i]);
      const int32_t chunk = sq->path.back();
      h->append_items[i] = AppendItem{h->append_rows[i], chunk,
                                      (int32_t)(sq->len - h->tree.node(chunk).start_pos), (int32_t)(sq->len + 1)};
    }
    const DevTables t = h->dev_tables();
    cudaError_t e = h->timed_launch(chunkattn::K_APPEND, st, [&] {
      return launch_append_kv(h->pool, t, h->append_items.data(), (int32_t)n, k, v, st);
    });
    if (e != cudaSuccess) return h->cuda_fail(e, "append_kv");
    h->n_launches += (n + kMaxAppendItems - 1) / kMaxAppendItems;
  }
  h->tree.append_tokens(seq_ids, tokens, n);
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_remove_sequence(chunkattn_t h, int64_t seq_id, int64_t* released) {
  CA_GUARD_BEGIN
  if (!h) return fail(CA_EINVAL, "null handle");
  if (!h->tree.find(seq_id)) return fail(CA_ENOSEQ, "unknown seq id " + std::to_string(seq_id));
  const auto rel = h->tree.remove(seq_id);
  if (released) *released = (int64_t)rel.size();
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_prefill_attend(chunkattn_t h, int32_t layer, int64_t n, const int64_t* seq_ids,
                                          const int64_t* first_pos, const void* q, void* out, void* stream) {
  CA_GUARD_BEGIN
  if (!h || n < 0 || (n > 0 && (!seq_ids || !first_pos))) return fail(CA_EINVAL, "bad argument");
  if (h->host_only) return fail(CA_EINVAL, "host-only handle");
  if (h->failed) return fail(CA_ECUDA, "handle failed on an earlier CUDA error");
  if (layer < 0 || layer >= h->cfg.num_layers) return fail(CA_EINVAL, "layer out of range");
  if (!prefill_supported(h->pool)) return fail(CA_EDTYPE, "prefill needs F16/BF16, d in {64, 128}, c % 16 == 0");
  // tiles of <= 64 (mma.sync) or 128 (tcgen05) consecutive query positions; chunk lists in path order
  const bool umma = h->cf_umma && prefill_umma_supported(h->pool);
  const int64_t tile_rows = umma ? kPfTileRowsUmma : kPfTileRows;
  std::vector<int32_t> chunks, tiles;
  int64_t row = 0;
  for (int64_t k = 0; k < n; ++k) {
    const Sequence* sq = h->tree.find(seq_ids[k]);
    if (!sq) return fail(CA_ENOSEQ, "unknown seq id " + std::to_string(seq_ids[k]));
    if (first_pos[k] < 0 || first_pos[k] > sq->len) return fail(CA_EINVAL, "first_pos out of range");
    const int32_t off = (int32_t)chunks.size();
    chunks.insert(chunks.end(), sq->path.begin(), sq->path.end());
    for (int64_t p = first_pos[k]; p < sq->len; p += tile_rows) {
      const int32_t nq = (int32_t)std::min<int64_t>(tile_rows, sq->len - p);
      tiles.insert(tiles.end(), {off, (int32_t)(row + p - first_pos[k]), nq, (int32_t)p, (int32_t)sq->len, 0, 0, 0});
    }
    row += sq->len - first_pos[k];
  }
  if (row > 0 && (!q || !out)) return fail(CA_EINVAL, "null q/out");
  if ((int64_t)(tiles.size() + chunks.size()) > h->ws.pf_cap) return fail(CA_ENOMEM, "prefill tables exceed workspace");
  const int32_t n_tiles = (int32_t)(tiles.size() / kPfTileInts);
  if (n_tiles == 0) return CA_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (h->set_device() != CA_OK) return CA_ECUDA;
  const size_t tb = tiles.size();
  tiles.insert(tiles.end(), chunks.begin(), chunks.end());
  chunkattn_status s = h->upload(h->wsp + h->ws.prefill, tiles.data(), tiles.size() * 4, st);
  if (s != CA_OK) return s;
  PrefillLaunch a{};
  a.pool = h->pool;
  a.layer = layer;
  a.q = q;
  a.out = out;
  a.out_dtype = h->cfg.out_dtype;
  a.tiles = reinterpret_cast<const int32_t*>(h->wsp + h->ws.prefill);
  a.chunks = a.tiles + tb;
  a.n_tiles = n_tiles;
  a.scale_log2 = h->scale() * 1.4426950408889634f;
  cudaError_t e =
      h->timed_launch(chunkattn::K_COPY, st, [&] { return umma ? launch_prefill_umma(a, st) : launch_prefill(a, st); });
  if (e != cudaSuccess) return h->cuda_fail(e, "prefill");
  ++h->n_launches;
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_attend(chunkattn_t h, int32_t layer, int64_t n, const int64_t* seq_ids, const void* q,
                                  void* out, void* stream) {
  CA_GUARD_BEGIN
  if (!h || n < 0 || (n > 0 && !seq_ids)) return fail(CA_EINVAL, "bad argument");
  if (h->failed) return fail(CA_ECUDA, "handle failed on an earlier CUDA error");
  if (layer < 0 || layer >= h->cfg.num_layers) return fail(CA_EINVAL, "layer out of range");
  if (n != h->tree.live_count())
    return fail(CA_ESTATE, "attend needs all " + std::to_string(h->tree.live_count()) + " live sequences");
  if (!h->host_only && n > 0 && (!q || !out)) return fail(CA_EINVAL, "null q/out");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!h->host_only && h->set_device() != CA_OK) return CA_ECUDA;
  chunkattn_status s = h->prepare_attend(n, seq_ids, st);
  if (s != CA_OK) return s;
  if (h->host_only || n == 0) return CA_OK;
  const AttnLaunch a = h->attn_launch(layer, q, out);
  const DevTables t = h->dev_tables();
  cudaError_t e = cudaSuccess;
  if (h->ctx.dk) {  // K5: one cluster launch (attend only: lengths from the current buffer)
    const DkAppend ap{nullptr, nullptr, nullptr, 0};
    e = h->timed_launch(chunkattn::K_SF, st, [&] { return launch_decode(a, t, ap, st); });
    if (e != cudaSuccess) return h->cuda_fail(e, "decode");
    ++h->n_launches;
    return CA_OK;
  }
  if (t.n_cf_tiles > 0 && !t.fused) {
    e = h->timed_launch(chunkattn::K_CF, st, [&] { return launch_chunk_first(a, t, st); });
    if (e != cudaSuccess) return h->cuda_fail(e, "chunk_first");
    ++h->n_launches;
  }
  e = h->timed_launch(chunkattn::K_SF, st, [&] { return launch_seq_first(a, t, st); });
  if (e != cudaSuccess) return h->cuda_fail(e, "seq_first");
  ++h->n_launches;
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_append_attend(chunkattn_t h, int32_t layer, int64_t n, const int64_t* seq_ids,
                                         const int32_t* tokens, const void* k, const void* v, const void* q,
                                         void* out, void* stream) {
  CA_GUARD_BEGIN
  if (!h || n < 0 || (n > 0 && !seq_ids)) return fail(CA_EINVAL, "bad argument");
  if (h->host_only) return fail(CA_EINVAL, "host-only handle");
  if (h->failed) return fail(CA_ECUDA, "handle failed on an earlier CUDA error");
  if (layer < 0 || layer >= h->cfg.num_layers) return fail(CA_EINVAL, "layer out of range");
  if (n != h->tree.live_count())
    return fail(CA_ESTATE, "append_attend needs all " + std::to_string(h->tree.live_count()) + " live sequences");
  if (n == 0) return CA_OK;
  if (!k || !v || !q || !out) return fail(CA_EINVAL, "null k/v/q/out");
  if (layer == 0 && !tokens) return fail(CA_EINVAL, "null tokens");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (h->set_device() != CA_OK) return CA_ECUDA;
  if (layer == 0) {  // the tree grows once per step
    for (int64_t i = 0; i < n; ++i) {
      const Sequence* sq = h->tree.find(seq_ids[i]);
      if (!sq) return fail(CA_ENOSEQ, "unknown seq id " + std::to_string(seq_ids[i]));
      if (sq->len + 1 > h->cfg.max_seq_len) return fail(CA_EINVAL, "sequence would exceed max_seq_len");
    }
    h->scratch_ids.assign(seq_ids, seq_ids + n);
    std::sort(h->scratch_ids.begin(), h->scratch_ids.end());
    if (std::adjacent_find(h->scratch_ids.begin(), h->scratch_ids.end()) != h->scratch_ids.end())
      return fail(CA_EINVAL, "duplicate seq id in append_attend");
    const int64_t need = h->tree.append_needs(seq_ids, n);
    if (need > h->tree.pool().available()) return fail(CA_ENOMEM, "chunk pool exhausted");
    if (need > 0) h->tree.append_grow(seq_ids, n);  // structural: "chunk full" trigger
  }
  chunkattn_status s = h->prepare_attend(n, seq_ids, st);  // tables with pre-step lengths
  if (s != CA_OK) return s;
  const AttnLaunch a = h->attn_launch(layer, q, out);
  const DevTables t = h->dev_tables();
  cudaError_t e = cudaSuccess;
  if (h->ctx.dk) {  // one K5 launch: the scatter of this layer's K/V rows inside the attention kernel
    const DkAppend ap{k, v, h->other_len(), layer == 0 ? 3 : 1};
    e = h->timed_launch(chunkattn::K_SF, st, [&] { return launch_decode(a, t, ap, st); });
    if (e != cudaSuccess) return h->cuda_fail(e, "decode");
    ++h->n_launches;
  } else {
    // the schedule took the persistent kernels (shape without K5, or runs
    // wider than a K5 row block): K1 for this layer, then the attend launches
    h->append_items.resize(n);
    for (int64_t i = 0; i < n; ++i) {
      const Sequence* sq = h->tree.find(seq_ids[i]);
      const int32_t chunk = sq->path.back();
      const int64_t pre = layer == 0 ? sq->len : sq->len - 1;  // the tree advanced at layer 0
      h->append_items[i] = AppendItem{h->ctx.row_of.at(seq_ids[i]), chunk,
                                      (int32_t)(pre - h->tree.node(chunk).start_pos), (int32_t)(pre + 1)};
    }
    PoolGeom g = h->pool;  // this layer's slice, [n][h][d] sources
    g.k = static_cast<char*>(g.k) + (size_t)layer * g.layer_stride * dtype_bytes(g.dtype);
    g.v = static_cast<char*>(g.v) + (size_t)layer * g.layer_stride * dtype_bytes(g.dtype);
    g.num_layers = 1;
    e = h->timed_launch(chunkattn::K_APPEND, st,
                        [&] { return launch_append_kv(g, t, h->append_items.data(), (int32_t)n, k, v, st); });
    if (e != cudaSuccess) return h->cuda_fail(e, "append_kv");
    h->n_launches += (n + kMaxAppendItems - 1) / kMaxAppendItems;
    if (t.n_cf_tiles > 0 && !t.fused) {
      e = h->timed_launch(chunkattn::K_CF, st, [&] { return launch_chunk_first(a, t, st); });
      if (e != cudaSuccess) return h->cuda_fail(e, "chunk_first");
      ++h->n_launches;
    }
    e = h->timed_launch(chunkattn::K_SF, st, [&] { return launch_seq_first(a, t, st); });
    if (e != cudaSuccess) return h->cuda_fail(e, "seq_first");
    ++h->n_launches;
  }
  if (layer == 0) {
    if (h->ctx.dk) h->len_parity ^= 1;  // K5 wrote the advanced lengths to the other buffer
    h->tree.append_tokens(seq_ids, tokens, n);
  }
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_decode_step_host(chunkattn_t h, int32_t layer, int64_t n, const int64_t* seq_ids,
                                            const int32_t* tokens, const void* in_host, void* out_host,
                                            void* staging, size_t staging_bytes, void* stream) {
  CA_GUARD_BEGIN
  if (!h || n < 0 || (n > 0 && (!seq_ids || !tokens))) return fail(CA_EINVAL, "bad argument");
  if (h->host_only) return fail(CA_EINVAL, "host-only handle");
  if (h->failed) return fail(CA_ECUDA, "handle failed on an earlier CUDA error");
  if (n == 0) return CA_OK;
  if (!in_host || !out_host || !staging) return fail(CA_EINVAL, "null buffer");
  if ((uintptr_t)staging & 15) return fail(CA_EINVAL, "staging must be 16-byte aligned");
  const size_t E = dtype_bytes(h->cfg.dtype);
  const size_t q_bytes = (size_t)n * h->cfg.num_heads * h->cfg.head_dim * E;
  const size_t kv_bytes = q_bytes * (size_t)h->cfg.num_layers;
  const size_t in_bytes = q_bytes + 2 * kv_bytes;
  const size_t out_off = (in_bytes + 15) / 16 * 16;
  const size_t out_bytes = (size_t)n * h->cfg.num_heads * h->cfg.head_dim * dtype_bytes(h->cfg.out_dtype);
  if (staging_bytes < out_off + out_bytes) return fail(CA_EINVAL, "staging buffer too small");
  if (h->set_device() != CA_OK) return CA_ECUDA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* dev = static_cast<char*>(staging);
  cudaError_t e = cudaMemcpyAsync(dev, in_host, in_bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return h->cuda_fail(e, "decode_step_host H2D");
  chunkattn_status s;
  if (h->cfg.num_layers == 1) {  // append + attend in one call (one launch on the K5 schedule)
    s = chunkattn_append_attend(h, layer, n, seq_ids, tokens, dev + q_bytes, dev + q_bytes + kv_bytes, dev,
                                dev + out_off, stream);
    if (s != CA_OK) return s;
  } else {
    s = chunkattn_append_kv(h, n, seq_ids, tokens, dev + q_bytes, dev + q_bytes + kv_bytes, stream);
    if (s != CA_OK) return s;
    s = chunkattn_attend(h, layer, n, seq_ids, dev, dev + out_off, stream);
    if (s != CA_OK) return s;
  }
  e = cudaMemcpyAsync(out_host, dev + out_off, out_bytes, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return h->cuda_fail(e, "decode_step_host D2H");
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_batch_order(chunkattn_t h, int64_t* ids, int64_t cap, int64_t* n) {
  CA_GUARD_BEGIN
  if (!h || !n || (cap > 0 && !ids)) return fail(CA_EINVAL, "bad argument");
  std::vector<int64_t> order;
  std::vector<ChunkRec> recs;
  h->tree.dfs(&order, &recs);
  *n = (int64_t)order.size();
  if (cap < *n) return fail(CA_ERANGE, "buffer too small");
  std::copy(order.begin(), order.end(), ids);
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_export_context(chunkattn_t h, char* buf, size_t cap, size_t* len) {
  CA_GUARD_BEGIN
  if (!h || !len) return fail(CA_EINVAL, "bad argument");
  Context x;
  h->tree.dfs(&x.order, &x.recs);
  const std::string s = export_text(h->tree, x, h->cfg.share_threshold);
  *len = s.size();
  if (!buf || cap <= s.size()) return fail(CA_ERANGE, "buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_memory_stats(chunkattn_t h, int64_t out[6]) {
  if (!h || !out) return fail(CA_EINVAL, "bad argument");
  const ChunkPool& p = h->tree.pool();
  out[0] = p.used();
  out[1] = p.free_count();
  out[2] = p.created();
  out[3] = p.hwm();
  out[4] = p.used() * 2 * h->cfg.num_layers * h->cfg.num_heads * (int64_t)h->cfg.chunk_size * h->cfg.head_dim *
           dtype_bytes(h->cfg.dtype);
  out[5] = h->tree.waste_slots();
  return CA_OK;
}

chunkattn_status chunkattn_counters(chunkattn_t h, int64_t out[6]) {
  if (!h || !out) return fail(CA_EINVAL, "bad argument");
  out[0] = h->n_builds;
  out[1] = h->n_uploads;
  out[2] = h->upload_bytes;
  out[3] = h->n_launches;
  out[4] = h->tree.epoch();
  out[5] = h->ctx.n_slots;
  return CA_OK;
}

chunkattn_status chunkattn_schedule_info(chunkattn_t h, int64_t out[9]) {
  if (!h || !out) return fail(CA_EINVAL, "bad argument");
  out[0] = h->ctx.dk ? 1 : 0;
  out[1] = h->ctx.dk_cs;
  out[2] = h->ctx.dk_groups;
  out[3] = h->ctx.dk_blocks;
  out[4] = h->ctx.dk_units;
  out[5] = h->ctx.dk_hg;
  out[6] = h->ctx.fused ? 1 : 0;
  out[7] = h->ctx.n_sf_ctas;
  out[8] = h->ctx.dk && h->ctx.dk_um ? 1 : 0;
  return CA_OK;
}

chunkattn_status chunkattn_set_option(chunkattn_t h, const char* key, int64_t value) {
  if (!h || !key) return fail(CA_EINVAL, "bad argument");
  const std::string k(key);
  if (k == "cf_splits") {
    h->cf_cpt_forced = value < 0 ? 0 : value;
  } else if (k == "cf_target_ctas") {
    h->sopt.cf_target_ctas = value < 1 ? 1 : value;
  } else if (k == "sf_ctas") {  // clamped to one resident wave at the next build
    h->sf_ctas_req = value < 1 ? 1 : std::min<int64_t>(value, kMaxSfCtas);
  } else if (k == "cf_simt") {
    h->cf_simt = value != 0;
  } else if (k == "sf_simt") {
    h->sf_simt = value != 0;
    h->resident_cache = -1;
  } else if (k == "fused") {
    h->fused_opt = value != 0;
  } else if (k == "cf_unit_cost") {
    h->sopt.cf_unit_cost = value < 1 ? 0.1 : (double)value / 10.0;  // tenths of a seq-first unit
  } else if (k == "cf_lane_merge") {
    h->sopt.cf_lane_merge = value != 0;
  } else if (k == "fused_tile_rows") {
    h->sopt.fused_tile_rows = value;
  } else if (k == "sf_unit_fixed") {
    h->sopt.sf_unit_fixed = value < 0 ? 0.0 : std::min<int64_t>(value, 10) / 10.0;  // tenths
  } else if (k == "sf_item_cost") {
    h->sopt.sf_item_cost = value < 0 ? 0.0 : (double)value / 10.0;  // tenths of a unit
  } else if (k == "dk") {
    h->dk_opt = (int)std::max<int64_t>(0, std::min<int64_t>(value, 2));
  } else if (k == "dk_cs") {
    h->sopt.dk_cs_forced = (int32_t)std::max<int64_t>(0, std::min<int64_t>(value, kDkMaxCluster));
  } else if (k == "dk_max_rows") {
    h->sopt.dk_max_rows = (int32_t)std::max<int64_t>(16, std::min<int64_t>(value, kDkMaxRows));
  } else if (k == "dk_shared_fixed") {  // hundredths
    h->sopt.dk_shared_fixed = std::max<int64_t>(0, value) / 100.0;
  } else if (k == "dk_shared_row") {  // thousandths
    h->sopt.dk_shared_row = std::max<int64_t>(0, value) / 1000.0;
  } else if (k == "dk_hg") {
    h->sopt.dk_hg_forced = (int32_t)std::max<int64_t>(0, value);
  } else if (k == "dk_umma") {
    h->sopt.dk_umma = (int32_t)std::max<int64_t>(0, std::min<int64_t>(value, 2));
  } else if (k == "dk_umma_ratio") {  // hundredths
    h->sopt.dk_umma_ratio = std::max<int64_t>(0, value) / 100.0;
  } else if (k == "dk_pack_fixed") {  // hundredths
    h->sopt.dk_pack_fixed = std::min<int64_t>(100, std::max<int64_t>(0, value)) / 100.0;
  } else if (k == "cf_umma") {
    h->cf_umma = value != 0;
  } else if (k == "cf_small") {
    h->cf_small = value != 0;
  } else if (k == "diag_nocompute") {
    h->diag_nocompute = value != 0;
  } else if (k == "dk_slots") {
    // +64: 2-D TMA at d = 64 too (A/B); +128: DIAGNOSTIC ONLY, K5 CTAs return at entry (launch cost)
    // +256: DIAGNOSTIC, no private units; +512 / +1024: DIAGNOSTIC, no UMMA / no softmax math
    // +16384: 2-D maps at d = 128 (A/B); + 32768 v: V ring slots v (1..7)
    // + 262144 s: private-unit stages s; + 1048576: keep the chunk-first state set (A/B)
    h->dk_slots = (int)std::max<int64_t>(0, std::min<int64_t>(value, 2097151));
    return CA_OK;
  } else if (k == "sf_prefetch") {
    h->sf_prefetch = value < 0 ? 0 : (int)std::min<int64_t>(value, 31);
    return CA_OK;
  } else if (k == "trace") {
    h->trace_kernel = (int)value;
    return CA_OK;
  } else if (k == "sf_ctas_per_sm") {
    h->sf_ctas_per_sm = value <= 1 ? 1 : 2;
    h->sf_ctas_req = (int64_t)h->sf_ctas_per_sm * h->num_sms;
    h->resident_cache = -1;
  } else if (k == "pdl") {
    h->use_pdl = value != 0;
  } else if (k == "kernel_events") {
    if (h->host_only) return fail(CA_EINVAL, "host-only handle");
    h->kernel_events = value != 0;
    return CA_OK;
  } else {
    return fail(CA_EINVAL, "unknown option " + k);
  }
  h->ctx.epoch = -1;  // force a rebuild with the new schedule
  h->attend_epoch = h->append_epoch = -1;
  return CA_OK;
}

chunkattn_status chunkattn_kernel_times(chunkattn_t h, double ms[4], int64_t launches[4]) {
  if (!h || !ms || !launches) return fail(CA_EINVAL, "bad argument");
  if (h->host_only) return fail(CA_EINVAL, "host-only handle");
  if (h->set_device() != CA_OK) return CA_ECUDA;
  cudaError_t e = h->flush_times();
  if (e != cudaSuccess) return h->cuda_fail(e, "kernel_times");
  for (int k = 0; k < 4; ++k) {
    ms[k] = h->acc_ms[k];
    launches[k] = h->acc_n[k];
    h->acc_ms[k] = 0;
    h->acc_n[k] = 0;
  }
  return CA_OK;
}

chunkattn_status chunkattn_host_tables(chunkattn_t h, void* dst, size_t cap, size_t* len) {
  CA_GUARD_BEGIN
  if (!h || !len) return fail(CA_EINVAL, "bad argument");
  const size_t bytes = h->ctx.blob.size() * 4;
  *len = bytes;
  if (!dst || cap < bytes) return fail(CA_ERANGE, "buffer too small");
  std::memcpy(dst, h->ctx.blob.data(), bytes);
  return CA_OK;
  CA_GUARD_END
}

chunkattn_status chunkattn_download_tables(chunkattn_t h, void* dst, size_t cap, size_t* len, void* stream) {
  CA_GUARD_BEGIN
  if (!h || !len) return fail(CA_EINVAL, "bad argument");
  if (h->host_only) return fail(CA_EINVAL, "host-only handle");
  if (h->failed) return fail(CA_ECUDA, "handle failed on an earlier CUDA error");
  const size_t bytes = h->ctx.blob.size() * 4;
  *len = bytes;
  if (!dst || cap < bytes) return fail(CA_ERANGE, "buffer too small");
  if (h->set_device() != CA_OK) return CA_ECUDA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dst, h->wsp + h->ws.tables, bytes, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return h->cuda_fail(e, "download");
  return CA_OK;
  CA_GUARD_END
}

}  // extern "C"
