// Host-side launch interface of the CUDA kernels (internal; not part of the C ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pakv {

enum DType : int32_t { DT_F32 = 0, DT_F16 = 1, DT_BF16 = 2 };

inline int dtype_bytes(int32_t dt) { return dt == DT_F32 ? 4 : 2; }

// Device views of the context tables of one epoch (pointers into the workspace).
struct DevTables {
  const int32_t* row_caller;  // row -> index in the caller's attend order
  int32_t* seq_len;           // [b] tokens per row (bumped by the append kernel)
  const int32_t* sf_first;    // [b] position of the first seq-first chunk
  const int32_t* sf_ptr;      // [b+1] CSR into sf_chunk
  const int32_t* sf_chunk;    // seq-first (private) chunk ids, path order
  const int32_t* mg_ptr;      // [b+1] CSR into mg_slot
  const int32_t* mg_slot;     // partial slots merged into each row, fixed order
  const int32_t* cf_chunk;    // chunk-first chunk ids (runs, path order)
  const int32_t* cf_tile;     // [n_cf_tiles][8] tile records (schedule.h)
  const int32_t* last_chunk;  // [b] append target chunk
  const int32_t* last_start;  // [b] its start position
  const int32_t* sf_cta;      // [n_sf_ctas][4] persistent seq-first ranges
  const int32_t* sf_item;     // [b*h][4] split-item records
  const int32_t* sf_unit;     // [units][4] unit descriptors
  const int32_t* mg_tile;     // chunk-first tile owning each merge-list slot (fused readiness flags)
  const int32_t* cf_unit;     // fused: [units][4] {tile, head, k, flags}
  int32_t n_cf_units;
  int32_t fused;              // chunk-first runs inside the persistent seq-first kernel
  int32_t b, n_cf_tiles, max_tile_rows, n_sf_ctas;
  // K5 cluster decode (decode.cu, schedule.h "dk" tables)
  const int32_t* dk_block;    // [blocks][4] {first row, rows}
  const int32_t* dk_cta;      // [blocks * cs][4] {u0, u1}: units of CTA rank r of the block's clusters
  const int32_t* dk_unit;     // [units][4] {chunk, row0, rows, DK_* flags}
  int32_t dk_cs, dk_groups, dk_max_rows, dk_blocks, dk_hg;
  int32_t dk_um;              // chunk-first units on tcgen05 (UM variant) when its layout fits
  int32_t dk_all_solo;        // every CTA has at most one chunk-first job (UM: one state set suffices)
  int32_t row_identity;       // row_caller[r] == r for every row (the caller's order is the row order)
};



// Trace record per CTA (debug timing, option "trace"): words
//   [0] kernel entry, [1] producer done, [2] consumers done,
//   [3 + 4u] producer issue time of unit u, [4 + 4u] consumer data-ready time,
//   [5 + 4u] consumer done time, [6 + 4u] bytes the unit's copies move, for the
//   first kTraceUnits units (fused: chunk-first units first).
// Chunk-first uses the same layout per tile.
constexpr int kTraceUnits = 31;
constexpr int kTraceWords = 3 + 4 * kTraceUnits;  // 127 -> padded to 128
constexpr int kTraceStride = 128;
constexpr int kTraceCtas = 2048;

struct PoolGeom {
  void* k;  // base of layer 0
  void* v;
  int64_t layer_stride;  // elements per layer = max_chunks*h*c*d
  int64_t max_chunks;
  int32_t h, c, d, num_layers;
  int32_t dtype;
};

struct AttnLaunch {
  PoolGeom pool;
  int32_t layer;
  const void* q;   // [n][h][d] dtype, caller order
  void* out;       // [n][h][d] out_dtype, caller order
  int32_t out_dtype;
  float* pO;       // [slots][h][d+4]: o, then m (log2 units), n
  float* segO;     // [seg slots][d+4] seq-first segment partials, same format
  uint32_t* counters;  // [b * h] per-item contribution counters (zero between launches)
  float scale_log2;
  uint64_t* trace;       // optional per-CTA timeline ([cta][kTraceWords] globaltimer ns), or null
  bool trace_cf;         // trace the chunk-first kernel instead of seq-first
  int sf_ctas_per_sm;    // 1 or 2: shared-memory budget of the seq-first CTA
  int sf_prefetch;       // seq-first L2 prefetch distance in units (0 = off)
  bool cf_tensor_cores;  // use the mma chunk-first kernel
  bool cf_small;         // 4-warp chunk-first CTA (co-resident with seq-first) when tiles allow
  bool cf_umma;          // tcgen05 chunk-first kernel when supported (two-kernel path)
  int dk_slots;          // K5 tcgen05 variant: cap on K + V ring slots (0 = as many as fit)
  bool sf_tensor_cores;  // use the mma consumers in the seq-first kernel (16-bit types)
  bool use_pdl;
};

// K5 cluster decode launch: the step's append (mode bit 0: scatter k/v, the
// caller-order [n][h][d] rows of this layer; bit 1: lengths advance by one and
// are written to len_out, the other length buffer) folded into the attend.
struct DkAppend {
  const void* k;
  const void* v;
  int32_t* len_out;
  int32_t mode;
};
bool dk_supported(const PoolGeom& pool);
// 2-D TMA views of the K / V pools (boxes of 64 elements x c rows; the pool
// rows are XOR pre-swizzled, so a box lands as SWIZZLE_128B atoms), cached
bool pool_maps(const PoolGeom& p, int D, int C, CUtensorMap* mk, CUtensorMap* mv);
// d = 128 only: 3-D views {64, rows, 2 halves} so one box moves a whole tile as
// its two SWIZZLE_128B images (false if the driver rejects the map)
bool pool_maps3(const PoolGeom& p, int C, CUtensorMap* mk, CUtensorMap* mv);
size_t dk_stage_bytes(int32_t dtype, int32_t c, int32_t d);
size_t dk_state_bytes(int32_t d);
size_t dk_recv_bytes(int32_t d, int32_t nstate, int32_t cs);
int dk_stages(int32_t dtype, int32_t c, int32_t d, size_t recv);
size_t dk_smem_bytes(int32_t dtype, int32_t c, int32_t d, size_t recv);
int dk_consumer_warps();
// the UM variant (tcgen05 chunk-first units) exists for this pool shape
bool dk_umma_supported(const PoolGeom& pool);
// ... and its shared-memory layout fits nstate (head, row) states in clusters of cs
bool dk_um_fits(const PoolGeom& pool, int nstate, int cs);
// clusters of cs CTAs that can be co-resident (cudaOccupancyMaxActiveClusters), 0 if unsupported
int dk_max_active_clusters(const PoolGeom& pool, int out_dtype, int cs);
cudaError_t launch_decode(const AttnLaunch& a, const DevTables& t, const DkAppend& ap, cudaStream_t st);

// Prefill attention with prefix lookup (prefill.cu): tile record (kPfTileInts
// int32) {chunk list offset, first query row, queries (<= 64), position of the
// first query, sequence length, 0, 0, 0}; chunk lists are path order.
constexpr int kPfTileInts = 8;
constexpr int kPfTileRows = 64;
struct PrefillLaunch {
  PoolGeom pool;
  int32_t layer;
  const void* q;  // [total queries][h][d] dtype
  void* out;      // [total queries][h][d] out_dtype
  int32_t out_dtype;
  const int32_t* tiles;
  const int32_t* chunks;
  int32_t n_tiles;
  float scale_log2;
};
bool prefill_supported(const PoolGeom& pool);
// tcgen05 prefill (chunk_first_umma.cu, PREFILL mode): tiles of <= kPfTileRowsUmma queries
constexpr int kPfTileRowsUmma = 128;  // one 128-row UMMA group per CTA (chunk_first_umma.cu kPfGroups)
bool prefill_umma_supported(const PoolGeom& pool);
cudaError_t launch_prefill_umma(const PrefillLaunch& a, cudaStream_t st);
cudaError_t launch_prefill(const PrefillLaunch& a, cudaStream_t st);

// K1: scatter one decode step's K/V into the leaf chunks and set seq_len.
struct AppendItem {
  int32_t row, chunk, slot, new_len;
};
constexpr int kMaxAppendItems = 1024;  // per launch (items travel as kernel parameters)
cudaError_t launch_append_kv(const PoolGeom& pool, const DevTables& t, const AppendItem* items, int32_t n,
                             const void* k, const void* v, cudaStream_t st);

// Copy rows [first_pos, first_pos+m) of one sequence into its chunks
// (chunk of position p = chunks[p/c - first_pos/c]); src [m][L][h][d].
cudaError_t launch_copy_rows(const PoolGeom& pool, const int32_t* chunks, int32_t n_chunks, int64_t first_pos,
                             int64_t m, const void* k, const void* v, cudaStream_t st);

// Tokens per consumer warp of the MMA seq-first kernel for (dtype, chunk size),
// 0 when that kernel does not take the shape (fp32, or no tpw in {16, 32, 64}
// with c % tpw == 0 and c / tpw <= 4 consumer warps) and the SIMT consumers
// run instead.  The fused schedule (chunk-first units inside the persistent
// kernel) needs the MMA kernel: the SIMT consumers never run chunk-first units.
inline int sf_mma_tpw(int32_t dtype, int32_t c, bool sf_tensor_cores) {
  if (dtype == DT_F32 || !sf_tensor_cores) return 0;
  for (int tpw : {16, 32, 64})
    if (c % tpw == 0 && c / tpw <= 4) return tpw;
  return 0;
}
// Shared memory of one persistent seq-first CTA at its minimum ring depth (2
// stages) and whether it fits the 227 KB opt-in limit (valid_config rejects
// shapes that do not).
size_t seq_first_min_smem(int32_t dtype, int32_t c, int32_t d);
constexpr size_t kMaxSmemPerCta = 227 * 1024;
// CTAs of the persistent seq-first kernel that can be resident at once on the
// current device for this launch configuration (occupancy x SMs), 0 on error.
// The fused schedule's cross-CTA merges assume the grid is one wave: the
// host clamps the grid to this.
int seq_first_resident_ctas(const PoolGeom& pool, int out_dtype, int sf_ctas_per_sm, bool sf_tensor_cores);

// K3: chunk-first phase (Alg 1) -> partial slots.
cudaError_t launch_chunk_first(const AttnLaunch& a, const DevTables& t, cudaStream_t st);
// K4: seq-first phase (Alg 2) -> merged, normalised output.
cudaError_t launch_seq_first(const AttnLaunch& a, const DevTables& t, cudaStream_t st);

bool cf_mma_supported(const PoolGeom& pool);
// tcgen05 chunk-first (chunk_first_umma.cu): 16-bit, d in {64, 128}, c = 64, tiles <= 128 rows
bool cf_umma_supported(const PoolGeom& pool, int max_tile_rows);
cudaError_t launch_chunk_first_umma(const AttnLaunch& a, const DevTables& t, cudaStream_t st);

}  // namespace pakv
