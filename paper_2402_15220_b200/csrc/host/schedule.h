// Context generation for the two-phase partition (§3.3): from the
// prefix tree build, on the host, the chunk-first work list (C, i, j) and the
// per-sequence private chunk lists, plus the scheduling tables the kernels use
// (runs split into tiles sized for 148 SMs, merge lists fixing the Eqn 2
// reduction order).  The result is one packed int32 blob copied to the GPU in a
// single cudaMemcpyAsync when the tree structure changed (lazy context copy).
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "tree.h"

namespace pakv {

// Chunk-first tile record in the blob (kCfTileInts int32 each).
// CF_LANES: token lanes of the tile (1 in the two-kernel chunk-first CTA,
// which merges its lanes itself; L = 4 / row groups in the fused kernel).
// CF_PARTS: partials written per row: 1 when the fused kernel merges its lanes
// in the stage's shared memory (fits when (4 - G) lane states fit the K/V
// tiles), else L (slot = CF_SLOT + lane * rows + (row - CF_ROW0)).
enum CfTileField { CF_CHUNK_OFF = 0, CF_NCHUNK, CF_ROW0, CF_ROW1, CF_SLOT, CF_RUN, CF_LANES, CF_PARTS };
constexpr int kCfTileInts = 8;
constexpr int kMaxCfTileRows = 128;  // rows of one chunk-first tile (8 warps x 16 rows)
constexpr int kFusedTileRows = 64;   // fused kernel: 4 consumer warps x 16 rows
// Fused-kernel chunk-first unit (kCfUnitInts int32): {chunk id, tile, head,
// k << 2 | flags (1 first, 2 last)}
constexpr int kCfUnitInts = 4;

// Seq-first CTA record (kSfCtaInts int32 each): {u0, u1, cf0, cf1, ...}:
// seq-first units [u0, u1) and fused chunk-first units [cf0, cf1).
constexpr int kSfCtaInts = 8;
// Seq-first item record (kSfItemInts int32 each), item = row * h + head:
// segment-partial slot base (-1: the item is finished in place, no merge),
// number of CTA segments, first CTA.
constexpr int kSfItemInts = 4;
constexpr int kMaxSfCtas = 2048;
// Contributions one seq-first CTA makes (and merges it may owe) at its end:
// the host checks the bound per CTA (fused: its chunk-first rows + its items).
constexpr int kMaxPendingMerges = 256;
// Seq-first unit descriptor (kSfUnitInts int32 each), resolved on the host so
// the producer issues its copies after one load: {chunk id or -1 (row without
// private chunks), item, chunk index k in the item, units of the item, merge
// list [mg0, mg1) of the row, segment slot of this CTA's part of the item (-1:
// finished in place), segments of the item | kSfMerger on the merger's units}.
constexpr int kSfUnitInts = 8;
// bit of the {nsegs} word: this CTA's segment is the item's last -- its merger
constexpr int kSfMerger = 1 << 30;

// K5 cluster decode tables (decode.cu).  Unit record (kDkUnitInts int32):
// {chunk id, first row, rows, DK_* flags}; CTA record (kDkCtaInts): {u0, u1}
// = units of CTA rank r of the block's clusters; block record: {row0, rows}.
// DK_PACK: a row's last chunk packed with other rows' into one stage (one
// row per consumer warp); DK_END: the producer's end marker (device only);
// DK_FINAL: the CTA's last chunk-first unit; DK_SOLO (with DK_FINAL): the
// CTA's chunk-first units form one job.
enum DkFlags : int32_t {
  DK_FIRST = 1, DK_LAST = 2, DK_TAIL = 4, DK_PRIV = 8, DK_PACK = 16, DK_END = 32, DK_FINAL = 64, DK_SOLO = 128
};
constexpr int kDkUnitInts = 4;
constexpr int kDkCtaInts = 32;    // {u0, u1, npre, 0, descriptors of the first npre <= kDkCtaPre units}
constexpr int kDkCtaPre = 7;
constexpr int kDkBlockInts = 4;
constexpr int kDkMaxRows = 64;     // (head, row) states of one CTA: head-set size x block rows
constexpr int kDkPack = 4;         // rows' last chunks dealt per pack (16-token slots of a c = 64 stage)
constexpr int kDkMaxCluster = 16;  // cluster sizes considered (> 8: non-portable)

struct ScheduleOptions {
  int32_t share_threshold = 2;
  int32_t num_heads = 1;
  int64_t cf_chunks_per_tile = 0;  // 0 = auto
  int64_t cf_target_ctas = 296;    // auto rule: heads * tiles >= this
  int64_t sf_ctas = 296;           // persistent seq-first grid (<= kMaxSfCtas)
  bool fused = false;              // chunk-first units run inside the persistent seq-first kernel
  double cf_unit_cost = 1.6;       // fused balance: cost of a chunk-first unit in seq-first units (swept on cfg2)
  int64_t fused_tile_rows = kFusedTileRows;  // fused chunk-first tile rows (16..64): smaller = more, lighter jobs
  double sf_unit_fixed = 1.0;       // seq-first range split: fixed share of a unit's cost (1 = unit counts)
  double sf_item_cost = 0.0;        // ... plus this per item end (finalize), in units
  int32_t head_dim = 128;          // fused lane merge: scratch bytes vs the stage's K/V tiles
  int32_t elem_bytes = 2;
  bool cf_lane_merge = true;       // fused: merge token lanes in shared memory (one partial per row)
  int64_t slot_capacity = 0;       // partial slots available in the workspace
  int64_t table_capacity = 0;      // int32 entries available for the blob
  int64_t seg_capacity = 0;        // seq-first segment partial rows available
  // K5 cluster decode
  bool dk = false;
  bool dk_force = false;  // K5 even when a shared run spans several row blocks
  int32_t dk_max_rows = kDkMaxRows;
  int32_t dk_cs_forced = 0;                        // > 0: cluster size to use
  int32_t dk_max_clusters[kDkMaxCluster + 1] = {};  // co-resident clusters of each size (0: unsupported)
  double dk_shared_fixed = 1.0;  // unit costs for the per-cluster split: chunk-first unit = fixed + per_row * rows
  double dk_shared_row = 0.01;
  double dk_pack_fixed = 1.3;    // a pack of last chunks = fixed + sum of valid / c / 2
  int32_t dk_hg_forced = 0;      // > 0: heads per cluster group (divides num_heads)
  // K5 chunk-first units on tcgen05 (decode.cu UM variant): 0 off, 1 when the
  // chunk-first units are at least dk_umma_ratio x the full private chunks,
  // 2 always; dk_umma_ok = the shape has the variant (16-bit, c = 64)
  int32_t dk_umma = 1;
  bool dk_umma_ok = false;
  double dk_umma_ratio = 0.5;
};

// Offsets (int32 units) of the arrays inside the blob.
struct BlobLayout {
  int64_t seq_len2 = 0, dk_block = 0, dk_cta = 0, dk_unit = 0;
  int64_t seq_len = 0, sf_first = 0, last_chunk = 0, last_start = 0, sf_ptr = 0, mg_ptr = 0,
          sf_chunk = 0, mg_slot = 0, cf_chunk = 0, cf_tile = 0, sf_cta = 0, sf_item = 0, sf_unit = 0, mg_tile = 0,
          cf_unit = 0, total = 0;
};

struct Context {
  int64_t epoch = -1;
  std::vector<int64_t> order;                  // seq ids by row
  std::unordered_map<int64_t, int32_t> row_of;  // seq id -> row
  std::vector<ChunkRec> recs;                   // DFS pre-order chunk records
  std::vector<int32_t> blob;                    // packed tables
  BlobLayout lay;
  int32_t b = 0;
  int32_t n_cf_tiles = 0;
  int32_t n_runs = 0;
  int32_t max_tile_rows = 0;
  int64_t n_slots = 0;
  int64_t cf_chunks_per_tile = 0;
  int32_t n_sf_ctas = 0;
  int32_t n_seg_slots = 0;  // segment partials of items split across CTAs
  int32_t n_cf_units = 0;   // fused: chunk-first units (all CTAs)
  bool fused = false;
  // K5 cluster decode
  bool dk = false;
  int32_t dk_cs = 0, dk_blocks = 0, dk_groups = 0, dk_max_rows = 0, dk_hg = 1;
  int64_t dk_units = 0;
  bool dk_um = false;  // chunk-first units on tcgen05 requested (the launch checks the shared-memory layout)
  bool dk_all_solo = false;  // every CTA's chunk-first units form at most one job (no second state set needed)
};

// Build the context of the current tree.  Returns false (and sets *err) when
// the tables or the partial slots do not fit the capacities.
bool build_context(const PrefixTree& tree, const ScheduleOptions& opt, Context* ctx, std::string* err);

// Canonical export text (T5) from a built context.
std::string export_text(const PrefixTree& tree, const Context& ctx, int32_t share_threshold);

}  // namespace pakv
