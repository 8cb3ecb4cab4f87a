// Context builder.  See schedule.h.
#include "schedule.h"

#include <algorithm>
#include <cmath>
#include <cstdio>

namespace pakv {

namespace {

struct Run {
  std::vector<int32_t> chunks;  // path order (root -> leaf)
  int32_t i, j;                 // inclusive rows (PAPER.md:162 tuple convention)
};

// Tiles of one run for a chunks-per-tile value: (splits, row tiles, rows per tile).
struct RunTiling {
  int64_t splits, row_tiles, rows_per_tile;
};

RunTiling tile_run(const Run& r, int64_t cpt, int64_t max_rows) {
  const int64_t rows = r.j - r.i + 1;
  const int64_t n = (int64_t)r.chunks.size();
  RunTiling t;
  t.splits = (n + cpt - 1) / cpt;
  t.row_tiles = (rows + max_rows - 1) / max_rows;
  // balanced row tiles, multiples of 16 rows (one MMA row group) where possible
  int64_t per = (rows + t.row_tiles - 1) / t.row_tiles;
  per = std::min<int64_t>(max_rows, (per + 15) / 16 * 16);
  t.rows_per_tile = per;
  t.row_tiles = (rows + per - 1) / per;
  return t;
}

// Fused kernel: 4 consumer warps = G row groups (16 rows each, G a power of
// two) x L token lanes; each lane writes its own partial row.
int32_t fused_lanes(int64_t rows) {
  int32_t g = 1;
  while (g * 16 < rows) g *= 2;
  return 4 / g;
}

}  // namespace

bool build_context(const PrefixTree& tree, const ScheduleOptions& opt, Context* ctx, std::string* err) {
  const int32_t c = tree.c();
  const int32_t thr = opt.share_threshold;
  Context& X = *ctx;
  tree.dfs(&X.order, &X.recs);
  const int32_t b = (int32_t)X.order.size();
  X.b = b;
  X.row_of.clear();
  X.row_of.reserve(b * 2 + 1);
  for (int32_t r = 0; r < b; ++r) X.row_of[X.order[r]] = r;

  // ---- runs: maximal chains of shared chunks with one row range (pre-order)
  std::vector<Run> runs;
  std::unordered_map<int32_t, int32_t> run_of;  // chunk id -> run index
  for (const ChunkRec& rec : X.recs) {
    const Node& nd = tree.node(rec.id);
    if (nd.ref < thr) continue;
    int32_t ri = -1;
    if (nd.parent >= 0) {
      auto it = run_of.find(nd.parent);
      if (it != run_of.end() && runs[it->second].i == rec.i && runs[it->second].j == rec.j) ri = it->second;
    }
    if (ri < 0) {
      ri = (int32_t)runs.size();
      runs.push_back(Run{{}, rec.i, rec.j});
    }
    runs[ri].chunks.push_back(rec.id);
    run_of[rec.id] = ri;
  }
  X.n_runs = (int32_t)runs.size();

  // ---- seq-first lists: path suffix with ref < threshold (Alg 2 "chunks in T
  // with respect to q only")
  std::vector<int32_t> sf_ptr(b + 1, 0), sf_first(b), last_chunk(b), last_start(b), seq_len(b);
  std::vector<int32_t> sf_chunk;
  for (int32_t r = 0; r < b; ++r) {
    const Sequence* s = tree.find(X.order[r]);
    const auto& p = s->path;
    size_t k = p.size();
    while (k > 0 && tree.node(p[k - 1]).ref < thr) --k;
    sf_first[r] = (int32_t)k * c;
    for (size_t q = k; q < p.size(); ++q) sf_chunk.push_back(p[q]);
    sf_ptr[r + 1] = (int32_t)sf_chunk.size();
    last_chunk[r] = p.back();
    last_start[r] = tree.node(p.back()).start_pos;
    seq_len[r] = (int32_t)s->len;
  }

  // ---- K5 cluster decode: groups = row blocks x head sets (hg heads), one
  // cluster of cs CTAs each (hg, cs: the most CTAs with every group
  // co-resident).  Per group the work list (per head: shared runs clipped to
  // the block, then full private chunks) is cut into cs contiguous pieces of
  // equal cost; the rows' last chunks are dealt in packs to the least-loaded
  // ranks.  Units carry the head of the set in the flags word (bits 8+).
  std::vector<int32_t> dk_block, dk_cta, dk_unit;
  // K5 takes the step unless a shared run spans more rows than one block
  // holds: there the persistent kernels (tcgen05 chunk-first over up to 128
  // rows per tile) read each shared chunk once instead of once per block
  int32_t max_run_rows = 0;
  for (const Run& r : runs) max_run_rows = std::max(max_run_rows, r.j - r.i + 1);
  X.dk = opt.dk && b > 0 && (opt.dk_force || max_run_rows <= std::min(opt.dk_max_rows, kDkMaxRows));
  if (X.dk) {
    const int32_t H = opt.num_heads;
    int32_t hg = 1, cs = 1, nblk = 1;
    int64_t best = -1;
    for (int32_t g = 1; g <= H && g <= kDkMaxRows; g *= 2) {
      if (H % g != 0 || (opt.dk_hg_forced > 0 && g != opt.dk_hg_forced)) continue;
      const int32_t rows_cap = std::min<int32_t>(opt.dk_max_rows, kDkMaxRows / g);
      if (g > 1 && b > rows_cap) continue;  // head sets only for batches within one block
      const int32_t nb = (b + rows_cap - 1) / rows_cap;
      const int64_t groups = (int64_t)nb * (H / g);
      int32_t k = 1;
      if (opt.dk_cs_forced > 0) {
        k = std::min<int32_t>(opt.dk_cs_forced, kDkMaxCluster);
      } else {  // the largest cluster with every group co-resident (one wave)
        for (int32_t kk = kDkMaxCluster; kk >= 1; --kk)
          if (opt.dk_max_clusters[kk] > 0 && groups <= opt.dk_max_clusters[kk]) {
            k = kk;
            break;
          }
      }
      const int64_t ctas = groups * k;
      if (ctas > best) {
        best = ctas;
        hg = g;
        cs = k;
        nblk = nb;
      }
    }
    const int32_t per = (b + nblk - 1) / nblk;  // balanced blocks
    X.dk_cs = cs;
    X.dk_hg = hg;
    X.dk_blocks = nblk;
    X.dk_groups = nblk * (H / hg);
    X.dk_max_rows = 0;
    std::vector<int32_t> units;  // this block's {chunk, row0, rows, flags | hh << 8}
    std::vector<double> pre;
    for (int32_t bl = 0; bl < nblk; ++bl) {
      const int32_t r0 = bl * per, r1 = std::min(b, r0 + per);
      X.dk_max_rows = std::max(X.dk_max_rows, r1 - r0);
      dk_block.insert(dk_block.end(), {r0, r1 - r0, 0, 0});
      units.clear();
      pre.assign(1, 0.0);
      auto add = [&](int32_t chunk, int32_t a, int32_t n, int32_t fl, double cost) {
        units.insert(units.end(), {chunk, a, n, fl});
        pre.push_back(pre.back() + cost);
      };
      for (int32_t hh = 0; hh < hg; ++hh)
        for (const Run& r : runs) {
          const int32_t a = std::max(r.i, r0), e = std::min(r.j + 1, r1);
          if (a >= e) continue;
          for (int32_t ch : r.chunks) add(ch, a, e - a, hh << 8, opt.dk_shared_fixed + opt.dk_shared_row * (e - a));
        }
      // private chunks: every row's full chunks (cooperative units) ...
      for (int32_t hh = 0; hh < hg; ++hh)
        for (int32_t row = r0; row < r1; ++row) {
          const int32_t n = sf_ptr[row + 1] - sf_ptr[row];
          for (int32_t k = 0; k + 1 < n; ++k) add(sf_chunk[sf_ptr[row] + k], row, 1, DK_PRIV | (hh << 8), 1.0);
        }
      // ... and every row's last chunk (PACK: several rows per stage, one per
      // consumer warp -- decode tails are short), dealt to the ranks below
      std::vector<std::pair<int32_t, int32_t>> tails;  // (hh, row)
      std::vector<int32_t> tail_nt;
      for (int32_t hh = 0; hh < hg; ++hh)
        for (int32_t row = r0; row < r1; ++row) {
          if (sf_ptr[row + 1] == sf_ptr[row]) continue;
          tails.push_back({hh, row});
          tail_nt.push_back(std::max<int32_t>(1, std::min<int32_t>(c, seq_len[row] - last_start[row])));
        }
      // packs as the device forms them: consecutive tails while their 16-token
      // slots fit one chunk and at most kDkPack rows (lengths at build time)
      std::vector<size_t> pack_at;  // first tail of each pack
      std::vector<double> pack_w;
      {
        int32_t used = 0, n = 0;
        for (size_t k = 0; k < tails.size(); ++k) {
          const int32_t sl = (tail_nt[k] + 15) / 16;
          if (n == 0 || used + sl > c / 16 || n == kDkPack) {
            pack_at.push_back(k);
            pack_w.push_back(opt.dk_pack_fixed);
            used = n = 0;
          }
          used += sl;
          ++n;
          pack_w.back() += 0.5 * tail_nt[k] / c;
        }
        pack_at.push_back(tails.size());
      }
      double W_tail = 0.0;
      for (double w : pack_w) W_tail += w;
      // the main list is cut into cs contiguous pieces of equal cost, and the
      // packs of last chunks are spread evenly over the ranks (contiguous
      // groups): their length grows between rebuilds, so no size model
      const int64_t nu = (int64_t)units.size() / kDkUnitInts;
      const double W = pre.back();
      std::vector<int64_t> cut(cs + 1, 0);
      cut[cs] = nu;
      for (int32_t rk = 1; rk < cs; ++rk) {
        const double target = W * rk / cs;
        int64_t k = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
        if (k > nu) k = nu;
        if (k > 0 && target - pre[k - 1] < pre[k] - target) --k;
        cut[rk] = std::max<int64_t>(cut[rk - 1], k);
      }
      std::vector<std::vector<std::pair<int32_t, int32_t>>> rank_tails(cs);
      const int64_t npk = (int64_t)pack_at.size() - 1;
      for (int32_t rk = 0; rk < cs; ++rk)
        for (int64_t pk = npk * rk / cs; pk < npk * (rk + 1) / cs; ++pk)
          for (size_t k = pack_at[pk]; k < pack_at[pk + 1]; ++k) rank_tails[rk].push_back(tails[k]);
      (void)W_tail;
      for (int32_t rk = 0; rk < cs; ++rk) {
        const int64_t g0 = (int64_t)dk_unit.size() / kDkUnitInts;
        for (int64_t u = cut[rk]; u < cut[rk + 1]; ++u) {
          const int32_t* d = &units[kDkUnitInts * u];
          // a job = consecutive units of one head, row range and kind inside this piece
          auto same = [&](int64_t v) {
            const int32_t* e = &units[kDkUnitInts * v];
            return e[1] == d[1] && e[2] == d[2] && e[3] == d[3];
          };
          const bool first = u == cut[rk] || !same(u - 1);
          const bool last = u == cut[rk + 1] - 1 || !same(u + 1);
          dk_unit.insert(dk_unit.end(), {d[0], d[1], d[2], d[3] | (first ? DK_FIRST : 0) | (last ? DK_LAST : 0)});
        }
        for (const auto& tl : rank_tails[rk])
          dk_unit.insert(dk_unit.end(), {sf_chunk[sf_ptr[tl.second + 1] - 1], tl.second, 1,
                                         DK_PRIV | DK_TAIL | DK_PACK | DK_FIRST | DK_LAST | (tl.first << 8)});
        const int64_t g1 = (int64_t)dk_unit.size() / kDkUnitInts;
        {  // the CTA's last chunk-first unit (and whether its chunk-first units are one job)
          int64_t last_cf = -1, jobs = 0;
          for (int64_t u = g0; u < g1; ++u) {
            const int32_t f = dk_unit[(size_t)kDkUnitInts * u + 3];
            if (f & DK_PRIV) continue;
            last_cf = u;
            if (f & DK_FIRST) ++jobs;
          }
          if (last_cf >= 0) dk_unit[(size_t)kDkUnitInts * last_cf + 3] |= DK_FINAL | (jobs == 1 ? DK_SOLO : 0);
        }
        const int32_t npre = (int32_t)std::min<int64_t>(kDkCtaPre, g1 - g0);
        dk_cta.insert(dk_cta.end(), {(int32_t)g0, (int32_t)g1, npre, 0});
        for (int32_t k = 0; k < kDkCtaPre; ++k)
          for (int32_t f = 0; f < kDkUnitInts; ++f)
            dk_cta.push_back(k < npre ? dk_unit[(size_t)kDkUnitInts * (g0 + k) + f] : 0);
      }
    }
    X.dk_units = (int64_t)dk_unit.size() / kDkUnitInts;
    int64_t n_cf = 0, n_pv = 0;  // chunk-first units, full private chunks
    for (int64_t u = 0; u < X.dk_units; ++u) {
      const int32_t f = dk_unit[(size_t)kDkUnitInts * u + 3];
      if (!(f & DK_PRIV)) ++n_cf;
      else if (!(f & DK_PACK)) ++n_pv;
    }
    X.dk_um = opt.dk_umma_ok && n_cf > 0 && (opt.dk_umma == 2 || (opt.dk_umma == 1 && n_cf >= opt.dk_umma_ratio * n_pv));
    X.dk_all_solo = true;  // every FINAL unit also SOLO
    for (int64_t u = 0; u < X.dk_units; ++u) {
      const int32_t f = dk_unit[(size_t)kDkUnitInts * u + 3];
      if ((f & DK_FINAL) && !(f & DK_SOLO)) X.dk_all_solo = false;
    }
  }
  // old schedules (two-kernel / fused persistent): not built when the K5
  // cluster decode runs the step
  std::vector<int32_t> cf_chunk, cf_tile, mg_ptr(b + 1, 0), mg_slot, mg_tile, sf_cta, sf_item, sf_unit, cf_unit;
  if (!X.dk) {
    // ---- split rule: chunks per tile so that heads * tiles >= target CTAs
    int64_t max_n = 1;
    for (const Run& r : runs) max_n = std::max<int64_t>(max_n, (int64_t)r.chunks.size());
    if (opt.fused) {  // a run wider than the fused tile would re-read its K/V per 64-row tile
      for (const Run& r : runs)
        if (r.j - r.i + 1 > kFusedTileRows) {
          ScheduleOptions o2 = opt;
          o2.fused = false;
          return build_context(tree, o2, ctx, err);
        }
    }
    const int64_t tile_rows = opt.fused ? std::min<int64_t>(kFusedTileRows, std::max<int64_t>(16, opt.fused_tile_rows))
                                        : kMaxCfTileRows;
    auto lanes_of = [&](const RunTiling& t) { return opt.fused ? fused_lanes(t.rows_per_tile) : 1; };
    // partials per row: the fused kernel merges its L lanes in the stage's K/V
    // tiles when the (4 - G) foreign lane states fit there
    auto parts_of = [&](const RunTiling& t) {
      const int32_t L = lanes_of(t);
      if (L == 1 || !opt.cf_lane_merge) return L;
      const int64_t G = 4 / L;
      const int64_t scratch = (4 - G) * (opt.head_dim / 2 + 4) * 32 * 4;
      return scratch <= 2LL * c * opt.head_dim * opt.elem_bytes ? 1 : L;
    };
    auto count = [&](int64_t cpt, int64_t* tiles, int64_t* slots) {
      *tiles = 0;
      *slots = 0;
      for (const Run& r : runs) {
        RunTiling t = tile_run(r, cpt, tile_rows);
        *tiles += t.splits * t.row_tiles;
        *slots += t.splits * (r.j - r.i + 1) * parts_of(t);
      }
    };
    int64_t cpt = max_n, tiles = 0, slots = 0;
    if (opt.cf_chunks_per_tile > 0) {
      cpt = std::min<int64_t>(opt.cf_chunks_per_tile, max_n);
    } else if (!runs.empty()) {
      // cost = waves x (chunks per tile + fixed per-CTA overhead, in chunk
      // loads: prologue/epilogue latency and the partial written here and read
      // back by the seq-first phase); ties go to the larger tile (fewer
      // partials).  One wave = cf_target_ctas CTAs (1 CTA per SM).
      constexpr int64_t kTileOverhead = 3;
      int64_t best = -1;
      for (int64_t t = max_n; t >= 1; --t) {
        count(t, &tiles, &slots);
        const int64_t waves = (tiles * opt.num_heads + opt.cf_target_ctas - 1) / opt.cf_target_ctas;
        const int64_t cost = waves * (t + kTileOverhead);
        if (best < 0 || cost < best) {
          best = cost;
          cpt = t;
        }
      }
    }
    count(cpt, &tiles, &slots);
    while (slots > opt.slot_capacity && cpt < max_n) count(++cpt, &tiles, &slots);
    if (slots > opt.slot_capacity) {
      if (opt.fused) {  // the fused schedule's per-lane partials do not fit: two-kernel schedule (one per row)
        ScheduleOptions o2 = opt;
        o2.fused = false;
        return build_context(tree, o2, ctx, err);
      }
      *err = "partial slots exceed workspace capacity";
      return false;
    }
    X.cf_chunks_per_tile = cpt;
    X.n_slots = slots;

    // ---- tiles, cf chunk lists, merge lists (fixed order: runs root->leaf,
    // splits ascending: reading A12)
    std::vector<int32_t> mg_cnt(b + 1, 0);
    for (const Run& r : runs) {
      RunTiling t = tile_run(r, cpt, tile_rows);
      for (int32_t row = r.i; row <= r.j; ++row) mg_cnt[row + 1] += (int32_t)(t.splits * parts_of(t));
    }
    mg_ptr.assign(b + 1, 0);
    for (int32_t r = 0; r < b; ++r) mg_ptr[r + 1] = mg_ptr[r] + mg_cnt[r + 1];
    mg_slot.assign(mg_ptr[b], 0);
    mg_tile.assign(mg_ptr[b], 0);
    std::vector<int32_t> mg_fill(mg_ptr.begin(), mg_ptr.end() - 1);
    int64_t slot = 0;
    int32_t max_rows = 0;
    for (size_t ri = 0; ri < runs.size(); ++ri) {
      const Run& r = runs[ri];
      RunTiling t = tile_run(r, cpt, tile_rows);
      const int32_t L = lanes_of(t), P = parts_of(t);
      const int64_t n = (int64_t)r.chunks.size();
      for (int64_t s = 0; s < t.splits; ++s) {
        const int64_t k0 = s * n / t.splits, k1 = (s + 1) * n / t.splits;  // balanced split
        const int32_t off = (int32_t)cf_chunk.size();
        for (int64_t k = k0; k < k1; ++k) cf_chunk.push_back(r.chunks[k]);
        for (int64_t rt = 0; rt < t.row_tiles; ++rt) {
          const int32_t r0 = r.i + (int32_t)(rt * t.rows_per_tile);
          const int32_t r1 = std::min<int32_t>(r.j + 1, r0 + (int32_t)t.rows_per_tile);
          const int32_t tile_id = (int32_t)(cf_tile.size() / kCfTileInts);
          cf_tile.insert(cf_tile.end(), {off, (int32_t)(k1 - k0), r0, r1, (int32_t)slot, (int32_t)ri, L, P});
          for (int32_t row = r0; row < r1; ++row)
            for (int32_t l = 0; l < P; ++l) {  // lane partials in lane order (fixed merge order, A12)
              mg_tile[mg_fill[row]] = tile_id;
              mg_slot[mg_fill[row]++] = (int32_t)(slot + (int64_t)l * (r1 - r0) + (row - r0));
            }
          slot += (int64_t)(r1 - r0) * P;
          max_rows = std::max(max_rows, r1 - r0);
        }
      }
    }
    X.n_cf_tiles = (int32_t)(cf_tile.size() / kCfTileInts);
    X.max_tile_rows = max_rows;

    // ---- persistent seq-first schedule: items (row, head) in row-major order,
    // each worth max(1, private chunks) units; CTA g takes units
    // [U g / G, U (g+1) / G) (balanced, contiguous; stream-K style).  Items cut
    // by a CTA boundary are merged by their last contributor, in CTA order
    // (deterministic).
    const int32_t H = opt.num_heads;
    std::vector<int64_t> row_u0(b + 1, 0);  // first unit of row r (all heads)
    for (int32_t r = 0; r < b; ++r)
      row_u0[r + 1] = row_u0[r] + (int64_t)H * std::max<int32_t>(1, sf_ptr[r + 1] - sf_ptr[r]);
    const int64_t U = row_u0[b];
    const int64_t G = b == 0 ? 0 : std::max<int64_t>(1, std::min<int64_t>({U, opt.sf_ctas, kMaxSfCtas}));
    sf_cta.assign(kSfCtaInts * G, 0);
    sf_item.assign((size_t)kSfItemInts * b * H, 0);
    // per-unit descriptors {chunk id or -1, item, k, units of the item}
    sf_unit.assign((size_t)kSfUnitInts * U, 0);
    for (int32_t r = 0; r < b; ++r) {
      const int32_t n = sf_ptr[r + 1] - sf_ptr[r], per = std::max<int32_t>(1, n);
      for (int32_t hh = 0; hh < H; ++hh) {
        const int64_t base = row_u0[r] + (int64_t)hh * per;
        for (int32_t k = 0; k < per; ++k) {
          int32_t* d = &sf_unit[(size_t)kSfUnitInts * (base + k)];
          d[0] = n > 0 ? sf_chunk[sf_ptr[r] + k] : -1;
          d[1] = r * H + hh;
          d[2] = k;
          d[3] = per;
          d[4] = mg_ptr[r];
          d[5] = mg_ptr[r + 1];
        }
      }
    }
    // Fused: chunk-first jobs (tile, head) go first, by longest-processing-time
    // greedy to the least-loaded CTA; the seq-first units then fill every CTA up
    // to the common target (contiguous ranges, proportional to the room left).
    // seq-first unit costs for the range split: a fixed share per unit plus its
    // valid-token fraction, plus an item-end (finalize) cost; with the defaults
    // (fixed 1, item 0) every unit weighs 1 (plain unit counts)
    std::vector<double> ucost_pre((size_t)U + 1, 0.0);
    {
      const double a = opt.sf_unit_fixed, wf = opt.sf_item_cost;
      int64_t u = 0;
      for (int32_t r = 0; r < b; ++r) {
        const int32_t n = sf_ptr[r + 1] - sf_ptr[r], per = std::max<int32_t>(1, n);
        const int32_t last_tok = n > 0 ? std::min<int32_t>(c, seq_len[r] - sf_first[r] - (per - 1) * c) : 0;
        for (int32_t hh = 0; hh < H; ++hh)
          for (int32_t k = 0; k < per; ++k, ++u) {
            const double frac = n == 0 ? 0.0 : (k < per - 1 ? 1.0 : (double)last_tok / c);
            ucost_pre[u + 1] = ucost_pre[u] + a + (1.0 - a) * frac + (k == per - 1 ? wf : 0.0);
          }
      }
    }
    const double T_sf = ucost_pre[U];
    auto unit_at = [&](double cost) -> int64_t {  // first unit whose prefix cost reaches `cost`
      if (cost <= 0) return 0;
      if (cost >= T_sf) return U;
      const int64_t i = std::lower_bound(ucost_pre.begin(), ucost_pre.end(), cost) - ucost_pre.begin();
      // round to the nearer boundary
      return (i > 0 && cost - ucost_pre[i - 1] < ucost_pre[i] - cost) ? i - 1 : i;
    };
    std::vector<int64_t> ubound(G + 1, 0);
    std::vector<int32_t> cf_range(2 * G, 0);
    if (opt.fused && G > 0 && X.n_cf_tiles > 0) {
      const int64_t n_tiles = X.n_cf_tiles;
      std::vector<std::pair<int64_t, int64_t>> jobs;  // (-chunks, job) -> sorted: big first, then index
      for (int64_t tl = 0; tl < n_tiles; ++tl)
        for (int32_t hh = 0; hh < H; ++hh) jobs.push_back({-(int64_t)cf_tile[kCfTileInts * tl + CF_NCHUNK], tl * H + hh});
      std::sort(jobs.begin(), jobs.end());
      std::vector<double> load(G, 0.0);
      std::vector<std::vector<int64_t>> mine(G);
      for (const auto& jb : jobs) {
        int64_t best = 0;
        for (int64_t g = 1; g < G; ++g)
          if (load[g] < load[best]) best = g;
        load[best] += (double)(-jb.first) * opt.cf_unit_cost;
        mine[best].push_back(jb.second);
      }
      double total = T_sf;
      for (double l : load) total += l;
      const double target = total / (double)G;
      std::vector<double> room(G);
      double room_sum = 0;
      for (int64_t g = 0; g < G; ++g) room_sum += (room[g] = std::max(0.0, target - load[g]));
      double acc = 0;
      for (int64_t g = 0; g < G; ++g) {
        ubound[g] = room_sum > 0 ? unit_at(T_sf * acc / room_sum) : U * g / G;
        acc += room[g];
        cf_range[2 * g] = (int32_t)(cf_unit.size() / kCfUnitInts);
        for (int64_t job : mine[g]) {
          const int64_t tl = job / H;
          const int32_t nk = cf_tile[kCfTileInts * tl + CF_NCHUNK];
          const int32_t off = cf_tile[kCfTileInts * tl + CF_CHUNK_OFF];
          for (int32_t k = 0; k < nk; ++k)
            cf_unit.insert(cf_unit.end(), {cf_chunk[off + k], (int32_t)tl, (int32_t)(job % H),
                                           (k << 2) | (k == 0 ? 1 : 0) | (k == nk - 1 ? 2 : 0)});
        }
        cf_range[2 * g + 1] = (int32_t)(cf_unit.size() / kCfUnitInts);
      }
      ubound[G] = U;
    } else {
      for (int64_t g = 0; g <= G; ++g) ubound[g] = G > 0 ? unit_at(T_sf * (double)g / (double)G) : 0;
    }
    X.n_cf_units = (int32_t)(cf_unit.size() / kCfUnitInts);
    X.fused = opt.fused && X.n_cf_tiles > 0;
    int32_t seg_slots = 0;
    for (int64_t g = 0; g < G; ++g) {
      const int64_t u0 = ubound[g], u1 = ubound[g + 1];
      sf_cta[kSfCtaInts * g + 0] = (int32_t)u0;
      sf_cta[kSfCtaInts * g + 1] = (int32_t)u1;
      sf_cta[kSfCtaInts * g + 2] = cf_range[2 * g];
      sf_cta[kSfCtaInts * g + 3] = cf_range[2 * g + 1];
      // one segment for every item this CTA touches
      int64_t u = u0;
      while (u < u1) {
        const int32_t* d = &sf_unit[(size_t)kSfUnitInts * u];
        int32_t* rec = &sf_item[kSfItemInts * d[1]];
        if (rec[1] == 0) rec[2] = (int32_t)g;  // first CTA of the item
        rec[1] += 1;
        u += d[3] - d[2];
      }
    }
    // Segment slots for the items merged by their last contributor: split
    // items, and (fused) items whose chunk-first partials come from this same
    // launch.  Every other item is finished in place (slot base -1).
    for (int64_t i = 0; i < (int64_t)b * H; ++i) {
      int32_t* rec = &sf_item[kSfItemInts * i];
      const int32_t row = (int32_t)(i / H);
      if (rec[1] > 1 || (X.fused && mg_ptr[row + 1] > mg_ptr[row])) {
        rec[0] = seg_slots;
        seg_slots += rec[1];
      } else {
        rec[0] = -1;
      }
    }
    // each unit's segment slot: base + ordinal of its CTA among the item's CTAs
    {
      std::vector<int32_t> ord((size_t)b * H, 0);
      for (int64_t g = 0; g < G; ++g) {
        for (int64_t u = ubound[g]; u < ubound[g + 1];) {
          int32_t* d = &sf_unit[(size_t)kSfUnitInts * u];
          const int32_t item = d[1], left = d[3] - d[2];
          const int32_t* rec = &sf_item[kSfItemInts * item];
          const int32_t o = ord[item]++;
          const int32_t seg = rec[0] < 0 ? -1 : rec[0] + o;
          // the CTA holding the item's last segment is its merger (kSfMerger bit)
          const int32_t word = rec[1] | (rec[0] >= 0 && o == rec[1] - 1 ? kSfMerger : 0);
          const int64_t end = std::min<int64_t>(u + left, ubound[g + 1]);
          for (int64_t v = u; v < end; ++v) {
            sf_unit[(size_t)kSfUnitInts * v + 6] = seg;
            sf_unit[(size_t)kSfUnitInts * v + 7] = word;
          }
          u += left;
        }
      }
    }
    if (seg_slots > opt.seg_capacity) {
      *err = "segment partials exceed workspace capacity";
      return false;
    }
    // merges a CTA may owe at its end / segment contributions it records: at
    // most the items it touches that have slots
    for (int64_t g = 0; g < G; ++g) {
      int64_t owed = 0;
      for (int64_t u = ubound[g]; u < ubound[g + 1];) {
        const int32_t* d = &sf_unit[(size_t)kSfUnitInts * u];
        owed += sf_item[kSfItemInts * d[1]] >= 0 ? 1 : 0;
        u += d[3] - d[2];
      }
      if (owed > kMaxPendingMerges) {
        if (X.fused) {  // too many merges for one CTA: run the two-kernel schedule instead
          ScheduleOptions o2 = opt;
          o2.fused = false;
          return build_context(tree, o2, ctx, err);
        }
        *err = "too many pending merges per seq-first CTA";
        return false;
      }
    }
    X.n_sf_ctas = (int32_t)G;
    X.n_seg_slots = seg_slots;
  }

  // ---- pack the blob (seq_len first: the device copy is authoritative between
  // structural changes and is bumped by the append kernel)
  BlobLayout& L = X.lay;
  int64_t o = 0;
  auto place = [&](int64_t n) {
    int64_t at = o;
    o += (n + 3) / 4 * 4;  // 16-byte aligned sub-arrays
    return at;
  };
  L.seq_len = place(b);
  L.seq_len2 = place(b);  // second length buffer (K5 ping-pong: read one, write the other)
  L.sf_first = place(b);
  L.last_chunk = place(b);
  L.last_start = place(b);
  L.sf_ptr = place(b + 1);
  L.mg_ptr = place(b + 1);
  L.sf_chunk = place((int64_t)sf_chunk.size());
  L.mg_slot = place((int64_t)mg_slot.size());
  L.cf_chunk = place((int64_t)cf_chunk.size());
  L.cf_tile = place((int64_t)cf_tile.size());
  L.sf_cta = place((int64_t)sf_cta.size());
  L.sf_item = place((int64_t)sf_item.size());
  L.sf_unit = place((int64_t)sf_unit.size());
  L.mg_tile = place((int64_t)mg_tile.size());
  L.cf_unit = place((int64_t)cf_unit.size());
  L.dk_block = place((int64_t)dk_block.size());
  L.dk_cta = place((int64_t)dk_cta.size());
  L.dk_unit = place((int64_t)dk_unit.size());
  L.total = o;
  if (o > opt.table_capacity) {
    *err = "context tables exceed workspace capacity";
    return false;
  }
  X.blob.assign(o, 0);
  auto put = [&](int64_t at, const std::vector<int32_t>& v) {
    std::copy(v.begin(), v.end(), X.blob.begin() + at);
  };
  put(L.seq_len, seq_len);
  put(L.seq_len2, seq_len);
  put(L.sf_first, sf_first);
  put(L.last_chunk, last_chunk);
  put(L.last_start, last_start);
  put(L.sf_ptr, sf_ptr);
  put(L.mg_ptr, mg_ptr);
  put(L.sf_chunk, sf_chunk);
  put(L.mg_slot, mg_slot);
  put(L.cf_chunk, cf_chunk);
  put(L.cf_tile, cf_tile);
  put(L.sf_cta, sf_cta);
  put(L.sf_item, sf_item);
  put(L.sf_unit, sf_unit);
  put(L.mg_tile, mg_tile);
  put(L.cf_unit, cf_unit);
  put(L.dk_block, dk_block);
  put(L.dk_cta, dk_cta);
  put(L.dk_unit, dk_unit);
  X.epoch = tree.epoch();
  return true;
}

std::string export_text(const PrefixTree& tree, const Context& X, int32_t thr) {
  std::string out = "chunks:\n";
  char buf[160];
  for (const ChunkRec& rec : X.recs) {
    const Node& nd = tree.node(rec.id);
    const int32_t* t = tree.tokens(rec.id);
    std::snprintf(buf, sizeof buf, "%d %d %d %d %d %d %d\n", rec.id, nd.parent, nd.start_pos, nd.len,
                  nd.ref, t[0], t[nd.len - 1]);
    out += buf;
  }
  out += "order:";
  for (int64_t s : X.order) out += " " + std::to_string(s);
  out += "\nshared:";
  for (const ChunkRec& rec : X.recs)
    if (tree.node(rec.id).ref >= thr)
      out += " (" + std::to_string(rec.id) + "," + std::to_string(rec.i) + "," + std::to_string(rec.j) + ")";
  out += "\n";
  for (size_t r = 0; r < X.order.size(); ++r) {
    out += "private[" + std::to_string(r) + "]:";
    for (int32_t id : tree.find(X.order[r])->path)
      if (tree.node(id).ref < thr) out += " " + std::to_string(id);
    out += "\n";
  }
  out += "tuples:";
  for (const ChunkRec& rec : X.recs)
    out += " (" + std::to_string(rec.id) + "," + std::to_string(rec.i) + "," + std::to_string(rec.j) + ")";
  const ChunkPool& p = tree.pool();
  std::snprintf(buf, sizeof buf, "\nalloc: %lld %lld %lld %lld\n", (long long)p.used(),
                (long long)p.free_count(), (long long)p.created(), (long long)p.hwm());
  out += buf;
  return out;
}

}  // namespace pakv
