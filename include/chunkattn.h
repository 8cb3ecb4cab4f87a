/*
 * chunkattn.h — C ABI of the B200-native ChunkAttention decode library.
 *
 * What it computes (PAPER.md = arXiv 2402.15220 text under /root/reference):
 *   decode-time self-attention over a prefix-aware chunked KV cache (PAKV,
 *   §3.1) with the two-phase partition (TPP, §3.2,
 *   PAPER.md:51-158):
 *     chunk-first  (Alg 1):  every chunk C shared by rows i..j
 *                  is attended by Q[i..j] at once -> partial (O, m, n) (Eqn 1,
 *                  PAPER.md:95-108);
 *     seq-first    (Alg 2): every row walks its private
 *                  chunks and merges all partials with attn_reduce (Eqn 2,
 *                  PAPER.md:145-158), then O / n.
 *   The result equals softmax(s * q K^T) V per sequence over its whole KV
 *    up to rounding.  The prefix tree lives in host memory
 *   (PAPER.md:162); the context (C, i, j) plus private lists is built on the
 *   host and copied lazily (triggers "chunk full", "new sequence
 *   joining", "completed sequence leaving").
 *
 * Conventions
 *   - All functions return chunkattn_status; no C++ exception crosses the ABI.
 *     On any error the host state is unchanged (strong guarantee) and
 *     chunkattn_last_error() (thread-local) describes it.
 *   - A CUDA error makes the handle sticky-failed: every later call that would
 *     touch the device returns CA_ECUDA.
 *   - A handle is NOT thread-safe (single writer).  All calls that take a
 *     `stream` must be issued on one stream (or be ordered by the caller); the
 *     library keeps one set of device tables and relies on stream order.
 *   - "device" pointers are CUDA device pointers valid on config.device;
 *     "host" pointers are plain host memory.  Device inputs must stay valid
 *     until `stream` has passed the call (as with cudaMemcpyAsync).  The
 *     per-step tensors of append_kv (k, v) and attend (q, out) may also be
 *     PINNED host memory (cudaHostAlloc / page-locked, UVA): the kernels then
 *     read and write them over PCIe directly (zero-copy; no staging copy).
 *   - Layouts are dense, row-major, element type config.dtype unless stated.
 *     h = num_heads, d = head_dim, c = chunk_size, L = num_layers.
 *   - Host-only mode: config.device = -1 builds the prefix tree and tables
 *     without touching CUDA (k/v/q pointers ignored; attend/append return
 *     CA_EINVAL).  Used for host-logic tests on machines without a GPU.
 */
#ifndef CHUNKATTN_H
#define CHUNKATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct chunkattn* chunkattn_t; /* opaque handle */

typedef enum {
  CA_OK = 0,
  CA_EINVAL = -1,  /* bad argument (null pointer, size, layer, shape)            */
  CA_ENOSEQ = -2,  /* unknown (or removed) sequence id                           */
  CA_ENOMEM = -3,  /* chunk pool / table / workspace capacity exhausted          */
  CA_ESTATE = -4,  /* attend: n != live count, duplicate ids                     */
  CA_ECUDA = -5,   /* CUDA runtime error (sticky)                                */
  CA_EDTYPE = -6,  /* unsupported dtype / head_dim / chunk_size combination      */
  CA_ERANGE = -7   /* output buffer too small (export_context, batch_order)      */
} chunkattn_status;

typedef enum { CA_F32 = 0, CA_F16 = 1, CA_BF16 = 2 } chunkattn_dtype;

/* Static configuration (h = 32, d = 128, c = 64, FP16 in the
 * paper's experiments).  Supported: d in {64, 128}; c in [1, 256] (the tensor
 * core chunk-first path needs c % 16 == 0 and dtype F16/BF16; other shapes use
 * the SIMT chunk-first path). */
typedef struct {
  int32_t num_heads;       /* heads held by THIS handle (a rank's head slice)          */
  int32_t head_dim;        /* d                                                        */
  int32_t chunk_size;      /* c ("a segment of c context tokens")          */
  int32_t num_layers;      /* layers sharing one tree and one context (>= 1)           */
  int32_t dtype;           /* chunkattn_dtype of K, V, Q                               */
  int32_t out_dtype;       /* chunkattn_dtype of the attention output                   */
  int32_t share_threshold; /* chunk-first takes chunks with ref >= this (default 2,
                              PAPER.md:80 "shared by multiple sequences"); a huge value
                              disables TPP (baseline B1 = the paper's PagedAttn*)     */
  int32_t prefix_match;    /* 1: share matched prompt prefixes (PAKV); 0: every
                              sequence owns private copies (baseline B0 = PagedAttn)  */
  float scale;             /* softmax scale s; 0 -> 1/sqrt(d)           */
  int32_t device;          /* CUDA ordinal, or -1 for host-only mode                   */
  int64_t max_chunks;      /* pool capacity in chunks                                  */
  int64_t max_batch;       /* max live sequences                                       */
  int64_t max_seq_len;     /* max tokens per sequence                                  */
} chunkattn_config;

/* Caller-owned device memory (the library never calls cudaMalloc). */
typedef struct {
  void* k_pool;            /* device [L][max_chunks][h][c][d] dtype; chunk id = index.
                              Within a token row the 16-byte groups are stored
                              XOR-permuted by (slot % 8): logical group g of slot s
                              lives at group g ^ (s & 7) -- a (chunk, head) tile is
                              then bank-conflict free for ldmatrix after one 1-D
                              bulk copy                    */
  void* v_pool;            /* device, same layout as k_pool                            */
  void* workspace;         /* device, >= chunkattn_workspace_bytes(config) bytes,
                              16-byte aligned, ZERO-INITIALISED by the caller; holds
                              the context tables, the fp32 chunk-first partials
                              [slot][h][d + 4] (o, then m in log2 units, n) and the
                              seq-first split-item counters (kept zero between calls) */
  size_t workspace_bytes;
} chunkattn_buffers;

/* Bytes of device workspace the handle needs for `cfg` (0 on invalid cfg). */
size_t chunkattn_workspace_bytes(const chunkattn_config* cfg);

/* Create a handle.  Pools and workspace must outlive it.  The pool contents
 * need not be initialised (stale slots are masked by select). */
chunkattn_status chunkattn_create(const chunkattn_config* cfg, const chunkattn_buffers* buf,
                                  chunkattn_t* out);
chunkattn_status chunkattn_destroy(chunkattn_t h);

/* Prefix lookup without mutation ("prefix lookup to avoid repeated
 * computation of KV projection"): *matched = number of leading tokens covered
 * by full, aligned, matching chunks (a multiple of c).  tokens: host int32[n]. */
chunkattn_status chunkattn_match_prefix(chunkattn_t h, const int32_t* tokens, int64_t n,
                                        int64_t* matched);

/* New sequence joins (PAPER.md:507 scenario i): match the longest prefix of full
 * chunks, insert private chunks for the rest, copy their K/V into the pool.
 *   tokens        host int32[n], n >= 1
 *   k, v          device [n - kv_first_pos][L][h][d] dtype: K/V of positions
 *                 kv_first_pos..n-1 (rows for matched positions are skipped)
 *   kv_first_pos  0 <= kv_first_pos <= matched (call match_prefix first to
 *                 skip computing K/V for the matched prefix); CA_EINVAL if the
 *                 K/V rows do not cover every unmatched position
 *   *seq_id       new id (monotone 0, 1, 2, ...; never reused)
 *   *matched      matched token count */
chunkattn_status chunkattn_add_sequence(chunkattn_t h, const int32_t* tokens, int64_t n,
                                        const void* k, const void* v, int64_t kv_first_pos,
                                        void* stream, int64_t* seq_id, int64_t* matched);

/* One decode step for n sequences (PAPER.md:507 scenario iii: "append new
 * tokens into leaf chunks or grow a new chunk when the leaf chunk is full").
 * Processed in call order.  seq_ids host int64[n] (distinct, live); tokens
 * host int32[n]; k, v device [n][L][h][d] dtype in seq_ids order.  Must precede
 * the attend of the same step (the query attends to its own key). */
chunkattn_status chunkattn_append_kv(chunkattn_t h, int64_t n, const int64_t* seq_ids,
                                     const int32_t* tokens, const void* k, const void* v,
                                     void* stream);

/* Completed sequence leaves (PAPER.md:507 scenario ii): release the chunks its
 * path held alone (leaf -> root) to the LIFO free list.
 * *released = number of chunks released (may be NULL). */
chunkattn_status chunkattn_remove_sequence(chunkattn_t h, int64_t seq_id, int64_t* released);

/* Two-phase attention of one layer for ALL live sequences.
 *   seq_ids  host int64[n], n == live count, any order (CA_ESTATE otherwise)
 *   q        device [n][h][d] dtype, row k is the query of seq_ids[k]
 *   out      device [n][h][d] out_dtype, row k receives seq_ids[k]'s output
 * Asynchronous on `stream` (cudaStream_t; NULL = legacy default stream). */
chunkattn_status chunkattn_attend(chunkattn_t h, int32_t layer, int64_t n, const int64_t* seq_ids,
                                  const void* q, void* out, void* stream);

/* One decode step of one layer in ONE kernel launch (SURVEY §8 a4 + a5 + a6):
 * append one token per sequence (PAPER.md:507 scenario iii: "append new
 * tokens into leaf chunks or grow a new chunk when the leaf chunk is full")
 * and attend (Alg 1 + Alg 2 + Eqn 2) for ALL live sequences;
 * the query attends to its own new key (reading A8).
 *   layer    0 advances the tree by one token per sequence (lazy context
 *            rebuild and upload on a structural change); for
 *            num_layers > 1 call layers 1..L-1 of the same step after layer 0
 *            (they only scatter their K/V and attend; tokens is ignored)
 *   seq_ids  host int64[n], n == live count, distinct, any order
 *   tokens   host int32[n] (layer 0), the new token of seq_ids[k]
 *   k, v     device [n][h][d] dtype: THIS layer's new K/V rows, seq_ids order
 *   q        device [n][h][d] dtype;  out  device [n][h][d] out_dtype
 * On the K5 schedule (16-bit dtype, d in {64, 128}, c in {16, 32, 48, 64,
 * 96, 128}) the K/V scatter happens inside the attention
 * kernel; otherwise this call launches K1 for this layer and the persistent
 * attention kernels.  Errors before the launch leave the state unchanged.
 * Asynchronous on `stream`. */
chunkattn_status chunkattn_append_attend(chunkattn_t h, int32_t layer, int64_t n, const int64_t* seq_ids,
                                         const int32_t* tokens, const void* k, const void* v, const void* q,
                                         void* out, void* stream);

/* Prefill attention with prefix lookup (§2.2/§3.1):
 * after add_sequence matched a cached prefix and wrote the K/V of the rest,
 * every query position p >= first_pos[k] of sequence seq_ids[k] attends
 * causally over positions 0..p of that sequence in the pool (matched shared
 * chunks + its own):  out_p = softmax(s q_p K[0..p]^T) V[0..p]  (PAPER.md:344
 * per row, causal).  The projection of the matched prefix is never redone.
 *   seq_ids    host int64[n], live sequences (any subset, any order)
 *   first_pos  host int64[n], 0 <= first_pos[k] <= length (typically the
 *              matched length returned by add_sequence)
 *   q          device [Q][h][d] dtype, Q = sum(length - first_pos): the
 *              queries of seq_ids[0] (ascending positions), then seq_ids[1], ...
 *   out        device [Q][h][d] out_dtype, same order
 * Needs dtype F16/BF16, d in {64, 128}, c % 16 == 0 (CA_EDTYPE otherwise).
 * Asynchronous on `stream`; the pool must hold the K/V of every attended
 * position (stream order after add_sequence / append_kv). */
chunkattn_status chunkattn_prefill_attend(chunkattn_t h, int32_t layer, int64_t n, const int64_t* seq_ids,
                                          const int64_t* first_pos, const void* q, void* out, void* stream);

/* One whole decode step from HOST buffers (append_kv of the step's new K/V,
 * then attend of `layer`), with the host<->device copies inside the call:
 *   in_host   host (pinned for asynchrony) packed [q | k_new | v_new]:
 *             q [n][h][d] dtype, k_new and v_new [n][L][h][d] dtype, all in
 *             seq_ids order (the layouts of attend / append_kv)
 *   out_host  host [n][h][d] out_dtype (pinned for asynchrony)
 *   staging   device scratch, 16-byte aligned, >= in bytes + out bytes
 *             (caller-owned, as all device memory; must not be in use)
 * Enqueues one H2D copy, the append, the attend and one D2H copy on `stream`;
 * the output is in out_host once `stream` has passed the call.  Errors as
 * append_kv / attend; CA_EINVAL if staging_bytes is too small. */
chunkattn_status chunkattn_decode_step_host(chunkattn_t h, int32_t layer, int64_t n, const int64_t* seq_ids,
                                            const int32_t* tokens, const void* in_host, void* out_host,
                                            void* staging, size_t staging_bytes, void* stream);

/* Sequence ids in batch-row order (DFS of the prefix tree). */
chunkattn_status chunkattn_batch_order(chunkattn_t h, int64_t* seq_ids_out, int64_t cap,
                                       int64_t* n);

/* Canonical text of the tree and context (format in DESIGN.md §T5); *len is the
 * byte length without the trailing NUL.  CA_ERANGE if cap <= *len. */
chunkattn_status chunkattn_export_context(chunkattn_t h, char* buf, size_t cap, size_t* len);

/* out[6] = {chunks used, chunks free, chunks created, high-water mark,
 *           K+V bytes of used chunks (all layers), unused token slots}. */
chunkattn_status chunkattn_memory_stats(chunkattn_t h, int64_t out[6]);

/* out[6] = {context builds, H2D table uploads, H2D bytes uploaded,
 *           kernels launched, current epoch, partial slots of the context}. */
chunkattn_status chunkattn_counters(chunkattn_t h, int64_t out[6]);

/* Schedule of the current context (built by the last append / attend):
 * out[8] = {K5 cluster decode in use (0/1), K5 cluster size, K5 groups
 * (row blocks x head sets), K5 row blocks, K5 work units, K5 heads per
 * group, persistent fused schedule (0/1), persistent grid CTAs, K5 runs its
 * chunk-first units on tcgen05 (0/1)}. */
chunkattn_status chunkattn_schedule_info(chunkattn_t h, int64_t out[9]);

/* Tuning / test knobs (scheduling only; any setting gives the same result
 * within rounding, and a fixed setting is bitwise reproducible).  Unknown keys
 * fail with CA_EINVAL.
 *   "dk"               1 (default, auto) = the cluster decode kernel K5 (one
 *                      launch: append + both phases + the cluster merge) when
 *                      the shape allows and no shared run spans more rows than
 *                      one K5 row block; 2 = K5 whenever the shape allows; 0 =
 *                      the persistent-kernel paths below
 *   "dk_cs"            0 = auto (largest cluster with all (row block, head)
 *                      groups co-resident), else force the cluster size 1..16
 *   "dk_max_rows"      rows per K5 row block, 16..64 (default 64)
 *   "dk_hg"            0 = auto, else heads per K5 cluster group
 *   "dk_shared_fixed", "dk_shared_row", "dk_pack_fixed"  K5 work-split unit
 *                      costs (hundredths / thousandths; defaults 100, 10, 15)
 *   "dk_slots"         K5 tcgen05 variant: cap on its K + V ring slots (>= 4;
 *                      0 = default = as many as fit in shared memory).
 *                      DIAGNOSTIC bits (wrong outputs, timing studies only):
 *                      +64 2-D TMA also at d = 64, +128 every CTA returns at
 *                      entry (launch cost), +256 no private units, +512 no
 *                      UMMA issued, +1024 no softmax math, +2048 no P.V
 *                      UMMA, +4096 no S UMMA
 *   "dk_umma"          K5's chunk-first units on the tcgen05 tensor cores
 *                      (16-bit, d in {64, 128}, c = 64; S and O in TMEM, K/V
 *                      by 2-D TMA): 1 (default) when the step's chunk-first
 *                      units are at least "dk_umma_ratio" (hundredths, default
 *                      50) x its full private chunks, 2 always, 0 never (the
 *                      mma.sync consumers run them)
 *   "fused"            1 (default) = both phases in one persistent launch
 *                      (chunk-first units first in each CTA, last-contributor
 *                      merges); 0 = chunk-first kernel + seq-first kernel
 *   "cf_unit_cost"     fused balance: a chunk-first unit's weight in tenths of
 *                      a seq-first unit (default 16)
 *   "cf_splits"        0 = auto, else force chunks-per-split of chunk-first tiles
 *   "cf_target_ctas"   chunk-first CTA target for the auto split rule
 *   "cf_simt"          1 = force the SIMT chunk-first kernel (no tensor cores;
 *                      implies fused = 0)
 *   "sf_simt"          1 = SIMT seq-first consumers (implies fused = 0)
 *   "cf_umma"          1 (default) = tcgen05 chunk-first kernel in the two-kernel
 *                      path when supported (16-bit, d in {64, 128}, c = 64);
 *                      0 = the mma.sync kernel
 *   "cf_lane_merge"    1 (default) = the fused kernel merges its token lanes in
 *                      shared memory (one partial per row and job)
 *   "fused_tile_rows"  fused chunk-first tile rows, 16..64 (default 64)
 *   "sf_unit_fixed"    seq-first range split: fixed share of a unit's cost in
 *                      tenths (default 10 = plain unit counts; below 10 the rest
 *                      is proportional to the unit's valid tokens)
 *   "sf_item_cost"     ... plus this per item end, in tenths of a unit (default 0)
 *   "cf_small"         1 = 4-warp chunk-first CTA when tiles have <= 64 rows
 *                      (two-kernel path; default 0)
 *   "sf_ctas"          persistent grid size (default 296 = 2 per SM)
 *   "sf_ctas_per_sm"   1 or 2: shared-memory budget per seq-first CTA
 *   "sf_prefetch"      L2 bulk-prefetch distance in units (default 0 = off)
 *   "pdl"              1 (default) = programmatic dependent launch after the append
 *   "kernel_events"    1 = time every kernel launch (chunkattn_kernel_times)
 *   "trace"            debug timeline in the workspace tail (1 seq-first, 2 chunk-first)
 *   "diag_nocompute"   DIAGNOSTIC ONLY, outputs are wrong: consumers skip the math */
chunkattn_status chunkattn_set_option(chunkattn_t h, const char* key, int64_t value);

/* Per-kernel device time, measured with CUDA events recorded on the launch
 * stream around every kernel launch while the option "kernel_events" is 1
 * (PDL is not used between the two phases in that mode).  Synchronises on the
 * recorded events, accumulates, and resets the accumulators.
 *   ms[4]       total milliseconds of {append, chunk_first, seq_first, copy};
 *               "seq_first" = the attention kernel (persistent seq-first,
 *               fused, or the K5 cluster decode kernel)
 *   launches[4] launches of each kind that were timed */
chunkattn_status chunkattn_kernel_times(chunkattn_t h, double ms[4], int64_t launches[4]);

/* Copy the device-resident context tables (int32) to host memory `dst` (for
 * tests: they must equal the host-built tables).  *len = bytes. */
chunkattn_status chunkattn_download_tables(chunkattn_t h, void* dst, size_t cap, size_t* len,
                                           void* stream);

/* Copy the host-built context tables of the current epoch (the blob the
 * lazy upload copies) to `dst`; *len = bytes.  With
 * chunkattn_download_tables a test checks the upload byte for byte. */
chunkattn_status chunkattn_host_tables(chunkattn_t h, void* dst, size_t cap, size_t* len);

/* Message of the last error on this thread ("" if none). */
const char* chunkattn_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CHUNKATTN_H */
