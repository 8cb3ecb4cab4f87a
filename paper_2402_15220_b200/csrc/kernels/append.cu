// K1 append_kv: "At each decoding iteration, we append new tokens
// into leaf chunks" — scatter each sequence's new K/V row into slot
// seq_len - start_pos of its leaf chunk and bump the device-resident seq_len
// (so steps that do not change the tree upload nothing: lazy context copy,
// PAPER.md:162).  Plus the prefill copy of a new sequence's private chunks.
// Pure data movement: 16-byte vector loads/stores, one CTA per appended row.
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace pakv {

namespace {

constexpr int kThreads = 128;

template <int NI>
struct AppendList {
  AppendItem it[NI];
};

// One thread per 16-byte vector of the step's new K (and V): fully parallel,
// no dependent loads (the scatter list arrives as kernel parameters, sized to
// the batch so small steps do not pay for a large parameter block).
template <int NI>
__global__ void __launch_bounds__(kThreads) append_kv_kernel(uint4* __restrict__ kpool, uint4* __restrict__ vpool,
                                                             const uint4* __restrict__ knew,
                                                             const uint4* __restrict__ vnew,
                                                             const __grid_constant__ AppendList<NI> list, int32_t n,
                                                             int32_t* __restrict__ seq_len, int64_t layer_stride_v,
                                                             int32_t L, int32_t h, int32_t c, int32_t dv) {
  dev::pdl_launch_dependents();  // chunk-first reads only shared chunks: it may start now
  const int per_layer = h * dv;  // 16-byte vectors per layer of one token
  const int total = L * per_layer;
  const int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (e >= (int64_t)n * total) return;
  const int i = (int)(e / total);
  const int r0 = (int)(e - (int64_t)i * total);
  const int l = r0 / per_layer;
  const int r = r0 - l * per_layer;
  const int hh = r / dv;
  const int x = r - hh * dv;
  const AppendItem it = list.it[i];
  const int64_t dst = l * layer_stride_v + ((int64_t)(it.chunk * h + hh) * c + it.slot) * dv + dev::swz_chunk(it.slot, x);
  kpool[dst] = knew[e];
  vpool[dst] = vnew[e];
  if (r0 == 0) seq_len[it.row] = it.new_len;
}

struct ChunkList {
  int32_t ids[256];
};

__global__ void __launch_bounds__(kThreads) copy_rows_kernel(uint4* __restrict__ kpool, uint4* __restrict__ vpool,
                                                             const uint4* __restrict__ ksrc,
                                                             const uint4* __restrict__ vsrc, ChunkList list,
                                                             int64_t first_pos, int64_t layer_stride_v, int32_t L,
                                                             int32_t h, int32_t c, int32_t dv) {
  const int64_t i = blockIdx.x;  // source row
  const int64_t pos = first_pos + i;
  const int chunk = list.ids[pos / c - first_pos / c];
  const int slot = (int)(pos % c);
  const int per_layer = h * dv;
  const int total = L * per_layer;
  for (int e = threadIdx.x; e < total; e += kThreads) {
    const int l = e / per_layer;
    const int r = e - l * per_layer;
    const int hh = r / dv;
    const int x = r - hh * dv;
    const int64_t dst = l * layer_stride_v + ((int64_t)(chunk * h + hh) * c + slot) * dv + dev::swz_chunk(slot, x);
    const int64_t src = i * total + e;
    kpool[dst] = ksrc[src];
    vpool[dst] = vsrc[src];
  }
}

}  // namespace

cudaError_t launch_append_kv(const PoolGeom& p, const DevTables& t, const AppendItem* items, int32_t n,
                             const void* k, const void* v, cudaStream_t st) {
  const int E = dtype_bytes(p.dtype);
  const int dv = p.d * E / 16;
  const int64_t total = (int64_t)p.num_layers * p.h * dv;
  auto run = [&](auto tag, int32_t i0, int32_t m) {
    constexpr int NI = decltype(tag)::value;
    thread_local AppendList<NI> list;  // host staging of the parameter block
    std::copy(items + i0, items + i0 + m, list.it);
    const int64_t vecs = (int64_t)m * total;
    append_kv_kernel<NI><<<(unsigned)((vecs + kThreads - 1) / kThreads), kThreads, 0, st>>>(
        (uint4*)p.k, (uint4*)p.v, (const uint4*)k + i0 * total, (const uint4*)v + i0 * total, list, m, t.seq_len,
        p.layer_stride * E / 16, p.num_layers, p.h, p.c, dv);
    return cudaGetLastError();
  };
  for (int32_t i0 = 0; i0 < n; i0 += kMaxAppendItems) {
    const int32_t m = std::min<int32_t>(kMaxAppendItems, n - i0);
    cudaError_t e;
    if (m <= 32) e = run(std::integral_constant<int, 32>{}, i0, m);
    else if (m <= 256) e = run(std::integral_constant<int, 256>{}, i0, m);
    else e = run(std::integral_constant<int, kMaxAppendItems>{}, i0, m);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_copy_rows(const PoolGeom& p, const int32_t* chunks, int32_t n_chunks, int64_t first_pos,
                             int64_t m, const void* k, const void* v, cudaStream_t st) {
  const int E = dtype_bytes(p.dtype);
  const int dv = p.d * E / 16;
  const int64_t row_vecs = (int64_t)p.num_layers * p.h * dv;
  // launch in pieces of <= 256 chunks (the chunk list travels as a kernel parameter)
  int64_t done = 0;
  int32_t ci = 0;
  while (done < m) {
    const int64_t pos = first_pos + done;
    const int64_t chunk_end_pos = (pos / p.c + 256) * (int64_t)p.c;  // exclusive
    const int64_t rows = std::min<int64_t>(m - done, chunk_end_pos - pos);
    ChunkList list;
    const int32_t cnt = (int32_t)std::min<int64_t>(256, n_chunks - ci);
    for (int32_t q = 0; q < cnt; ++q) list.ids[q] = chunks[ci + q];
    copy_rows_kernel<<<(unsigned)rows, kThreads, 0, st>>>(
        (uint4*)p.k, (uint4*)p.v, (const uint4*)k + done * row_vecs, (const uint4*)v + done * row_vecs, list, pos,
        p.layer_stride * E / 16, p.num_layers, p.h, p.c, dv);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    done += rows;
    ci += 256;
  }
  return cudaSuccess;
}

}  // namespace pakv
