// Device helpers for the sm_100a kernels: mbarrier + bulk/TMA async copies,
// ldmatrix + mma.sync fragments, fast exp2, vector conversions.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <map>
#include <mutex>
#include <utility>

#define CA_DEV __device__ __forceinline__

namespace pakv {
namespace dev {

// ------------------------------------------------------------------ misc ---
CA_DEV float fast_exp2(float x) {  // ex2.approx: exp2(-inf) = +0
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

CA_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Pool layout: a (chunk, head) tile is c rows (tokens) x d elements, row-major,
// with the 16-byte chunk index of every row XOR-ed by (token % 8).  A 1-D bulk
// copy of the tile therefore lands in shared memory already bank-conflict free
// for ldmatrix (8 consecutive tokens at one logical column hit 8 distinct
// 16-byte bank groups).  Physical 16-byte chunk of logical chunk j of token t:
CA_DEV int swz_chunk(int t, int j) { return j ^ (t & 7); }

// ------------------------------------------------------------- mbarrier ---
CA_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
CA_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
CA_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

CA_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

CA_DEV void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

CA_DEV uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

#ifdef CA_HANG_CHECK
// Debug builds: a wait that has not completed after 2 s reports where it is
// and traps (an error the host sees) instead of hanging the GPU.
#define CA_HANG_TRAP(what, a, b)                                                                                \
  do {                                                                                                         \
    printf("chunkattn hang: %s (%d, %d) block %d thread %d line %d\n", what, (int)(a), (int)(b), blockIdx.x,  \
           threadIdx.x, __LINE__);                                                                             \
    __trap();                                                                                                  \
  } while (0)
#endif

CA_DEV bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

CA_DEV void mbar_wait(uint64_t* bar, uint32_t phase) {
#ifdef CA_HANG_CHECK
  if (mbar_try_wait(bar, phase)) return;
  const uint64_t t0 = globaltimer_ns();
  while (!mbar_try_wait(bar, phase))
    if (globaltimer_ns() - t0 > 2000000000ull) CA_HANG_TRAP("mbarrier", (int)(smem_u32(bar) & 0xffff), phase);
#elif defined(CA_MBAR_CLOOP)
  while (!mbar_try_wait(bar, phase)) {
  }
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
#endif
}

// 1-D bulk copy global -> shared, completion on an mbarrier (UBLKCP in SASS).
// dst/src 16-byte aligned, bytes a multiple of 16.
CA_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Bulk prefetch global -> L2 (no shared memory, no completion): lets a kernel
// keep far more HBM bytes in flight than its shared-memory ring holds.
CA_DEV void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// 2-D TMA tile load global -> shared (UTMALDG in SASS).
CA_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// 3-D TMA tile load global -> shared (one op for both d-halves of a tile).
CA_DEV void tma_load_3d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
CA_DEV void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// GPU-scope release store / acquire load (cross-CTA readiness flags).
CA_DEV void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
CA_DEV uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
CA_DEV uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// GPU-scope acquire-release fence: after a CTA barrier, one thread's fence is
// cumulative over the writes the barrier ordered before it (release side), and
// orders its later reads after what it observed (acquire side).
CA_DEV void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Warp-cooperative spin: until every lane's flag (lanes with `mine`) equals
// tag.  Control flow stays warp-uniform (no lane spins while its siblings sit
// at a barrier).
CA_DEV void spin_flags_warp(const uint32_t* f, bool mine, uint32_t tag, int who) {
#ifdef CA_HANG_CHECK
  const uint64_t t0 = globaltimer_ns();
#endif
  for (;;) {
    // relaxed polls (an acquire load invalidates the SM's L1 every time, which
    // stalls the co-resident CTA's memory pipe); one acquire once it matched
    const bool ok = !mine || ld_relaxed_gpu(f) == tag;
    if (__all_sync(0xffffffffu, ok)) {
      if (mine) (void)ld_acquire_gpu(f);
      break;
    }
    __nanosleep(32);
#ifdef CA_HANG_CHECK
    if (globaltimer_ns() - t0 > 2000000000ull) CA_HANG_TRAP("flag", who, ok ? 1 : 0);
#else
    (void)who;
#endif
  }
}

// PDL: let the dependent grid launch / wait for the primary grid.
CA_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
CA_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace dev

// Allow `smem` bytes of dynamic shared memory (and the max carveout) for a
// kernel, once per (kernel, device) and size: cudaFuncSetAttribute costs host
// microseconds per call, paid on every decode step otherwise.
inline cudaError_t set_smem_once(const void* kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({kern, dev});
  if (it != done.end() && it->second >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) done[{kern, dev}] = smem;
  return e;
}

// Launch `kern` on `st`; with pdl the launch may begin before the previous
// kernel in the stream finishes (programmatic dependent launch): the kernel
// must griddepcontrol.wait before touching anything that kernel writes.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

namespace dev {

// ----------------------------------------------------------- mma.sync -----
CA_DEV void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
CA_DEV void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

template <typename T>
struct Mma;
template <>
struct Mma<__half> {
  static CA_DEV void run(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  static CA_DEV uint32_t pack(float lo, float hi) {
    __half2 v = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  static CA_DEV float2 unpack(uint32_t u) { return __half22float2(*reinterpret_cast<__half2*>(&u)); }
};
template <>
struct Mma<__nv_bfloat16> {
  static CA_DEV void run(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  static CA_DEV uint32_t pack(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  static CA_DEV float2 unpack(uint32_t u) { return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u)); }
};

// --------------------------------------------------- element conversions ---
template <typename T>
struct Elem;
template <>
struct Elem<float> {
  static constexpr int kVec = 4;  // elements per 16 bytes
  static CA_DEV void to_float(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z);
    f[3] = __uint_as_float(u.w);
  }
  static CA_DEV float load1(const float* p) { return *p; }
  static CA_DEV void store1(float* p, float v) { *p = v; }
};
template <>
struct Elem<__half> {
  static constexpr int kVec = 8;
  static CA_DEV void to_float(const uint4& u, float* f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  static CA_DEV float load1(const __half* p) { return __half2float(*p); }
  static CA_DEV void store1(__half* p, float v) { *p = __float2half_rn(v); }
};
template <>
struct Elem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  static CA_DEV void to_float(const uint4& u, float* f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  static CA_DEV float load1(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  static CA_DEV void store1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

}  // namespace dev
}  // namespace pakv
