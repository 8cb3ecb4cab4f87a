// Probe of the tcgen05.ld .16x256b register layout (the K5 tcgen05 softmax
// reads S / O in this shape so that 4 threads share a row, as in the mma.sync
// accumulator fragment).  TMEM is filled with value(lane, col) = lane * 1000 +
// col through the known .32x32b shape (thread t <-> lane t, register i <->
// column i), then read back with .16x256b.x2 at lane offsets 0 and 16; the
// decoded (lane, col) of every register of a few threads is printed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_layout_probe tools/tmem_layout_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(int* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase;
  const uint32_t lanebase = (uint32_t)(warp * 32) << 16;
  // fill: 2 x 32 columns
  for (int c0 = 0; c0 < 64; c0 += 32) {
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = (uint32_t)((warp * 32 + lane) * 1000 + c0 + i);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(t + lanebase + c0),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  // read back: .16x256b.x2 at lane offsets 0 and 16, column 8
  for (int lo = 0; lo < 32; lo += 16) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(t + ((uint32_t)(warp * 32 + lo) << 16) + 8));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) out[((warp * 2 + lo / 16) * 32 + lane) * 8 + i] = (int)v[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(t));
}

int main() {
  int* d;
  cudaMalloc(&d, 4 * 2 * 32 * 8 * sizeof(int));
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  static int h[4 * 2 * 32 * 8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int w = 0; w < 4; w += 3)
    for (int lo = 0; lo < 2; ++lo)
      for (int th = 0; th < 32; th += (th < 8 ? 1 : 7)) {
        printf("warp %d laneoff %2d thread %2d:", w, lo * 16, th);
        for (int i = 0; i < 8; ++i) {
          const int v = h[((w * 2 + lo) * 32 + th) * 8 + i];
          printf(" (%d,%d)", v / 1000, v % 1000);
        }
        printf("\n");
      }
  return 0;
}
