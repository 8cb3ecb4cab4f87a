// Cost of reading %globaltimer (the trace timestamps of tools/kernel_timeline.py)
// in SM cycles, and its update granularity.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/timer_probe tools/timer_probe.cu
#include <cstdio>
#include <cstdint>

__global__ void k(long long* out, unsigned long long* gt) {
  unsigned long long t, t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long c0 = clock64();
  unsigned long long acc = 0;
  for (int i = 0; i < 1000; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    acc += t;
  }
  long long c1 = clock64();
  out[0] = (c1 - c0);
  out[1] = (long long)acc;
  // granularity: smallest non-zero step between consecutive reads
  unsigned long long prev = t, minstep = ~0ull;
  for (int i = 0; i < 200000; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) {
      if (t - prev < minstep) minstep = t - prev;
      prev = t;
    }
  }
  gt[0] = minstep;
  gt[1] = t - t0;
}

int main() {
  long long* o;
  unsigned long long* g;
  cudaMalloc(&o, 16);
  cudaMalloc(&g, 16);
  k<<<1, 1>>>(o, g);
  k<<<1, 1>>>(o, g);
  cudaDeviceSynchronize();
  long long ho[2];
  unsigned long long hg[2];
  cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(hg, g, 16, cudaMemcpyDeviceToHost);
  printf("globaltimer read: %.1f SM cycles each; smallest observed step %llu ns (span %llu ns)\n", ho[0] / 1000.0,
         hg[0], hg[1]);
  return 0;
}
