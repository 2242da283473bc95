// Microbenchmark: how long does __nanosleep(t) sleep on this GPU (one warp
// alone on an SM, and with 16 busy warps on the same SM)?
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(uint32_t ns, int iters, uint64_t* out, int busy) {
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    uint64_t t0 = gt();
    for (int i = 0; i < iters; ++i) __nanosleep(ns);
    uint64_t t1 = gt();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  } else if (busy) {
    uint32_t x = threadIdx.x;
    for (int i = 0; i < iters * 64; ++i) x = x * 1664525u + 1013904223u;
    if (x == 7) out[1000] = x;
  }
}
int main() {
  uint64_t* d; cudaMalloc(&d, 8 * 2048);
  uint64_t h[4];
  for (int busy = 0; busy < 2; ++busy)
    for (uint32_t ns : {0u, 32u, 128u, 512u, 1000u, 2000u, 5000u, 20000u}) {
      k<<<1, busy ? 640 : 32>>>(ns, 200, d, busy);
      cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      printf("busy=%d nanosleep(%u) -> %llu ns per call\n", busy, ns, (unsigned long long)h[0]);
    }
  return 0;
}
