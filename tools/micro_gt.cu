#include <cstdio>
#include <cstdint>
__global__ void k(unsigned long long* out) {
  unsigned long long g0, g1, c0, c1, acc = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  c0 = clock64();
  for (int i = 0; i < 100; ++i) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    acc += g;
  }
  c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  // distinct values seen in a tight loop -> resolution
  unsigned long long prev = 0, changes = 0, t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < 20000; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { ++changes; prev = t; }
  }
  out[0] = c1 - c0; out[1] = g1 - g0; out[2] = acc; out[3] = changes; out[4] = t - t0;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  for (int r = 0; r < 3; ++r) {
    k<<<1, 1>>>(d);
    unsigned long long h[5]; cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
    printf("100 globaltimer reads: %llu cycles, %llu ns; 20000-read loop: %llu distinct values over %llu ns\n", h[0], h[1], h[3], h[4]);
  }
}
