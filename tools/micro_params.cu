// micro_params.cu -- launch-to-launch cost vs kernel parameter size: N
// back-to-back launches of a 296-CTA kernel that does ~nothing, with a
// 64 B or a 4 KB __grid_constant__ parameter struct (the Flash Decode
// kernel's FdParams is ~3.9 KB), and a ~50 us spin kernel between.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_params micro_params.cu
#include <cuda_runtime.h>
#include <cstdio>

struct Small { unsigned long long a[8]; };
struct Big { unsigned long long a[500]; };

template <class P>
__global__ void k(const __grid_constant__ P p, unsigned long long spin_ns, int* sink) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < spin_ns);
  if (p.a[0] == 12345 && threadIdx.x == 0) *sink = 1;
}

int main() {
  int* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  Small s{};
  Big b{};
  for (unsigned long long spin : {0ull, 50000ull}) {
    for (int which = 0; which < 2; ++which) {
      const int n = 200;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        for (int i = 0; i < n; ++i) {
          if (which) k<Big><<<296, 256>>>(b, spin, sink);
          else k<Small><<<296, 256>>>(s, spin, sink);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("spin %5llu ns params %4zu B: %.2f us per launch (%s)\n", spin, which ? sizeof(Big) : sizeof(Small),
             ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
