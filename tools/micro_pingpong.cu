// micro_pingpong.cu -- floor of the GEMM's producer/MMA mbarrier ring with no
// data: warp 0 lane 0 waits empty[s] and arrives on full[s]; warp 1 lane 0
// waits full[s] and releases empty[s] (plain arrive, or tcgen05.commit with
// no MMA in flight).  4 stages, 148 CTAs, `iters` k-blocks; ns per k-block.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_pingpong micro_pingpong.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par, int hint) {
  if (hint)
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par), "r"(100000u) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

__global__ void pp(int iters, int mode, int hint, int nthreads_extra, unsigned long long* out) {
  __shared__ __align__(8) uint64_t full[4], empty[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (mode == 1 && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i & 3;
      wait(&empty[s], ((i >> 2) & 1) ^ 1, hint);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 0;" ::"r"(su32(&full[s])) : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i & 3;
      wait(&full[s], (i >> 2) & 1, hint);
      if (mode == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[s])) : "memory");
      else
        arrive(&empty[s]);
    }
  }
  __syncthreads();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (mode == 1 && warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot) : "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  for (int threads : {64, 320})
    for (int mode = 0; mode < 2; ++mode)
      for (int hint = 0; hint < 2; ++hint) {
        unsigned long long ns = 0;
        for (int rep = 0; rep < 3; ++rep) {
          pp<<<148, threads>>>(4096, mode, hint, 0, d);
          cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        }
        printf("threads %3d %s hint %d: %.1f ns per k-block (%s)\n", threads, mode ? "tcgen05.commit" : "arrive       ",
               hint, ns / 4096.0, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
