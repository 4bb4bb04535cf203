// micro_cluster.cu -- cross-CTA signalling latency inside a 2-CTA cluster.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_cluster micro_cluster.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(smem_u32(p)), "r"(r)); return o; }
__device__ __forceinline__ void arrive_remote(uint32_t a) { asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(a) : "memory"); }
__device__ __forceinline__ void wait_test(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" :: "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void wait_try(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" :: "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// mode 0: ping-pong remote arrive + test_wait; mode 1: + try_wait;
// mode 2: tcgen05.commit.cta_group::2 multicast from CTA0, CTA1 arrives back.
__global__ void __cluster_dims__(2, 1, 1) pingpong(int iters, int mode, long long* out) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t r = ctarank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (mode == 2 && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  __syncthreads();
  csync();
  const uint32_t peer_bar = mapa(&bar, r ^ 1);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const uint32_t ph = i & 1;
      if (r == 0) {
        if (mode == 2) {
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                       :: "r"(smem_u32(&bar)), "h"((uint16_t)2) : "memory");
        } else {
          arrive_remote(peer_bar);
        }
        if (mode == 1) wait_try(&bar, ph); else wait_test(&bar, ph);
      } else {
        if (mode == 1) wait_try(&bar, ph); else wait_test(&bar, ph);
        arrive_remote(peer_bar);
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  csync();
  if (mode == 2 && threadIdx.x < 32) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 32;" :: "r"(tslot));
  }
  if (threadIdx.x == 0 && r == 0) *out = (t1 - t0) / iters;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int mode = 0; mode < 3; ++mode) {
    pingpong<<<2, 128>>>(10000, mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = -1;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %lld cycles per round trip (%s)\n", mode, h, cudaGetErrorString(e));
  }
  return 0;
}
