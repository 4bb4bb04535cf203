// micro_dsmem.cu -- DSMEM bandwidth for the split-K reduction: a cluster of S
// CTAs, each holding a 128 x 256 fp32 partial (128 KB) in smem; CTA s owns
// rows [s*128/S, (s+1)*128/S).
//   mode 0 (pull, what ag_sm100.cu does): every thread ld.shared::cluster's
//          the owned rows from all S siblings (2*S 16-byte loads in flight).
//   mode 1 (bulk push): each CTA copies the S-1 slices it does not own to
//          their owners with cp.async.bulk.shared::cluster.shared::cta (the
//          TMA engine, one instruction per slice) and the owner waits on an
//          mbarrier for (S-1) slices of bytes, then sums locally.
// Reports cycles per reduction (clock64 on CTA 0, cluster-synced both sides).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_dsmem micro_dsmem.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int ROWS = 128, COLS = 256, PART = ROWS * COLS * 4;  // 128 KB

__global__ void __launch_bounds__(320, 1) reduce(int S, int mode, int iters, float* out, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  float* R = reinterpret_cast<float*>(smem);                  // own partial, 128 KB
  uint8_t* slots = smem + PART;                               // mode 1: S-1 received slices
  const uint32_t r = ctarank();
  const int rows_per = ROWS / S, slice = rows_per * COLS * 4;
  for (int i = threadIdx.x; i < ROWS * COLS; i += blockDim.x) R[i] = float(r + 1) * 0.5f + float(i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  csync();
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      const int tasks = rows_per * 32;
      for (int e = threadIdx.x; e < tasks; e += blockDim.x) {
        const int rl = int(r) * rows_per + e / 32, g = e % 32;
        const uint32_t off = su32(R) + uint32_t(rl * 1024 + g * 32);
        float4 x[8], y[8];
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < S) {
            const uint32_t a = mapa(off, uint32_t(s));
            asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(x[s].x), "=f"(x[s].y), "=f"(x[s].z), "=f"(x[s].w) : "r"(a));
            asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(y[s].x), "=f"(y[s].y), "=f"(y[s].z), "=f"(y[s].w) : "r"(a + 16));
          }
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < S) acc += x[s].x + x[s].y + x[s].z + x[s].w + y[s].x + y[s].y + y[s].z + y[s].w;
      }
    } else {
      const uint32_t par = uint32_t(it & 1);
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                     "r"(uint32_t(slice * (S - 1)))
                     : "memory");
      }
      csync();  // every owner armed before any push lands
      if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
          if (s == int(r)) continue;
          // my slice s -> owner s, into its slot for sender r (slot index skips the owner itself)
          const int slot = int(r) < s ? int(r) : int(r) - 1;
          const uint32_t dst = mapa(su32(slots + slot * slice), uint32_t(s));
          const uint32_t mb = mapa(su32(&bar), uint32_t(s));
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  dst),
              "r"(su32(R) + uint32_t(s * slice)), "r"(uint32_t(slice)), "r"(mb)
              : "memory");
        }
      }
      asm volatile(
          "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
              su32(&bar)),
          "r"(par)
          : "memory");
      const float* own = R + size_t(r) * rows_per * COLS;
      for (int i = threadIdx.x * 4; i < rows_per * COLS; i += blockDim.x * 4) {
        float4 v = *reinterpret_cast<const float4*>(own + i);
        float a4 = v.x + v.y + v.z + v.w;
        for (int s = 0; s < S - 1; ++s) {
          float4 w = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(slots + s * slice) + i);
          a4 += w.x + w.y + w.z + w.w;
        }
        acc += a4;
      }
    }
    csync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / iters;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 320 * 4);
  cudaMalloc(&cyc, 8);
  for (int S : {2, 4, 8}) {
    for (int mode = 0; mode < 2; ++mode) {
      const size_t smem = PART + (mode ? size_t(PART / S) * (S - 1) : 0);
      if (smem > 227 * 1024) { printf("S=%d mode %d: smem %zu too big\n", S, mode, smem); continue; }
      cudaFuncSetAttribute(reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      cudaFuncSetAttribute(reduce, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((148 / S) * S);
      cfg.blockDim = dim3(320);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = S;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, reduce, S, mode, 20, out, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double remote = double(PART / S) * (S - 1);
      printf("S=%d %-9s: %6lld cycles per reduction, %.1f remote B/clk per CTA (%s)\n", S,
             mode ? "bulk-push" : "pull", c, remote / double(c), cudaGetErrorString(e));
    }
  }
  return 0;
}
