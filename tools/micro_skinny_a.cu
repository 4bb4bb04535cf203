// micro_skinny_a.cu -- why are the skinny GEMM's A loads slow?  148 CTAs
// (one per SM) each stream `iters` 128-row x 64-column (16 KB, SWIZZLE_128B)
// boxes of a small bf16 A (rows x 8192, L2-resident) into a `stages`-deep
// smem ring, no compute -- the A side of a split-K / stream-K skinny GEMM
// where every CTA re-reads the same 2 MiB.
//   mode 0: row-major A [rows][8192], every CTA the same matrix
//   mode 1: panel-major A [128 kb][rows][64] (each box one contiguous 16 KB)
//   mode 2: row-major, every CTA its own private copy (no sharing)
//   mode 3: row-major, k-block order identical on every CTA (lockstep)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_skinny_a micro_skinny_a.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32) stream(const __grid_constant__ CUtensorMap map, int mode, int rows,
                                             int iters, int stages) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x != 0) return;
  const uint32_t box_bytes = 128 * rows;
  for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue = [&](int i) {
    const int s = i % stages;
    const int kb = mode == 3 ? (i % 128) : ((blockIdx.x * 13 + i) % 128);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(box_bytes)
                 : "memory");
    void* dst = smem + size_t(s) * box_bytes;
    if (mode == 1)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(su32(dst)), "l"(&map), "r"(0), "r"(0), "r"(kb), "r"(su32(&full[s]))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(dst)), "l"(&map), "r"(kb * 64), "r"(mode == 2 ? int(blockIdx.x) * rows : 0), "r"(su32(&full[s]))
          : "memory");
  };
  for (int i = 0; i < stages && i < iters; ++i) issue(i);
  for (int i = 0; i < iters; ++i) {
    const int s = i % stages;
    const uint32_t par = (i / stages) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&full[s])), "r"(par)
        : "memory");
    if (i + stages < iters) issue(i + stages);
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fp;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int C = 8192, iters = getenv("ITERS") ? atoi(getenv("ITERS")) : 28;
  void* buf;
  const size_t bytes = size_t(sms) * 128 * C * 2;  // room for mode 2's private copies
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rows : {128, 64})
    for (int stages : {4, 8})
      for (int mode = 0; mode < 4; ++mode) {
        if (stages * 128 * rows > 190 * 1024) continue;
        CUtensorMap m;
        CUresult r;
        const CUtensorMapL2promotion pr = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
        if (mode == 1) {
          cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(C / 64)};
          cuuint64_t str[2] = {128, (cuuint64_t)rows * 128};
          cuuint32_t box[3] = {64, (cuuint32_t)rows, 1}, es[3] = {1, 1, 1};
          r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
          cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)(mode == 2 ? sms * rows : rows)};
          cuuint64_t str[1] = {(cuuint64_t)C * 2};
          cuuint32_t box[2] = {64, (cuuint32_t)rows}, es[2] = {1, 1};
          r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return 1; }
        const size_t smem = size_t(stages) * 128 * rows + 1024;
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          cudaEventRecord(e0);
          stream<<<sms, 32, smem>>>(m, mode, rows, iters, stages);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        const double tot = double(sms) * iters * 128 * rows;
        printf("rows %3d stages %d mode %d: %7.1f us  %6.2f TB/s  %5.1f GB/s per SM  (%s)\n", rows, stages, mode,
               best * 1e3, tot / (best * 1e-3) / 1e12, tot / sms / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
