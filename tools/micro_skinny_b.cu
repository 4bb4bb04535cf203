// micro_skinny_b.cu -- the B side of the skinny stream-K GEMM alone: 148
// CTAs (one per SM) stream a 8192 x 8192 bf16 row-major B (128 MiB, from
// HBM) as the GEMM does: units (256-column tile, 64-row k-block), CTA c
// takes units [c*U/148, (c+1)*U/148), one TMA issue thread, `stages` ring.
//   box 0: one 4-D box per unit (64 cols x 64 rows x 4 chunks = 32 KB)
//   box 1: four 2-D boxes (64 cols x 64 rows = 8 KB each)
//   box 2: one 2-D box of 64 cols x 256 rows (32 KB; a 64-column tile, 4 k-blocks)
//   box 3: 4-D box with 128 rows (64 KB per unit, half the units)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_skinny_b micro_skinny_b.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32) stream(const __grid_constant__ CUtensorMap m4, const __grid_constant__ CUtensorMap m2,
                                             int box, int stages, int kbt, int tiles, int evict) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x != 0) return;
  const uint32_t bytes = box == 3 ? 65536 : 32768;
  for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long long U = (long long)tiles * kbt;
  const int u0 = int(U * blockIdx.x / gridDim.x), u1 = int(U * (blockIdx.x + 1) / gridDim.x);
  const int n = u1 - u0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int i) {
    const int s = i % stages;
    const int u = u0 + i;
    const int T = u / kbt, kb = u % kbt;
    uint8_t* dst = smem + size_t(s) * bytes;
    const uint32_t bar = su32(&full[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    if (box == 0 || box == 3) {
      if (evict)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(su32(dst)),
            "l"(&m4), "r"(0), "r"(kb * (box == 3 ? 128 : 64)), "r"(0), "r"(T), "r"(bar), "l"(pol) : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(su32(dst)),
            "l"(&m4), "r"(0), "r"(kb * (box == 3 ? 128 : 64)), "r"(0), "r"(T), "r"(bar) : "memory");
    } else if (box == 1) {
      for (int c = 0; c < 4; ++c)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(dst + c * 8192)), "l"(&m2), "r"(T * 256 + c * 64), "r"(kb * 64), "r"(bar) : "memory");
    } else {
      // 64-column tiles, 256-row k-blocks: unit (T, kb) -> column chunk T*4 + kb%4, rows (kb/4)*256
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(dst)), "l"(&m2), "r"((T * 4 + kb % 4) * 64), "r"((kb / 4) * 256), "r"(bar) : "memory");
    }
  };
  for (int i = 0; i < stages && i < n; ++i) issue(i);
  for (int i = 0; i < n; ++i) {
    const int s = i % stages;
    const uint32_t par = (i / stages) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&full[s])), "r"(par) : "memory");
    if (i + stages < n) issue(i + stages);
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
  const int N = 8192, K = 8192;
  void *buf, *flush;
  cudaMalloc(&buf, size_t(N) * K * 2);
  cudaMemset(buf, 1, size_t(N) * K * 2);
  cudaMalloc(&flush, size_t(256) << 20);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int promo : {3, 0}) {
  CUtensorMap m4, m4b, m2;
  const CUtensorMapL2promotion pr = promo == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  {
    cuuint64_t dims[4] = {64, (cuuint64_t)K, 4, (cuuint64_t)N / 256};
    cuuint64_t str[3] = {(cuuint64_t)N * 2, 128, 512};
    cuuint32_t bx[4] = {64, 64, 4, 1}, es[4] = {1, 1, 1, 1};
    enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint32_t bx2[4] = {64, 128, 4, 1};
    enc(&m4b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, str, bx2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  for (int box = 0; box < 4; ++box)
    for (int stages : {3, 4, 6})
      for (int evict : {0, 1}) {
        if (evict && box != 0) continue;
        if (box == 3 && stages > 3) continue;
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
        cuuint64_t str[1] = {(cuuint64_t)N * 2};
        cuuint32_t bx[2] = {64, box == 2 ? 256u : 64u}, es[2] = {1, 1};
        enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int kbt = box == 3 ? 64 : 128;
        const size_t smem = size_t(stages) * (box == 3 ? 65536 : 32768) + 1024;
        float best = 1e9, sum = 0;
        for (int rep = 0; rep < 6; ++rep) {
          if (getenv("FLUSH")) cudaMemset(flush, rep, size_t(256) << 20);  // evict B from L2 (leaves dirty lines)
          cudaEventRecord(e0);
          stream<<<sms, 32, smem>>>(box == 3 ? m4b : m4, m2, box, stages, kbt, 32, evict);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
          if (rep) sum += ms;
        }
        const double tot = double(N) * K * 2;
        printf("promo %d box %d stages %d evict %d: best %6.1f us mean %6.1f  %5.2f TB/s (%s)\n", promo, box, stages, evict,
               best * 1e3, sum / 5 * 1e3, tot / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
