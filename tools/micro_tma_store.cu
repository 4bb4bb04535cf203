// TMA store / load throughput per SM: one-warp CTAs stream 2-D boxes of a
// bf16 [rows][cols] tensor between smem and a 1 GiB global buffer.
// ./micro_tma_store  -> GB/s for box shapes x CTA counts, stores and loads.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2511_02168_b200/csrc/sm100.cuh"
using namespace tfb::sm100;

__global__ void __launch_bounds__(32) store_k(const __grid_constant__ CUtensorMap map, int box_c, int box_r,
                                              int cols, int rows, int iters, int inflight, int load) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x) return;
  const uint32_t bytes = box_c * box_r * 2;
  for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
  fence_mbar_init();
  const int ncb = cols / box_c, nrb = rows / box_r;
  uint32_t ph[8] = {0};
  for (int it = 0; it < iters; ++it) {
    const int b = (blockIdx.x + it * gridDim.x) % (ncb * nrb);
    const int c = (b % ncb) * box_c, r = (b / ncb) * box_r;
    const int s = it % 4;
    if (load) {
      if (it >= 4) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
      mbar_arrive_expect_tx(&bar[s], bytes);
      tma_load_2d(sm + s * bytes, &map, &bar[s], c, r);
    } else {
      tma_store_2d(&map, sm + s * bytes, c, r);
      bulk_commit();
      if (inflight == 1) bulk_wait_read<1>();
      else if (inflight == 2) bulk_wait_read<2>();
      else bulk_wait_read<3>();
    }
  }
  if (load) for (int s = 0; s < 4; ++s) if (iters > s) mbar_wait(&bar[s], ph[s]);
  else bulk_wait_all();
  bulk_wait_all();
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  const int cols = 8192, rows = 65536;  // 1 GiB bf16
  void* buf;
  cudaMalloc(&buf, size_t(cols) * rows * 2);
  cudaFuncSetAttribute(store_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int shapes[][3] = {{256, 64, 0}, {128, 128, 0}, {64, 128, 1}, {64, 256, 1}, {256, 16, 0}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& sh : shapes) {
    CUtensorMap map;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t str[1] = {cuuint64_t(cols) * 2};
    cuuint32_t box[2] = {cuuint32_t(sh[0]), cuuint32_t(sh[1])}, es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sh[2] ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", r); continue; }
    const int bytes = sh[0] * sh[1] * 2;
    for (int load = 0; load < 2; ++load)
      for (int ctas : {1, 16, 148})
        for (int inf : {1, 3}) {
          if (load && inf != 3) continue;
          const int iters = 2000;
          store_k<<<ctas, 32, 4 * bytes>>>(map, sh[0], sh[1], cols, rows, 20, inf, load);
          cudaEventRecord(e0);
          store_k<<<ctas, 32, 4 * bytes>>>(map, sh[0], sh[1], cols, rows, iters, inf, load);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          if (cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); continue; }
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          const double gbs = double(bytes) * iters * ctas / ms / 1e6;
          printf("%s box %3dx%3d%s ctas %3d inflight %d: %8.1f GB/s total, %6.1f GB/s per CTA\n",
                 load ? "load " : "store", sh[0], sh[1], sh[2] ? " sw128" : "      ", ctas, inf, gbs, gbs / ctas);
        }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
}
