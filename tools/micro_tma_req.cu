// micro_tma_req.cu -- does the global-memory layout behind a TMA box change
// the L2->SM ingress rate?  Every CTA streams 128B-swizzled 64-column boxes of
// a bf16 matrix into an smem ring (no compute) with `stages` loads in flight.
//   layout 0: row-major [R][C] (C = 8192), 2D map, box (64, rows): each box
//             row is a separate 128 B piece of global memory (stride C*2).
//   layout 1: panel-major [C/64][R][64], 3D map, box (64, rows, 1): the box's
//             rows are back to back in global memory (one contiguous span).
// Same smem image, same MMA descriptor either way; only the TMA request
// stream differs.  Buffer sizes: 32 MiB (L2-resident) and 1 GiB (HBM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_tma_req micro_tma_req.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstdlib>

static bool layout_only_panel_skip(int rows, int pan) { return rows * pan > 512; }
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128) stream(const __grid_constant__ CUtensorMap map, int layout, int rows,
                                             int ntiles_r, int ntiles_c, int iters, int stages, int pan) {
  extern __shared__ __align__(1024) uint8_t smem_all[];
  __shared__ __align__(8) uint64_t full_all[4][16];
  const uint32_t box_bytes = 64 * 2 * rows * pan;
  if (threadIdx.x % 32 != 0) return;
  const int wi = threadIdx.x / 32, nw = blockDim.x / 32;
  uint64_t* full = full_all[wi];
  uint8_t* smem = smem_all + size_t(wi) * stages * box_bytes;
  const int vblock = blockIdx.x * nw + wi, vgrid = gridDim.x * nw;
  for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue = [&](int i) {
    const int s = i % stages;
    const int t = (vblock + i * vgrid) % (ntiles_r * ntiles_c);
    const int tr = t % ntiles_r, tc = t / ntiles_r;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(box_bytes)
                 : "memory");
    void* dst = smem + size_t(s) * box_bytes;
    if (layout == 0 && pan == 1)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(dst)),
          "l"(&map), "r"(tc * 64), "r"(tr * rows), "r"(su32(&full[s]))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(su32(dst)),
          "l"(&map), "r"(0), "r"(tr * rows), "r"(tc * pan), "r"(su32(&full[s]))
          : "memory");
  };
  for (int i = 0; i < stages && i < iters; ++i) issue(i);
  for (int i = 0; i < iters; ++i) {
    const int s = i % stages;
    const uint32_t par = (i / stages) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&full[s])),
        "r"(par)
        : "memory");
    if (i + stages < iters) issue(i + stages);
  }
}


// Multicast: a cluster of CL CTAs shares every box; CTA r fetches rows
// [r*rows/CL, (r+1)*rows/CL) and multicasts them to all CL CTAs, so each L2
// read lands in CL SMs.  empty[s] (count CL) gates stage reuse cluster-wide.
__global__ void __launch_bounds__(32) stream_mc(const __grid_constant__ CUtensorMap map, int rows, int ntiles_r,
                                                int ntiles_c, int iters, int stages, int CL) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const uint32_t box_bytes = 64 * 2 * rows;
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(CL));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
  const uint16_t mask = uint16_t((1u << CL) - 1);
  const int part = rows / CL;
  auto issue = [&](int i) {
    const int s = i % stages;
    if (i >= stages) {
      const uint32_t par = ((i / stages) - 1) & 1;
      asm volatile(
          "{\n.reg .pred p;\nE_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra E_%=;\n}\n" ::"r"(
              su32(&empty[s])),
          "r"(par)
          : "memory");
    }
    const int t = (cid + i * ncl) % (ntiles_r * ntiles_c);
    const int tr = t % ntiles_r, tc = t / ntiles_r;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(box_bytes)
                 : "memory");
    uint8_t* dst = smem + size_t(s) * box_bytes + size_t(r) * part * 128;
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
        "{%2, %3}], [%4], %5;" ::"r"(su32(dst)),
        "l"(&map), "r"(tc * 64), "r"(tr * rows + int(r) * part), "r"(su32(&full[s])), "h"(mask)
        : "memory");
  };
  for (int i = 0; i < stages && i < iters; ++i) issue(i);
  for (int i = 0; i < iters; ++i) {
    const int s = i % stages;
    const uint32_t par = (i / stages) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&full[s])),
        "r"(par)
        : "memory");
    for (int c = 0; c < CL; ++c) {
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(su32(&empty[s])), "r"(c));
      asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
    }
    if (i + stages < iters) issue(i + stages);
  }
  }
  __syncwarp();
  // drain: peers may still arrive on our empty barriers
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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
  const int C = 8192;
  if (getenv("TMA_WARPS")) {  // issuing warps per CTA: 1 CTA/SM, each warp its own ring
    const size_t bytes = size_t(32) << 20;
    const int R = int(bytes / (C * 2));
    void* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    for (int rows : {64, 128}) {
      CUtensorMap map;
      cuuint64_t dims[2] = {cuuint64_t(C), cuuint64_t(R)}, str[1] = {cuuint64_t(C) * 2};
      cuuint32_t box[2] = {64, cuuint32_t(rows)}, es[2] = {1, 1};
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int nw : {1, 2, 4}) {
        const int stages = 8 / nw;
        const size_t smem = size_t(nw) * stages * 128 * rows;
        const int ntr = R / rows, ntc = C / 64;
        const int iters = 400 / nw;
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        stream<<<sms, 32 * nw, smem>>>(map, 0, rows, ntr, ntc, iters, stages, 1);
        cudaEventRecord(e0);
        stream<<<sms, 32 * nw, smem>>>(map, 0, rows, ntr, ntc, iters, stages, 1);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double moved = double(iters) * nw * sms * 128 * rows;
        printf("warps %d box %3d rows (%2d KB) stages/warp %d: %7.1f GB/s, %5.1f per SM (%s)\n", nw, rows,
               rows * 128 / 1024, stages, moved / ms / 1e6, moved / ms / 1e6 / sms,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
    return 0;
  }
  {  // multicast sweep, L2-resident 32 MiB
    const size_t bytes = size_t(32) << 20;
    const int R = int(bytes / (C * 2));
    void* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    for (int rows : {128, 256}) {
      CUtensorMap map;
      for (int CL : {1, 2, 4}) {
        cuuint64_t dims[2] = {cuuint64_t(C), cuuint64_t(R)}, str[1] = {cuuint64_t(C) * 2};
        cuuint32_t box[2] = {64, cuuint32_t(rows / CL)}, es[2] = {1, 1};
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int stages : {3, 4, 6}) {
          const size_t smem = size_t(stages) * 128 * rows;
          if (smem > 200 * 1024) continue;
          const int ntr = R / rows, ntc = C / 64;
          const int grid = (sms / CL) * CL;
          const int iters = 400;
          cudaFuncSetAttribute(stream_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(grid);
          cfg.blockDim = dim3(32);
          cfg.dynamicSmemBytes = smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = CL;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          cudaLaunchKernelEx(&cfg, stream_mc, map, rows, ntr, ntc, iters, stages, CL);
          cudaEventRecord(e0);
          cudaLaunchKernelEx(&cfg, stream_mc, map, rows, ntr, ntc, iters, stages, CL);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double landed = double(iters) * grid * 128 * rows;
          printf("multicast CL %d box %3d rows stages %d: landed %7.1f GB/s, %5.1f per SM; L2 reads %7.1f GB/s (%s)\n",
                 CL, rows, stages, landed / ms / 1e6, landed / ms / 1e6 / grid, landed / CL / ms / 1e6,
                 cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
    cudaFree(buf);
  }
  if (getenv("TMA_MC_ONLY")) return 0;
  for (size_t bytes : {size_t(32) << 20, size_t(1) << 30}) {
    const int R = int(bytes / (C * 2));
    void* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    for (int rows : {64, 128, 256}) {
      for (int pan : {1, 2, 4}) {
        for (int cps : {1, 2}) {
          for (int stages : {2, 3, 4, 6, 8}) {
            const size_t smem = size_t(stages) * 128 * rows * pan;
            if (smem * cps > 200 * 1024 || smem * cps < 64 * 1024 || (layout_only_panel_skip(rows, pan))) continue;
            for (int layout = 0; layout < 2; ++layout) {
              CUtensorMap map;
              CUresult r;
              if (layout == 0 && pan == 1) {
                cuuint64_t dims[2] = {cuuint64_t(C), cuuint64_t(R)}, str[1] = {cuuint64_t(C) * 2};
                cuuint32_t box[2] = {64, cuuint32_t(rows)}, es[2] = {1, 1};
                r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
              } else {
                // layout 0 as a 3D view of the row-major matrix: (64 cols, rows, 64-col panels)
                cuuint64_t dims[3] = {64, cuuint64_t(R), cuuint64_t(C / 64)};
                cuuint64_t str[2] = {layout ? 128 : cuuint64_t(C) * 2, layout ? cuuint64_t(R) * 128 : 128};
                cuuint32_t box[3] = {64, cuuint32_t(rows), cuuint32_t(pan)}, es[3] = {1, 1, 1};
                r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
              }
              if (r != CUDA_SUCCESS) { printf("encode failed %d (layout %d pan %d)\n", int(r), layout, pan); continue; }
              const int ntr = R / rows, ntc = C / 64 / pan;
              const int grid = sms * cps;
              const int iters = 400 / cps;
              cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
              cudaEvent_t e0, e1;
              cudaEventCreate(&e0);
              cudaEventCreate(&e1);
              stream<<<grid, 32, smem>>>(map, layout, rows, ntr, ntc, iters, stages, pan);
              cudaEventRecord(e0);
              stream<<<grid, 32, smem>>>(map, layout, rows, ntr, ntc, iters, stages, pan);
              cudaEventRecord(e1);
              cudaEventSynchronize(e1);
              float ms = 0;
              cudaEventElapsedTime(&ms, e0, e1);
              const double moved = double(iters) * grid * 128 * rows * pan;
              printf("buf %5zu MiB box %3dx%d (%3zu KB) cta/SM %d stages %d inflight/SM %3zu KB %-8s: %7.1f GB/s, %5.1f per SM (%s)\n",
                     bytes >> 20, rows, pan, size_t(128) * rows * pan / 1024, cps, stages, smem * cps / 1024,
                     layout ? "panel" : "rowmajor", moved / ms / 1e6, moved / ms / 1e6 / sms,
                     cudaGetErrorString(cudaGetLastError()));
            }
          }
        }
      }
    }
    cudaFree(buf);
  }
  return 0;
}
