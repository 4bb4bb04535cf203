// ag_exact.cu -- the fp32 exact-order All-Gather+GEMM path (TF_F32).
//
// Every C element is ONE chain acc = 0; for k ascending: acc = acc + a*b,
// each multiply and add rounded separately (__fmul_rn/__fadd_rn; the
// reference builds with -ffp-contract=off for the same reason,
// proj/CMakeLists.txt:12-16, tilemath.hpp:90-96).  That makes the result
// bitwise equal to reference::gemm (reference.hpp:36-49) for any shape,
// tiling or world size, which is what config 1 and the reference's bitwise
// tests demand.  It runs on CUDA cores: tensor cores round differently.
//
// Schedules (ag_gemm.hpp):
//   baseline (:134-180)  barrier, gather kernel (every shard -> stage at
//                        column s*kw), barrier, GEMM over stage
//   pull     (:185-222)  one GEMM kernel whose A loads go straight to the
//                        owners' shards over NVLink (peer ld.global)
//   push     (:228-305)  producer kernel stores M x bk blocks into every
//                        dst's inbox at (0, self*kw + p0) and signals
//                        (dst, row=self, slot=kb); the consumer GEMM waits
//                        per (src, kb) block right before using it.
#include <cuda_runtime.h>

#include "ag_internal.hpp"

namespace tfb {

namespace {

constexpr int TM = 32, TN = 32, TK = 32;  // CTA tile; 256 threads, 4 outputs each

struct SrcTable {
  const float* p[64];
};

// C = concat_s(src[s]) * B with the ascending (s, p) chain.  src[s] is an
// m x cols row-major block with row stride `stride`.  When `flags` is set,
// (s, kb) must reach `epoch` before block kb of source s is read.
__global__ void __launch_bounds__(256) exact_gemm_kernel(
    SrcTable srcs, int nsrc, size_t cols, size_t stride, const float* __restrict__ B,
    float* __restrict__ C, size_t m, size_t n, size_t bk, const uint64_t* flags, int n_kb,
    uint64_t epoch, uint64_t watchdog_ns, DevErr* err, int rank, int board) {
  __shared__ float As[TM][TK + 1];
  __shared__ float Bs[TK][TN + 1];
  __shared__ int abort_flag;
  const size_t i0 = size_t(blockIdx.y) * TM, j0 = size_t(blockIdx.x) * TN;
  const int tx = threadIdx.x % TN, ty = threadIdx.x / TN;  // ty in [0, 8)
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  if (threadIdx.x == 0) abort_flag = 0;
  for (int s = 0; s < nsrc; ++s) {
    const float* A = srcs.p[s];
    for (size_t kb0 = 0; kb0 < cols; kb0 += bk) {
      const size_t kb_len = (cols - kb0 < bk) ? cols - kb0 : bk;
      if (flags) {
        if (threadIdx.x == 0) {
          const int kb = int(kb0 / bk);
          if (!wait_geq(flags + size_t(s) * n_kb + kb, epoch, watchdog_ns, err, kWaitSignal,
                        rank, board, s, kb, 0))
            abort_flag = 1;
        }
        __syncthreads();
        if (abort_flag) return;
      }
      for (size_t p0 = kb0; p0 < kb0 + kb_len; p0 += TK) {
        const int tk = int((kb0 + kb_len - p0 < TK) ? kb0 + kb_len - p0 : TK);
        __syncthreads();
        for (int e = threadIdx.x; e < TM * TK; e += 256) {
          const int r = e / TK, c = e % TK;
          // ld.cg: inbox bytes land from other SMs/GPUs during the launch and a
          // line shared with a not-yet-signalled block may sit stale in L1.
          As[r][c] = (i0 + r < m && c < tk) ? __ldcg(A + (i0 + r) * stride + p0 + c) : 0.0f;
        }
        for (int e = threadIdx.x; e < TK * TN; e += 256) {
          const int r = e / TN, c = e % TN;
          const size_t krow = size_t(s) * cols + p0 + r;
          Bs[r][c] = (r < tk && j0 + c < n) ? B[krow * n + j0 + c] : 0.0f;
        }
        __syncthreads();
        for (int kk = 0; kk < tk; ++kk) {
          const float b = Bs[kk][tx];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(As[ty + 8 * q][kk], b));
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const size_t i = i0 + ty + 8 * q, j = j0 + tx;
    if (i < m && j < n) C[i * n + j] = acc[q];
  }
}

// Copies every shard into `stage` (m x k) at column s*kw (ag_gemm.hpp:147-154).
__global__ void exact_gather_kernel(SrcTable shards, int W, float* stage, size_t m, size_t k,
                                    size_t kw) {
  const size_t total = size_t(W) * m * kw;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total;
       e += size_t(gridDim.x) * blockDim.x) {
    const int s = int(e / (m * kw));
    const size_t rem = e % (m * kw);
    const size_t i = rem / kw, c = rem % kw;
    stage[i * k + size_t(s) * kw + c] = shards.p[s][i * kw + c];
  }
}

struct DstTable {
  float* inbox[64];
  uint64_t* flags[64];
};

// Producer (ag_gemm.hpp:241-260): block (kb, dst) stores rows x tk of this
// rank's shard into dst's inbox at (0, self*kw + kb*bk), then raises
// (dst, row=self, slot=kb) with release semantics.
__global__ void exact_push_kernel(const float* __restrict__ shard, DstTable dst, int self,
                                  size_t m, size_t k, size_t kw, size_t bk, int n_kb) {
  const int kb = blockIdx.x, d = blockIdx.y;
  const size_t p0 = size_t(kb) * bk;
  const size_t tk = (kw - p0 < bk) ? kw - p0 : bk;
  float* inbox = dst.inbox[d];
  for (size_t e = threadIdx.x; e < m * tk; e += blockDim.x) {
    const size_t i = e / tk, c = e % tk;
    inbox[i * k + size_t(self) * kw + p0 + c] = shard[i * kw + p0 + c];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_sys();
    red_release_sys(dst.flags[d] + size_t(self) * n_kb + kb, 1);
  }
}

}  // namespace

tf_status ag_exact_run(World* w, tf_ag_variant variant, const tf_ag_shape& sh,
                       void* const* a_shard, const void* const* b, void* const* c,
                       void* const* gathered, const std::vector<cudaStream_t>& streams) {
  const int W = w->W;
  const size_t m = sh.m, n = sh.n, k = sh.k, kw = k / W;
  const size_t bk = sh.bk;
  dim3 grid(unsigned((n + TN - 1) / TN), unsigned((m + TM - 1) / TM));
  if (grid.y > 65535) return set_error(TF_ERR_SHAPE, "ag_gemm(f32): m too large for this path");
  SrcTable shards{};
  for (int s = 0; s < W; ++s) shards.p[s] = static_cast<const float*>(a_shard[s]);

  w->record_ag(m, kw, 4);
  if (variant == TF_AG_PULL) {
    // No staged operand (ag_gemm.hpp:185-222): every block is read in place.
    for (int r = 0; r < W; ++r)
      for (int s = 0; s < W; ++s) w->ag_src[r][s] = {a_shard[s], kw};
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      cudaSetDevice(w->ranks[r].device);
      TFB_CHECK(launch_skew(w, r, streams[r]));
      exact_gemm_kernel<<<grid, 256, 0, streams[r]>>>(
          shards, W, kw, kw, static_cast<const float*>(b[r]), static_cast<float*>(c[r]), m, n,
          bk, nullptr, 0, 0, w->watchdog_ns, w->err_of(r), r, -1);
      TFB_CUDA(cudaGetLastError());
      ++w->launches;
    }
    return TF_OK;
  }

  // baseline and push both stage the gathered operand per rank.  PUSH's
  // internal inbox is written by peers, so it is double-buffered by the
  // flag epoch's parity: a fast peer's run N+1 lands in the other buffer
  // while this rank's run N still reads its inbox (the bf16 path does the
  // same, ag_sm100.cu).  A caller-supplied buffer is single: PUSH then
  // enters a world barrier first, so no peer stores into it before every
  // rank finished its previous run.
  const int n_kb = int((kw + bk - 1) / bk);
  BoardEntry fb{};
  if (variant == TF_AG_PUSH) {
    TFB_CHECK(board_next_epoch(w, "ag.flags", W, n_kb, &fb));
    w->ag_flags = FlagSnapshot{w->board_names[fb.id], size_t(W) * n_kb, fb.epoch};
  }
  std::vector<float*> stage(W, nullptr);
  size_t stage_off = 0;
  bool internal = false, caller = false;
  for (int r = 0; r < W; ++r) {
    if (gathered && gathered[r]) {
      stage[r] = static_cast<float*>(gathered[r]);
      caller = true;
    } else {
      internal = true;
    }
  }
  if (internal) {
    const bool push = variant == TF_AG_PUSH;
    TFB_CHECK(heap_get(w, push ? "ag.inbox" : "ag.stage", sizeof(float) * m * k * (push ? 2 : 1), &stage_off));
    const size_t half = push ? size_t(fb.epoch & 1) * m * k : 0;
    for (int r = 0; r < W; ++r)
      if (!(gathered && gathered[r])) stage[r] = reinterpret_cast<float*>(w->ptr(r, stage_off)) + half;
  }
  if (variant == TF_AG_PUSH && caller && W > 1) TFB_CHECK(world_barrier(w, streams));
  for (int r = 0; r < W; ++r)
    for (int s = 0; s < W; ++s) w->ag_src[r][s] = {stage[r] + size_t(s) * kw, k};

  for (int r = 0; r < W; ++r)
    if (w->ranks[r].local) w->stage(r, sizeof(float) * m * k);  // the gathered copy lands in HBM

  if (variant == TF_AG_BASELINE) {
    TFB_CHECK(world_barrier(w, streams));  // "ag.sync"
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      cudaSetDevice(w->ranks[r].device);
      const size_t total = size_t(W) * m * kw;
      const unsigned blocks = unsigned(std::min<size_t>((total + 255) / 256, 4096));
      exact_gather_kernel<<<blocks, 256, 0, streams[r]>>>(shards, W, stage[r], m, k, kw);
      TFB_CUDA(cudaGetLastError());
      ++w->launches;
    }
    TFB_CHECK(world_barrier(w, streams));
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      cudaSetDevice(w->ranks[r].device);
      SrcTable st{};
      st.p[0] = stage[r];
      TFB_CHECK(launch_skew(w, r, streams[r]));
      exact_gemm_kernel<<<grid, 256, 0, streams[r]>>>(
          st, 1, k, k, static_cast<const float*>(b[r]), static_cast<float*>(c[r]), m, n, bk,
          nullptr, 0, 0, w->watchdog_ns, w->err_of(r), r, -1);
      TFB_CUDA(cudaGetLastError());
      ++w->launches;
    }
    return TF_OK;
  }

  // push
  const uint64_t epoch = fb.epoch;
  DstTable dt{};
  for (int d = 0; d < W; ++d) {
    dt.inbox[d] = stage[d];
    dt.flags[d] = reinterpret_cast<uint64_t*>(w->ptr(d, fb.offset));
  }
  // Producers first (they never wait), on the side streams; consumers on the
  // main streams.  The consumer's stream waits for nothing: the flags order it.
  for (int r = 0; r < W; ++r) {
    if (!w->ranks[r].local) continue;
    cudaSetDevice(w->ranks[r].device);
    cudaEvent_t ev;
    TFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TFB_CUDA(cudaEventRecord(ev, streams[r]));
    TFB_CUDA(cudaStreamWaitEvent(w->ranks[r].side, ev, 0));  // inputs ready
    cudaEventDestroy(ev);
    exact_push_kernel<<<dim3(n_kb, W), 256, 0, w->ranks[r].side>>>(
        static_cast<const float*>(a_shard[r]), dt, r, m, k, kw, bk, n_kb);
    TFB_CUDA(cudaGetLastError());
    ++w->launches;
  }
  for (int r = 0; r < W; ++r) {
    if (!w->ranks[r].local) continue;
    cudaSetDevice(w->ranks[r].device);
    SrcTable st{};
    for (int s = 0; s < W; ++s) st.p[s] = stage[r] + size_t(s) * kw;
    TFB_CHECK(launch_skew(w, r, streams[r]));
    exact_gemm_kernel<<<grid, 256, 0, streams[r]>>>(
        st, W, kw, k, static_cast<const float*>(b[r]), static_cast<float*>(c[r]), m, n, bk,
        reinterpret_cast<const uint64_t*>(w->ptr(r, fb.offset)), n_kb, epoch, w->watchdog_ns,
        w->err_of(r), r, fb.id);
    TFB_CUDA(cudaGetLastError());
    ++w->launches;
    // The producer must finish before the caller reuses the shard.
    cudaEvent_t ev;
    TFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TFB_CUDA(cudaEventRecord(ev, w->ranks[r].side));
    TFB_CUDA(cudaStreamWaitEvent(streams[r], ev, 0));
    cudaEventDestroy(ev);
  }
  return TF_OK;
}

// Force-load this file's kernels on the current device (lazy module loading
// would otherwise load them inside the first schedule, serializing streams).
void ag_exact_preload() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, exact_gemm_kernel);
  cudaFuncGetAttributes(&a, exact_gather_kernel);
  cudaFuncGetAttributes(&a, exact_push_kernel);
}

}  // namespace tfb
