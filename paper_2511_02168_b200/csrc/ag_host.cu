// ag_host.cu -- tf_ag_gemm_host: All-Gather+GEMM with the reference's own
// calling convention -- operands in host memory, C returned to host memory
// (AgGemmProblem holds host vectors, AgGemmRun returns them, ag_gemm.hpp:47-99)
// -- with the PCIe transfers overlapped with the exchange and the GEMM.
//
// Per local rank, three streams:
//   h2d      A shard -> its symmetric-heap region, then B in column slabs
//            (cudaMemcpy2DAsync, row pitch n) into a device B buffer;
//   compute  the caller's stream: world barrier once every shard is placed,
//            then one All-Gather+GEMM per B slab as soon as that slab has
//            landed.  Slab 0 runs the requested schedule (pull / push /
//            baseline, including the exchange); later slabs reuse the
//            gathered inbox (AgLayout::inbox_complete) and only multiply;
//   d2h      each C slab back to the host as soon as its GEMM retired.
// Host->device and device->host use different copy engines and directions of
// the link, so the job costs ~ max(H2D bytes, D2H bytes) / PCIe + one small
// trailing slab, not the sum of the copies and the GEMM.  Slabs are
// multiples of the 512-column CTA-pair tile; the first is small so C starts
// flowing back early, the last ones shrink so the exposed tail (last GEMM +
// last D2H) is short.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "ag_internal.hpp"

namespace tfb {
namespace {

tf_status ensure_copy_streams(World* w, int r) {
  RankRes& rr = w->ranks[r];
  cudaSetDevice(rr.device);
  if (!rr.h2d) TFB_CUDA(cudaStreamCreateWithFlags(&rr.h2d, cudaStreamNonBlocking));
  if (!rr.d2h) TFB_CUDA(cudaStreamCreateWithFlags(&rr.d2h, cudaStreamNonBlocking));
  return TF_OK;
}

// `after` waits for everything enqueued on `before` so far.
tf_status join(cudaStream_t after, cudaStream_t before) {
  cudaEvent_t ev;
  TFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  TFB_CUDA(cudaEventRecord(ev, before));
  TFB_CUDA(cudaStreamWaitEvent(after, ev, 0));
  cudaEventDestroy(ev);  // released once the recorded work completes
  return TF_OK;
}

// TFB_HOST_TRACE=1: timing events after every copy / GEMM of rank 0,
// printed by the blocking entry point (a profiling aid; nsys is absent).
struct Trace {
  bool on = false;
  cudaEvent_t t0 = nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  void start(cudaStream_t s) {
    // Only the latest call is traced: drop what earlier (async) calls marked.
    for (auto& pe : ev) cudaEventDestroy(pe.second);
    ev.clear();
    if (t0) cudaEventDestroy(t0);
    t0 = nullptr;
    on = std::getenv("TFB_HOST_TRACE") != nullptr;
    if (!on) return;
    cudaEventCreate(&t0);
    cudaEventRecord(t0, s);
  }
  void mark(const std::string& what, cudaStream_t s) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(what, e);
  }
  void dump() {
    if (!on) return;
    for (auto& [what, e] : ev) {
      float ms = 0;
      cudaEventElapsedTime(&ms, t0, e);
      std::fprintf(stderr, "[host-trace] %8.3f ms  %s\n", ms, what.c_str());
      cudaEventDestroy(e);
    }
    cudaEventDestroy(t0);
    t0 = nullptr;
    ev.clear();
    on = false;
  }
};
// Debug timeline (TFB_HOST_TRACE); per host thread, so concurrent worlds on
// different threads never share it.
thread_local Trace g_trace;

}  // namespace

// Column slab widths for the host-streaming schedule.
std::vector<size_t> ag_host_slabs(size_t n, tf_dtype dt) {
  if (dt != TF_BF16 || n <= 2048) return {n};
  size_t main = std::max<size_t>(1024, (n / 8 + 511) / 512 * 512);
  if (const char* e = std::getenv("TFB_HOST_SLAB")) main = std::max<size_t>(512, std::strtoull(e, nullptr, 10));
  if (const char* e = std::getenv("TFB_HOST_ONESHOT"))
    if (std::atoi(e)) return {n};
  std::vector<size_t> v;
  size_t rem = n;
  // A small first slab: the D2H direction idles until the first C slab
  // exists, and everything before it (the whole shard plus slab 0 of B)
  // is exposed.
  if (!std::getenv("TFB_HOST_BIGFIRST") && rem > 2 * main) {
    v.push_back(1024);
    rem -= 1024;
  }
  while (rem) {
    size_t s;
    if (rem > 2 * main) s = main;
    else if (rem <= 1024) s = rem;
    else s = std::min(rem, (rem / 2 + 511) / 512 * 512);
    v.push_back(s);
    rem -= s;
  }
  return v;
}

}  // namespace tfb

using namespace tfb;

extern "C" tf_status tf_ag_gemm_host_async(tf_world* tw, tf_ag_variant variant, const tf_ag_shape* shape,
                                           const void* const* a_host, const void* const* b_host,
                                           void* const* c_host, void* const* streams) {
  if (!tw) return set_error(TF_ERR_CONFIG, "tf_ag_gemm_host: NULL world");
  World* w = &tw->impl;
  if (!shape || !a_host || !b_host || !c_host)
    return set_error(TF_ERR_CONFIG, "tf_ag_gemm_host: NULL argument");
  if (variant < TF_AG_BASELINE || variant > TF_AG_PUSH)
    return set_error(TF_ERR_CONFIG, "ag_gemm: unknown variant");
  tf_ag_shape sh = *shape;
  if (sh.m < 1 || sh.n < 1 || sh.k < 1) return set_error(TF_ERR_CONFIG, "ag_gemm: m, n, k must be >= 1");
  if (sh.k % size_t(w->W) != 0)
    return set_error(TF_ERR_CONFIG, "ag_gemm: k = " + std::to_string(sh.k) +
                                        " must be divisible by world_size = " + std::to_string(w->W));
  if (sh.dtype != TF_F32 && sh.dtype != TF_BF16) return set_error(TF_ERR_CONFIG, "ag_gemm: unknown dtype");
  if (sh.shard != TF_SHARD_K)
    return set_error(TF_ERR_CONFIG, "tf_ag_gemm_host: M-sharded A is supported by the device-resident entry points "
                                    "(tf_ag_gemm[_async]) only");
  if (sh.bm == 0) sh.bm = 16;
  if (sh.bn == 0) sh.bn = 16;
  if (sh.bk == 0) sh.bk = 16;
  const int W = w->W;
  const size_t esz = sh.dtype == TF_F32 ? 4 : 2;
  const size_t m = sh.m, n = sh.n, k = sh.k, kw = k / size_t(W);
  for (int r = 0; r < W; ++r)
    if (w->ranks[r].local && (!a_host[r] || !b_host[r] || !c_host[r]))
      return set_error(TF_ERR_CONFIG, "tf_ag_gemm_host: a/b/c for local rank " + std::to_string(r) +
                                          " is NULL");
  auto s = resolve_streams(w, streams);
  TFB_CHECK(refuse_multi_rank_capture(w, s, "tf_ag_gemm_host"));
  TFB_CHECK(order_after_legacy(w, streams));
  g_trace.start(s[w->first_local]);
  const int tr = w->first_local;

  // Buffer sets: a one-rank world alternates two (shard region, device B,
  // device C), so back-to-back calls on different streams overlap -- call
  // i+1's H2D streams in while call i's last slabs compute and read back.
  // Every call orders its copies after the caller's prior work on its own
  // stream, its H2D after the last GEMM that read the same set and its
  // GEMMs after the last read-back of the same C (events per set).  With
  // W > 1 (peers read the shard region) there is one set, so calls on
  // different streams still serialise through those events.
  const bool dual = W == 1;
  int par = 0;
  if (dual) {
    par = w->ranks[w->first_local].host_par;
    w->ranks[w->first_local].host_par ^= 1;
  }
  // Shards live in the symmetric heap (peers pull them / push from them).
  size_t shard_off = 0;
  TFB_CHECK(heap_get(w, "ag.host.a" + std::string(par ? "1" : "") + "[" + std::to_string(m * kw * esz) + "]",
                     m * kw * esz, &shard_off));
  std::vector<void*> shard(W), bdev(W, nullptr), cdev(W, nullptr);
  for (int r = 0; r < W; ++r) shard[r] = w->ptr(r, shard_off);
  for (int r = 0; r < W; ++r) {
    if (!w->ranks[r].local) continue;
    TFB_CHECK(ensure_copy_streams(w, r));
    TFB_CHECK(ensure_scratch(w, r, par ? 3 : 0, k * n * esz, &bdev[r]));
    TFB_CHECK(ensure_scratch(w, r, par ? 4 : 1, m * n * esz, &cdev[r]));
    RankRes& rr = w->ranks[r];
    cudaSetDevice(rr.device);
    for (int i = 0; i < 2; ++i) {
      if (!rr.host_reads_done[i]) TFB_CUDA(cudaEventCreateWithFlags(&rr.host_reads_done[i], cudaEventDisableTiming));
      if (!rr.host_d2h_done[i]) TFB_CUDA(cudaEventCreateWithFlags(&rr.host_d2h_done[i], cudaEventDisableTiming));
    }
    // Copies start after the caller's prior work on its stream, the H2D
    // after the set's previous readers, the GEMMs after the set's previous
    // C read-back.
    TFB_CHECK(join(rr.h2d, s[r]));
    TFB_CHECK(join(rr.d2h, s[r]));
    TFB_CUDA(cudaStreamWaitEvent(rr.h2d, rr.host_reads_done[par], 0));
    TFB_CUDA(cudaStreamWaitEvent(s[r], rr.host_d2h_done[par], 0));
    TFB_CUDA(cudaMemcpyAsync(shard[r], a_host[r], m * kw * esz, cudaMemcpyDefault, rr.h2d));
    if (r == tr) g_trace.mark("h2d shard", rr.h2d);
  }
  const std::vector<size_t> slabs = ag_host_slabs(n, sh.dtype);
  auto put_b = [&](size_t off, size_t ns) -> tf_status {
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      RankRes& rr = w->ranks[r];
      cudaSetDevice(rr.device);
      TFB_CUDA(cudaMemcpy2DAsync(static_cast<char*>(bdev[r]) + off * esz, n * esz,
                                 static_cast<const char*>(b_host[r]) + off * esz, n * esz, ns * esz, k,
                                 cudaMemcpyDefault, rr.h2d));
      if (r == tr) g_trace.mark("h2d B cols " + std::to_string(off) + "+" + std::to_string(ns), rr.h2d);
      TFB_CHECK(join(s[r], rr.h2d));
    }
    return TF_OK;
  };
  // Slab 0's B is queued behind the shard; compute waits for both, then
  // every rank's shard must be in place before any peer reads or pushes it.
  TFB_CHECK(put_b(0, slabs[0]));
  if (W > 1) TFB_CHECK(world_barrier(w, s));
  size_t off = 0;
  for (size_t j = 0; j < slabs.size(); ++j) {
    const size_t ns = slabs[j];
    if (j > 0) TFB_CHECK(put_b(off, ns));
    tf_ag_shape slab = sh;
    slab.n = ns;
    std::vector<const void*> bp(W, nullptr);
    std::vector<void*> cp(W, nullptr);
    for (int r = 0; r < W; ++r)
      if (w->ranks[r].local) {
        bp[r] = static_cast<const char*>(bdev[r]) + off * esz;
        cp[r] = static_cast<char*>(cdev[r]) + off * esz;
      }
    if (sh.dtype == TF_F32) {
      TFB_CHECK(ag_exact_run(w, variant, slab, shard.data(), bp.data(), cp.data(), nullptr, s));
    } else {
      AgLayout lay;
      lay.ldb = n;
      lay.ldc = n;
      lay.inbox_complete = j > 0;
      lay.split_k = false;
      TFB_CHECK(ag_bf16_run(w, variant, slab, shard.data(), bp.data(), cp.data(), nullptr, s, lay));
    }
    g_trace.mark("gemm cols " + std::to_string(off) + "+" + std::to_string(ns), s[tr]);
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      RankRes& rr = w->ranks[r];
      cudaSetDevice(rr.device);
      TFB_CHECK(join(rr.d2h, s[r]));
      TFB_CUDA(cudaMemcpy2DAsync(static_cast<char*>(c_host[r]) + off * esz, n * esz,
                                 static_cast<const char*>(cdev[r]) + off * esz, n * esz, ns * esz, m,
                                 cudaMemcpyDefault, rr.d2h));
      if (r == tr) g_trace.mark("d2h C cols " + std::to_string(off) + "+" + std::to_string(ns), rr.d2h);
    }
    off += ns;
  }
  // The set's readers and read-back are done at these events; the call
  // completes on the caller's streams.
  for (int r = 0; r < W; ++r)
    if (w->ranks[r].local) {
      RankRes& rr = w->ranks[r];
      cudaSetDevice(rr.device);
      TFB_CUDA(cudaEventRecord(rr.host_reads_done[par], s[r]));
      TFB_CUDA(cudaEventRecord(rr.host_d2h_done[par], rr.d2h));
      TFB_CHECK(join(s[r], rr.d2h));
    }
  return TF_OK;
}

extern "C" tf_status tf_ag_gemm_host(tf_world* tw, tf_ag_variant variant, const tf_ag_shape* shape,
                                     const void* const* a_host, const void* const* b_host,
                                     void* const* c_host, void* const* streams) {
  TFB_CHECK(tf_ag_gemm_host_async(tw, variant, shape, a_host, b_host, c_host, streams));
  tf_status st = sync_and_check(&tw->impl, resolve_streams(&tw->impl, streams));
  g_trace.dump();
  return st;
}
