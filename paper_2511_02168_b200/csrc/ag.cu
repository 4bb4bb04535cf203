// ag.cu -- tf_ag_gemm: validation (AgGemmProblem::validate,
// ag_gemm.hpp:55-66; TileSpec::validate, tilemath.hpp:83-87) and dispatch to
// the fp32 exact-order path or the bf16 tensor-core path.
#include <algorithm>
#include <string>

#include "ag_internal.hpp"

using namespace tfb;

static tf_status ag_validate(World* w, const tf_ag_shape* sh, void* const* a_shard,
                             const void* const* b, void* const* c) {
  if (!sh || !a_shard || !b || !c) return set_error(TF_ERR_CONFIG, "tf_ag_gemm: NULL argument");
  if (sh->m < 1 || sh->n < 1 || sh->k < 1)
    return set_error(TF_ERR_CONFIG, "ag_gemm: m, n, k must be >= 1");
  if (sh->k % size_t(w->W) != 0)
    return set_error(TF_ERR_CONFIG, "ag_gemm: k = " + std::to_string(sh->k) +
                                        " must be divisible by world_size = " +
                                        std::to_string(w->W));
  if (sh->dtype != TF_F32 && sh->dtype != TF_BF16)
    return set_error(TF_ERR_CONFIG, "ag_gemm: unknown dtype");
  if (sh->shard != TF_SHARD_K && sh->shard != TF_SHARD_M)
    return set_error(TF_ERR_CONFIG, "ag_gemm: unknown shard layout");
  const bool msh = sh->shard == TF_SHARD_M;
  if (msh && sh->dtype != TF_BF16)
    return set_error(TF_ERR_CONFIG, "ag_gemm: M-sharded A is supported on the bf16 tensor-core path");
  if (msh && sh->m % (size_t(w->W) * 128) != 0)
    return set_error(TF_ERR_SHAPE, "ag_gemm (M-sharded): m = " + std::to_string(sh->m) +
                                       " must be a multiple of 128 * world_size");
  const size_t esz = sh->dtype == TF_F32 ? 4 : 2;
  const size_t kw = sh->k / size_t(w->W);
  const size_t shard_elems = msh ? sh->m / size_t(w->W) * sh->k : sh->m * kw;
  for (int r = 0; r < w->W; ++r) {
    if (!a_shard[r])
      return set_error(TF_ERR_CONFIG, "ag_gemm: a_shard[" + std::to_string(r) + "] is NULL");
    if (!in_heap(w, r, a_shard[r], esz * shard_elems))
      return set_error(TF_ERR_BOUNDS, "ag_gemm: a_shard[" + std::to_string(r) + "] is not an " +
                                          (msh ? "m/W x k" : "m x k/W") + " region of rank " +
                                          std::to_string(r) + "'s symmetric heap");
    if (w->ranks[r].local && (!b[r] || !c[r]))
      return set_error(TF_ERR_CONFIG, "ag_gemm: b/c for local rank " + std::to_string(r) +
                                          " is NULL");
  }
  return TF_OK;
}

extern "C" tf_status tf_ag_gemm_async(tf_world* tw, tf_ag_variant variant,
                                      const tf_ag_shape* shape, void* const* a_shard,
                                      const void* const* b, void* const* c,
                                      void* const* gathered_opt, void* const* streams) {
  if (!tw) return set_error(TF_ERR_CONFIG, "tf_ag_gemm: NULL world");
  World* w = &tw->impl;
  TFB_CHECK(ag_validate(w, shape, a_shard, b, c));
  if (variant < TF_AG_BASELINE || variant > TF_AG_PUSH)
    return set_error(TF_ERR_CONFIG, "ag_gemm: unknown variant");
  tf_ag_shape sh = *shape;
  if (sh.bm == 0) sh.bm = 16;
  if (sh.bn == 0) sh.bn = 16;
  if (sh.bk == 0) sh.bk = 16;
  auto s = resolve_streams(w, streams);
  TFB_CHECK(refuse_multi_rank_capture(w, s, "tf_ag_gemm"));
  TFB_CHECK(order_after_legacy(w, streams));
  if (sh.dtype == TF_F32) return ag_exact_run(w, variant, sh, a_shard, b, c, gathered_opt, s);
  return ag_bf16_run(w, variant, sh, a_shard, b, c, gathered_opt, s);
}

extern "C" tf_status tf_ag_gemm(tf_world* tw, tf_ag_variant variant, const tf_ag_shape* shape,
                                void* const* a_shard, const void* const* b, void* const* c,
                                void* const* gathered_opt, void* const* streams) {
  TFB_CHECK(tf_ag_gemm_async(tw, variant, shape, a_shard, b, c, gathered_opt, streams));
  return sync_and_check(&tw->impl, resolve_streams(&tw->impl, streams));
}

extern "C" tf_status tf_ag_flag_counts(tf_world* tw, int rank, uint64_t* out, size_t cap,
                                       size_t* count) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  const FlagSnapshot& f = w->ag_flags;
  if (count) *count = f.cells;
  if (f.cells == 0 || !out) return TF_OK;
  if (rank < 0 || rank >= w->W) return set_error(TF_ERR_BOUNDS, "ag_flag_counts: bad rank");
  auto it = w->boards.find(f.board);
  if (it == w->boards.end()) return TF_OK;
  std::vector<uint64_t> v(f.cells);
  TFB_CUDA(cudaMemcpy(v.data(), w->ptr(rank, it->second.offset), sizeof(uint64_t) * f.cells,
                      cudaMemcpyDefault));
  for (size_t i = 0; i < f.cells && i < cap; ++i) out[i] = v[i] - (f.epoch - 1);
  return TF_OK;
}

extern "C" tf_status tf_world_set_events(tf_world* tw, int enable) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  tw->impl.events = enable != 0;
  return TF_OK;
}

extern "C" tf_status tf_ag_events(tf_world* tw, int rank, uint64_t* out, size_t cap, size_t* count) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  if (rank < 0 || rank >= w->W) return set_error(TF_ERR_BOUNDS, "ag_events: bad rank");
  if (count) *count = w->ag_events_n;
  if (!out || w->ag_events_n == 0) return TF_OK;
  const size_t n = std::min(cap, w->ag_events_n);
  TFB_CUDA(cudaDeviceSynchronize());
  TFB_CUDA(cudaMemcpy(out, w->ptr(rank, w->ag_events_off), n * sizeof(uint64_t), cudaMemcpyDefault));
  return TF_OK;
}

// The gathered operand of the last AG run on `rank`, m x k row-major into
// dst (host or device): the placement check (ag_gemm_test.cpp:113-169,
// the inbox/stage equals the logical A).  Blocks until the rank is idle.
extern "C" tf_status tf_ag_gathered(tf_world* tw, int rank, void* dst, size_t bytes) {
  if (!tw || !dst) return set_error(TF_ERR_CONFIG, "tf_ag_gathered: NULL argument");
  World* w = &tw->impl;
  if (rank < 0 || rank >= w->W || !w->ranks[rank].local)
    return set_error(TF_ERR_BOUNDS, "tf_ag_gathered: rank " + std::to_string(rank) + " is not local");
  if (w->ag_src.empty()) return set_error(TF_ERR_CONFIG, "tf_ag_gathered: no All-Gather+GEMM run yet");
  const size_t m = w->ag_m, kw = w->ag_kw, esz = w->ag_esz, k = kw * size_t(w->W);
  if (bytes < m * k * esz)
    return set_error(TF_ERR_BOUNDS, "tf_ag_gathered: need " + std::to_string(m * k * esz) + " bytes");
  TFB_CUDA(cudaSetDevice(w->ranks[rank].device));
  TFB_CHECK(sync_and_check(w, resolve_streams(w, nullptr)));
  for (int s = 0; s < w->W; ++s) {
    const World::AgBlock& b = w->ag_src[rank][s];
    if (w->ag_msharded)  // block s: rows [s*m/W, (s+1)*m/W), every column
      TFB_CUDA(cudaMemcpy2D(static_cast<char*>(dst) + size_t(s) * (m / w->W) * k * esz, k * esz,
                            static_cast<const char*>(b.p), b.pitch * esz, k * esz, m / w->W, cudaMemcpyDefault));
    else
      TFB_CUDA(cudaMemcpy2D(static_cast<char*>(dst) + size_t(s) * kw * esz, k * esz,
                            static_cast<const char*>(b.p), b.pitch * esz, kw * esz, m, cudaMemcpyDefault));
  }
  return TF_OK;
}
