// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference headers
// (compiled in place from /root/reference/proj/include by oracle/Makefile;
// nothing is copied).  TEST INFRASTRUCTURE ONLY: the output,
// oracle/_ref/libtfref.so, is the reference implementation run as-is.  It is
// used (1) to pin oracle/tf_oracle.c, (2) to generate tests/golden fixtures,
// and (3) as bench.py's `--impl reference` / cpu_baseline arm (the
// reference's own CPU path timed on the host cores).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tilefabric/tilefabric.hpp"

using namespace tilefabric;

namespace {
thread_local std::string g_err;

// Status codes mirror include/tilefabric_b200/tf_abi.h's tf_status.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const BoundsError& e) {
    g_err = e.what();
    return 2;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 3;
  } catch (const DeadlockError& e) {
    g_err = e.what();
    return 4;
  } catch (const WorldError& e) {
    g_err = e.what();
    return 5;
  } catch (const EmptyAttentionError& e) {
    g_err = e.what();
    return 6;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

WorldConfig config(int world, int64_t launch_cost_ns) {
  WorldConfig cfg;
  cfg.world_size = world;
  cfg.launch_cost = Duration(launch_cost_ns);
  return cfg;
}

// makespan and post-placement time (makespan - first launch start), the two
// numbers SURVEY.md §8(d) asks for.
void timing(const std::vector<TaskEvent>& ev, const tax::TaxReport& t,
            double* makespan_ns, double* post_ns) {
  if (makespan_ns) *makespan_ns = static_cast<double>(t.makespan.count());
  if (post_ns) {
    Duration first = t.makespan;
    for (const auto& e : ev)
      if (e.kind == EventKind::kLaunch && e.t_start < first) first = e.t_start;
    *post_ns = static_cast<double>((t.makespan - first).count());
  }
}

ag::AgGemmRun ag_dispatch(int variant, const ag::AgGemmProblem& p,
                          const WorldConfig& cfg) {
  switch (variant) {
    case 0: return ag::run_baseline(p, cfg);
    case 1: return ag::run_pull(p, cfg);
    case 2: return ag::run_push(p, cfg);
  }
  throw ConfigError("tfr: unknown ag variant");
}

void ag_out(const ag::AgGemmRun& run, float* c_out, uint64_t* flags_out) {
  size_t off = 0;
  for (const auto& c : run.c) {
    if (c_out) std::memcpy(c_out + off, c.data(), c.size() * sizeof(float));
    off += c.size();
  }
  if (flags_out) {
    size_t f = 0;
    for (const auto& fl : run.flag_counts)
      for (auto v : fl) flags_out[f++] = v;
  }
}

void fd_out(const fd::FdRun& run, float* out, uint64_t* flags_out) {
  size_t off = 0;
  for (const auto& o : run.out) {
    if (out) std::memcpy(out + off, o.data(), o.size() * sizeof(float));
    off += o.size();
  }
  if (flags_out) {
    size_t f = 0;
    for (const auto& fl : run.flag_counts)
      for (auto v : fl) flags_out[f++] = v;
  }
}
}  // namespace

extern "C" {

const char* tfr_last_error() { return g_err.c_str(); }

int tfr_uniform_reals(uint64_t seed, size_t n, float* out) {
  return guarded([&] {
    auto v = uniform_reals(seed, n);
    std::memcpy(out, v.data(), n * sizeof(float));
  });
}

// ag::make_problem(seed, m, n, k, tiles) then run_{baseline,pull,push}.
// c_out: world * m * n (every rank's C); flags_out: world * W * n_kb (push).
int tfr_ag_run(int variant, uint64_t seed, size_t m, size_t n, size_t k,
               size_t bm, size_t bn, size_t bk, int world,
               int64_t launch_cost_ns, float* c_out, uint64_t* flags_out,
               double* makespan_ns, double* post_ns) {
  return guarded([&] {
    TileSpec t;
    t.bm = bm;
    t.bn = bn;
    t.bk = bk;
    const auto p = ag::make_problem(seed, m, n, k, t);
    const auto run = ag_dispatch(variant, p, config(world, launch_cost_ns));
    ag_out(run, c_out, flags_out);
    timing(run.events, run.taxes, makespan_ns, post_ns);
  });
}

// Same schedules over caller-supplied A (m x k) and B (k x n); rank 0's C.
int tfr_ag_run_inputs(int variant, const float* a, const float* b, size_t m,
                      size_t n, size_t k, size_t bm, size_t bn, size_t bk,
                      int world, float* c_rank0, double* makespan_ns,
                      double* post_ns) {
  return guarded([&] {
    ag::AgGemmProblem p;
    p.m = m;
    p.n = n;
    p.k = k;
    p.tiles.bm = bm;
    p.tiles.bn = bn;
    p.tiles.bk = bk;
    p.a.assign(a, a + m * k);
    p.b.assign(b, b + k * n);
    const auto run = ag_dispatch(variant, p, config(world, 0));
    if (c_rank0)
      std::memcpy(c_rank0, run.c[0].data(), m * n * sizeof(float));
    timing(run.events, run.taxes, makespan_ns, post_ns);
  });
}

// fd::make_problem(seed, heads, head_dim, kv_len) then run_fd(variant).
// out: world * heads * head_dim; flags_out: world * W (push-style variants).
int tfr_fd_run(int variant, uint64_t seed, int heads, int head_dim,
               size_t kv_len, int world, int64_t launch_cost_ns, float* out,
               uint64_t* flags_out, double* makespan_ns, double* post_ns) {
  return guarded([&] {
    const auto p = fd::make_problem(seed, heads, head_dim, kv_len);
    const auto run = fd::run_fd(p, static_cast<fd::Variant>(variant),
                                config(world, launch_cost_ns));
    fd_out(run, out, flags_out);
    timing(run.events, run.taxes, makespan_ns, post_ns);
  });
}

int tfr_fd_run_inputs(int variant, const float* q, const float* k,
                      const float* v, int heads, int head_dim, size_t kv_len,
                      float scale, int world, float* out_rank0,
                      double* makespan_ns, double* post_ns) {
  return guarded([&] {
    fd::DecodeProblem p;
    p.heads = heads;
    p.head_dim = head_dim;
    p.kv_len = kv_len;
    p.scale = scale;
    const size_t hd = static_cast<size_t>(heads) * head_dim;
    p.q.assign(q, q + hd);
    p.k.assign(k, k + hd * kv_len);
    p.v.assign(v, v + hd * kv_len);
    const auto run = fd::run_fd(p, static_cast<fd::Variant>(variant),
                                config(world, 0));
    if (out_rank0) std::memcpy(out_rank0, run.out[0].data(), hd * sizeof(float));
    timing(run.events, run.taxes, makespan_ns, post_ns);
  });
}

int tfr_gemm(const float* a, const float* b, size_t m, size_t n, size_t k,
             float* c) {
  return guarded([&] {
    auto v = reference::gemm(a, b, m, n, k);
    std::memcpy(c, v.data(), m * n * sizeof(float));
  });
}

int tfr_attention(const float* q, const float* k, const float* v,
                  size_t heads, size_t head_dim, size_t kv_len, float scale,
                  float* out) {
  return guarded([&] {
    auto o = reference::attention(q, k, v, heads, head_dim, kv_len, scale);
    std::memcpy(out, o.data(), o.size() * sizeof(float));
  });
}

// attention_partial + serialize_partial (tilemath.hpp:145-181, 249-258).
int tfr_attention_partial_wire(const float* q, const float* k, const float* v,
                               int heads, int head_dim, size_t len,
                               float scale, float* wire) {
  return guarded([&] {
    auto p = attention_partial(q, k, v, heads, head_dim, len, scale);
    serialize_partial(p, wire);
  });
}

// acc <- combine_partials(acc, x) on wire rows (tilemath.hpp:186-220).
int tfr_combine_wire(float* acc, const float* x, int heads, int head_dim) {
  return guarded([&] {
    auto a = deserialize_partial(acc, heads, head_dim);
    auto b = deserialize_partial(x, heads, head_dim);
    serialize_partial(combine_partials(a, b), acc);
  });
}

int tfr_finalize_wire(const float* acc, int heads, int head_dim, float* out) {
  return guarded([&] {
    auto o = finalize(deserialize_partial(acc, heads, head_dim));
    std::memcpy(out, o.data(), o.size() * sizeof(float));
  });
}

double tfr_max_head_relative_error(const float* a, const float* b, int heads,
                                   int head_dim) {
  const size_t n = static_cast<size_t>(heads) * head_dim;
  std::vector<float> x(a, a + n), y(b, b + n);
  return reference::max_head_relative_error(x, y, heads, head_dim);
}

unsigned tfr_hardware_concurrency() { return std::thread::hardware_concurrency(); }

}  // extern "C"
