// tilefabric.hpp -- C++ drop-in for the reference's hot-path operator API,
// rebuilt on the C ABI (tf_abi.h) of the B200-native kernels.
//
// A caller of the reference (proj/include/tilefabric/{ag_gemm,flash_decode}.hpp)
// switches by including this header instead: the namespaces, problem/run
// structs, make_problem generators, run_* entry points and exception classes
// keep their names and meaning.  Differences (all documented in DESIGN.md):
//   * WorldConfig keeps world_size/watchdog/seed/skew (inject_skew delays the
//     rank's first compute stage on the device); launch_cost and
//     spin_yield_every were CPU-simulation devices and are accepted but unused.
//   * AgGemmRun / FdRun carry results, flag counts and the per-rank Three
//     Taxes measured on the device (tf_taxes); the CPU event log is not
//     produced (the GPU measures real time instead).
//   * dtype selects the fp32 exact-order path (bitwise == reference) or the
//     bf16 tensor-core path; DecodeProblem gains batch and kv_heads (GQA).
// Link: -ltilefabric_b200 (paper_2511_02168_b200/libtilefabric_b200.so).
#pragma once

#include <cmath>
#include <cstdint>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "tilefabric_b200/tf_abi.h"

namespace tilefabric {

// ---- common.hpp:39-94 -------------------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConfigError : public Error { public: using Error::Error; };
class BoundsError : public Error { public: using Error::Error; };
class ShapeError : public Error { public: using Error::Error; };
class DeadlockError : public Error { public: using Error::Error; };
class WorldError : public Error { public: using Error::Error; };
class EmptyAttentionError : public Error { public: using Error::Error; };
class NumericError : public Error { public: using Error::Error; };
class CudaError : public Error { public: using Error::Error; };

namespace b200 {
inline void check(tf_status s) {
  if (s == TF_OK) return;
  const std::string msg = tf_last_error();
  switch (s) {
    case TF_ERR_CONFIG: throw ConfigError(msg);
    case TF_ERR_BOUNDS: throw BoundsError(msg);
    case TF_ERR_SHAPE: throw ShapeError(msg);
    case TF_ERR_DEADLOCK: throw DeadlockError(msg);
    case TF_ERR_WORLD: throw WorldError(msg);
    case TF_ERR_EMPTY_ATTENTION: throw EmptyAttentionError(msg);
    case TF_ERR_NUMERIC: throw NumericError(msg);
    default: throw CudaError(msg);
  }
}

// bf16 round-to-nearest-even of an fp32 value (input placement for TF_BF16).
inline uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return uint16_t((u | 0x00400000u) >> 16);
  return uint16_t((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}
inline float from_bf16(uint16_t h) {
  uint32_t u = uint32_t(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// RAII world + caller-owned device buffers.
struct World {
  tf_world* w = nullptr;
  std::vector<std::pair<int, void*>> owned;
  World(int world_size, const std::vector<int>& devices, size_t heap_bytes, double watchdog) {
    check(tf_world_create(world_size, devices.data(), heap_bytes, watchdog, &w));
  }
  ~World() {
    for (auto& o : owned) tf_device_free(w, o.first, o.second);
    tf_world_destroy(w);
  }
  World(const World&) = delete;
  World& operator=(const World&) = delete;
  void* device(int rank, size_t bytes) {
    void* p = nullptr;
    check(tf_device_alloc(w, rank, bytes, &p));
    owned.emplace_back(rank, p);
    return p;
  }
  std::vector<void*> heap(const std::string& name, size_t bytes) {
    std::vector<void*> p(tf_world_size(w));
    check(tf_heap_alloc(w, name.c_str(), bytes, p.data()));
    return p;
  }
  void put(void* dst, const void* src, size_t bytes) { check(tf_memcpy(w, dst, src, bytes)); }
  template <class Cfg>
  void apply(const Cfg& cfg) {
    for (const auto& [rank, delay] : cfg.skew) check(tf_world_set_skew(w, rank, uint64_t(delay.count())));
  }
  std::vector<tf_taxes> taxes() {
    std::vector<tf_taxes> t(tf_world_size(w));
    for (int r = 0; r < int(t.size()); ++r) check(tf_tax_report(w, r, &t[r]));
    return t;
  }
};
}  // namespace b200

// ---- common.hpp:132-140 -----------------------------------------------------
inline std::vector<float> uniform_reals(std::uint64_t seed, std::size_t n) {
  std::vector<float> out(n);
  b200::check(tf_uniform_reals(seed, n, out.data()));
  return out;
}

// ---- fabric.hpp:46-96 (the GPU-meaningful fields) ---------------------------
using Duration = std::chrono::nanoseconds;

struct WorldConfig {  // fabric.hpp:46-96
  int world_size = 1;
  double watchdog_secs = 0.0;      // 0 -> TILEFABRIC_WATCHDOG_SECS or 10 s
  std::uint64_t seed = 0;
  std::vector<int> devices;        // empty -> all ranks on GPU 0 (loopback world)
  std::size_t heap_bytes = 0;      // 0 -> sized from the problem
  std::map<int, Duration> skew;    // straggler delay of a rank's first compute stage
  Duration launch_cost{0};         // CPU-simulation knob: accepted, unused
  int spin_yield_every = 64;       // CPU-simulation knob: accepted, unused
  void validate() const {
    if (world_size < 1 || world_size > 64)
      throw ConfigError("world_size must be in [1, 64], got " + std::to_string(world_size));
    if (launch_cost < Duration::zero()) throw ConfigError("launch_cost must be >= 0");
    if (spin_yield_every < 1) throw ConfigError("spin_yield_every must be >= 1");
    for (const auto& [rank, delay] : skew) {
      if (rank < 0 || rank >= world_size)
        throw ConfigError("skew rank " + std::to_string(rank) + " out of range for world_size " +
                          std::to_string(world_size));
      if (delay < Duration::zero()) throw ConfigError("skew delay must be >= 0");
    }
  }
  std::vector<int> device_list() const {
    return devices.empty() ? std::vector<int>(std::size_t(world_size), 0) : devices;
  }
};

// fabric.hpp:100-110: validates eagerly, accumulates per rank.
template <class Rep, class Period>
inline void inject_skew(WorldConfig& cfg, int rank, std::chrono::duration<Rep, Period> delay) {
  if (rank < 0 || rank >= cfg.world_size)
    throw ConfigError("inject_skew: rank " + std::to_string(rank) + " out of range for world_size " +
                      std::to_string(cfg.world_size));
  if (delay < delay.zero()) throw ConfigError("inject_skew: delay must be >= 0");
  cfg.skew[rank] += std::chrono::duration_cast<Duration>(delay);
}

// ---- tilemath.hpp:78-88 ------------------------------------------------------
struct TileSpec {
  std::size_t bm = 16, bn = 16, bk = 16;
  void validate() const {
    if (bm < 1 || bn < 1 || bk < 1) throw ConfigError("tile extents must be >= 1");
  }
};

enum class Dtype { kF32 = TF_F32, kBF16 = TF_BF16 };

// ============================ ag_gemm.hpp =====================================
namespace ag {

// How A is sharded before the all-gather: by columns (the reference,
// fill_shard, ag_gemm.hpp:103-112) or by rows (extension, TF_SHARD_M: the
// sharding SPEC.md:265 leaves out; bf16, m a multiple of 128 * world_size).
enum class Shard { kK = TF_SHARD_K, kM = TF_SHARD_M };

struct AgGemmProblem {  // ag_gemm.hpp:47-66
  std::size_t m = 0, n = 0, k = 0;
  TileSpec tiles;
  std::vector<float> a;  // m x k
  std::vector<float> b;  // k x n
  Dtype dtype = Dtype::kF32;
  Shard shard = Shard::kK;
  void validate(int world_size) const {
    if (m < 1 || n < 1 || k < 1) throw ConfigError("ag_gemm: m, n, k must be >= 1");
    if (k % std::size_t(world_size) != 0)
      throw ConfigError("ag_gemm: k = " + std::to_string(k) + " must be divisible by world_size = " +
                        std::to_string(world_size));
    tiles.validate();
  }
};

// ag_gemm.hpp:71-83: one generator stream, A first, then B.
inline AgGemmProblem make_problem(std::uint64_t seed, std::size_t m, std::size_t n, std::size_t k,
                                  TileSpec tiles = {}) {
  AgGemmProblem p;
  p.m = m;
  p.n = n;
  p.k = k;
  p.tiles = tiles;
  std::vector<float> all = uniform_reals(seed, m * k + k * n);
  p.a.assign(all.begin(), all.begin() + std::ptrdiff_t(m * k));
  p.b.assign(all.begin() + std::ptrdiff_t(m * k), all.end());
  return p;
}

struct AgGemmRun {  // ag_gemm.hpp:85-92
  std::vector<std::vector<float>> c;                 // per rank, m x n
  std::vector<std::vector<std::uint64_t>> flag_counts;  // push only
  std::vector<std::vector<float>> gathered;          // per rank, m x k: the operand the GEMM consumed
  std::uint64_t launches = 0;                        // kernels this run launched
  std::vector<tf_taxes> taxes;                       // per rank, measured on the device
};

namespace detail {
inline AgGemmRun run(tf_ag_variant variant, const AgGemmProblem& p, const WorldConfig& cfg) {
  cfg.validate();
  p.validate(cfg.world_size);
  const int W = cfg.world_size;
  const std::size_t kw = p.k / std::size_t(W);
  const bool bf = p.dtype == Dtype::kBF16;
  const bool msh = p.shard == Shard::kM;
  const std::size_t mr = p.m / std::size_t(W);
  const std::size_t esz = bf ? 2 : 4;
  const std::size_t heap = cfg.heap_bytes ? cfg.heap_bytes
                                          : esz * (p.m * kw + 5 * p.m * p.k) + (16u << 20);
  b200::World w(W, cfg.device_list(), heap, cfg.watchdog_secs);
  w.apply(cfg);
  auto shards = w.heap("ag.a", esz * (msh ? mr * p.k : p.m * kw));
  std::vector<void*> B(W), C(W);
  auto pack = [&](const float* src, std::size_t n) {
    std::vector<uint8_t> out(n * esz);
    if (bf)
      for (std::size_t i = 0; i < n; ++i) reinterpret_cast<uint16_t*>(out.data())[i] = b200::to_bf16(src[i]);
    else
      std::memcpy(out.data(), src, n * 4);
    return out;
  };
  const auto hb = pack(p.b.data(), p.b.size());
  for (int r = 0; r < W; ++r) {
    // fill_shard (ag_gemm.hpp:103-112): columns [r*kw, (r+1)*kw) of A, or
    // (Shard::kM) rows [r*m/W, (r+1)*m/W).
    std::vector<float> shard;
    if (msh) {
      shard.assign(p.a.begin() + std::ptrdiff_t(std::size_t(r) * mr * p.k),
                   p.a.begin() + std::ptrdiff_t(std::size_t(r + 1) * mr * p.k));
    } else {
      shard.resize(p.m * kw);
      for (std::size_t i = 0; i < p.m; ++i)
        std::memcpy(&shard[i * kw], &p.a[i * p.k + std::size_t(r) * kw], kw * 4);
    }
    const auto hs = pack(shard.data(), shard.size());
    w.put(shards[r], hs.data(), hs.size());
    B[r] = w.device(r, hb.size());
    w.put(B[r], hb.data(), hb.size());
    C[r] = w.device(r, esz * p.m * p.n);
  }
  // setup_fence (ag_gemm.hpp:189-191, fabric.hpp:586-592): every shard is
  // placed before any rank's schedule reads or pushes it; untimed, so the
  // tax meter starts after it.
  b200::check(tf_world_barrier(w.w, -1));
  b200::check(tf_tax_reset(w.w));
  tf_ag_shape sh{p.m, p.n, p.k, p.tiles.bm, p.tiles.bn, p.tiles.bk, bf ? TF_BF16 : TF_F32,
                 static_cast<tf_ag_shard>(p.shard)};
  const std::uint64_t l0 = tf_launch_count(w.w);
  b200::check(tf_ag_gemm(w.w, variant, &sh, shards.data(), const_cast<const void* const*>(B.data()),
                         C.data(), nullptr, nullptr));
  AgGemmRun out;
  out.launches = tf_launch_count(w.w) - l0;
  out.taxes = w.taxes();
  auto unpack = [&](const void* dev, std::size_t n) {
    std::vector<uint8_t> raw(n * esz);
    w.put(raw.data(), dev, raw.size());
    std::vector<float> f(n);
    for (std::size_t i = 0; i < n; ++i)
      f[i] = bf ? b200::from_bf16(reinterpret_cast<uint16_t*>(raw.data())[i])
                : reinterpret_cast<float*>(raw.data())[i];
    return f;
  };
  for (int r = 0; r < W; ++r) {
    out.c.push_back(unpack(C[r], p.m * p.n));
    {
      // The operand rank r's GEMM consumed (tf_ag_gathered), every schedule.
      std::vector<uint8_t> raw(esz * p.m * p.k);
      b200::check(tf_ag_gathered(w.w, r, raw.data(), raw.size()));
      std::vector<float> f(p.m * p.k);
      for (std::size_t i = 0; i < f.size(); ++i)
        f[i] = bf ? b200::from_bf16(reinterpret_cast<uint16_t*>(raw.data())[i])
                  : reinterpret_cast<float*>(raw.data())[i];
      out.gathered.push_back(std::move(f));
    }
    if (variant == TF_AG_PUSH) {
      std::size_t cnt = 0;
      b200::check(tf_ag_flag_counts(w.w, r, nullptr, 0, &cnt));
      std::vector<std::uint64_t> f(cnt);
      b200::check(tf_ag_flag_counts(w.w, r, f.data(), cnt, &cnt));
      out.flag_counts.push_back(std::move(f));
    }
  }
  return out;
}
}  // namespace detail

// ag_gemm.hpp:134 / :185 / :228
inline AgGemmRun run_baseline(const AgGemmProblem& p, const WorldConfig& cfg) {
  return detail::run(TF_AG_BASELINE, p, cfg);
}
inline AgGemmRun run_pull(const AgGemmProblem& p, const WorldConfig& cfg) {
  return detail::run(TF_AG_PULL, p, cfg);
}
inline AgGemmRun run_push(const AgGemmProblem& p, const WorldConfig& cfg) {
  return detail::run(TF_AG_PUSH, p, cfg);
}

}  // namespace ag

// ============================ flash_decode.hpp ================================
namespace fd {

enum class Variant { kBsp = TF_FD_BSP, kIndependentAg = TF_FD_INDEPENDENT_AG,
                     kFineWaits = TF_FD_FINE_WAITS, kFused = TF_FD_FUSED };  // :50

inline const char* to_string(Variant v) {  // :52-64
  switch (v) {
    case Variant::kBsp: return "bsp";
    case Variant::kIndependentAg: return "independent_ag";
    case Variant::kFineWaits: return "fine_waits";
    case Variant::kFused: return "fused";
  }
  return "unknown";
}

struct DecodeProblem {  // :66-88, + batch and kv_heads (GQA)
  int heads = 0;
  int head_dim = 0;
  std::size_t kv_len = 0;
  float scale = 0.0f;
  std::vector<float> q;  // batch x heads x head_dim
  std::vector<float> k;  // batch x kv_heads x kv_len x head_dim
  std::vector<float> v;
  int batch = 1;
  int kv_heads = 0;  // 0 -> heads (MHA, the reference)
  Dtype dtype = Dtype::kF32;
  int kvh() const { return kv_heads ? kv_heads : heads; }
  void validate(int world_size) const {
    if (heads < 1 || head_dim < 1 || kv_len < 1)
      throw ConfigError("flash_decode: heads, head_dim, kv_len must be >= 1");
    if (kv_len % std::size_t(world_size) != 0)
      throw ConfigError("flash_decode: kv_len = " + std::to_string(kv_len) +
                        " must be divisible by world_size = " + std::to_string(world_size));
    if (!std::isfinite(scale)) throw ConfigError("flash_decode: scale must be finite");
  }
};

// :90-106: scale 1/sqrt(d); q, then K, then V from one stream.
inline DecodeProblem make_problem(std::uint64_t seed, int heads, int head_dim, std::size_t kv_len) {
  DecodeProblem p;
  p.heads = heads;
  p.head_dim = head_dim;
  p.kv_len = kv_len;
  p.scale = 1.0f / std::sqrt(static_cast<float>(head_dim));
  const std::size_t hd = std::size_t(heads) * head_dim;
  std::vector<float> all = uniform_reals(seed, hd + 2 * hd * kv_len);
  auto it = all.begin();
  p.q.assign(it, it + std::ptrdiff_t(hd));
  it += std::ptrdiff_t(hd);
  p.k.assign(it, it + std::ptrdiff_t(hd * kv_len));
  it += std::ptrdiff_t(hd * kv_len);
  p.v.assign(it, all.end());
  return p;
}

struct FdOptions {  // :108-114
  bool fold_by_arrival = false;  // fused only: fold in arrival order (not bitwise reproducible)
  bool owner_combine = false;    // extension: fused with per-group owners (TF_FD_FUSED_OWNER)
  // Extension (SPEC.md:327 lists paged KV as a non-goal): > 0 runs the problem
  // through tf_flash_decode_paged with pages of this many keys (a power of
  // two), scattered in reverse order over each rank's pool (HND layout).
  int page_size = 0;
};

struct FdRun {  // :116-123
  std::vector<std::vector<float>> out;                   // per rank, batch x heads x d
  std::vector<std::vector<std::uint64_t>> flag_counts;   // push-style variants
  std::vector<std::vector<float>> inbox;                 // per rank, W x batch x heads x (d+2)
  std::uint64_t launches = 0;
  std::vector<tf_taxes> taxes;                           // per rank, measured on the device
};

inline FdRun run_fd(const DecodeProblem& p, Variant variant, const WorldConfig& cfg,
                    const FdOptions& opts = {}) {
  if (opts.owner_combine) {
    if (variant != Variant::kFused || opts.fold_by_arrival)
      throw ConfigError("owner_combine applies to the fused schedule (ascending fold) only");
    variant = static_cast<Variant>(TF_FD_FUSED_OWNER);
  }
  if (opts.fold_by_arrival) {
    if (variant != Variant::kFused) throw ConfigError("fold_by_arrival applies to the fused schedule only");
    variant = static_cast<Variant>(TF_FD_FUSED_BY_ARRIVAL);
  }
  cfg.validate();
  p.validate(cfg.world_size);
  const int W = cfg.world_size;
  const int B = p.batch, H = p.heads, Hkv = p.kvh(), d = p.head_dim;
  const std::size_t L = p.kv_len, ln = L / std::size_t(W);
  const bool bf = p.dtype == Dtype::kBF16;
  const std::size_t esz = bf ? 2 : 4;
  const std::size_t row = std::size_t(B) * H * (d + 2);
  const std::size_t heap = cfg.heap_bytes ? cfg.heap_bytes
                                          : 4 * W * row * 6 + 4 * std::size_t(B) * Hkv * 4096 * (d + 2) * 8 + (16u << 20);
  b200::World w(W, cfg.device_list(), heap, cfg.watchdog_secs);
  w.apply(cfg);
  auto inbox = w.heap("fd.inbox.user", 4 * W * row);
  auto pack = [&](const float* src, std::size_t n) {
    std::vector<uint8_t> out(n * esz);
    if (bf)
      for (std::size_t i = 0; i < n; ++i) reinterpret_cast<uint16_t*>(out.data())[i] = b200::to_bf16(src[i]);
    else
      std::memcpy(out.data(), src, n * 4);
    return out;
  };
  std::vector<void*> Q(W), K(W), V(W), O(W), T(W);
  const int ps = opts.page_size;
  const std::size_t pps = ps > 0 ? (ln + std::size_t(ps) - 1) / std::size_t(ps) : 0;
  const std::size_t npages = std::size_t(B) * pps;
  const auto hq = pack(p.q.data(), p.q.size());
  for (int r = 0; r < W; ++r) {
    // slice_shard (flash_decode.hpp:140-160): positions [r*ln, (r+1)*ln) of every head.
    std::vector<float> ks(std::size_t(B) * Hkv * ln * d), vs(ks.size());
    for (std::size_t bh = 0; bh < std::size_t(B) * Hkv; ++bh) {
      std::memcpy(&ks[bh * ln * d], &p.k[(bh * L + std::size_t(r) * ln) * d], ln * d * 4);
      std::memcpy(&vs[bh * ln * d], &p.v[(bh * L + std::size_t(r) * ln) * d], ln * d * 4);
    }
    if (ps > 0) {
      // HND page pools [npages][Hkv][ps][d]; sequence b's page j lives in
      // pool slot npages - 1 - (b * pps + j) (reverse order); unused tail
      // keys of the last page are zero.
      std::vector<float> pk(npages * Hkv * std::size_t(ps) * d, 0.f), pv(pk.size(), 0.f);
      std::vector<int> tbl(npages);
      for (int b = 0; b < B; ++b)
        for (std::size_t j = 0; j < pps; ++j) {
          const std::size_t slot = npages - 1 - (std::size_t(b) * pps + j);
          tbl[std::size_t(b) * pps + j] = int(slot);
          for (int h = 0; h < Hkv; ++h)
            for (std::size_t x = j * ps; x < std::min(ln, (j + 1) * std::size_t(ps)); ++x) {
              const std::size_t src = ((std::size_t(b) * Hkv + h) * ln + x) * d;
              const std::size_t dst = ((slot * Hkv + h) * ps + (x - j * ps)) * d;
              std::memcpy(&pk[dst], &ks[src], d * 4);
              std::memcpy(&pv[dst], &vs[src], d * 4);
            }
        }
      ks.swap(pk);
      vs.swap(pv);
      T[r] = w.device(r, tbl.size() * sizeof(int));
      w.put(T[r], tbl.data(), tbl.size() * sizeof(int));
    }
    const auto hk = pack(ks.data(), ks.size()), hv = pack(vs.data(), vs.size());
    Q[r] = w.device(r, hq.size());
    K[r] = w.device(r, hk.size());
    V[r] = w.device(r, hv.size());
    O[r] = w.device(r, esz * std::size_t(B) * H * d);
    w.put(Q[r], hq.data(), hq.size());
    w.put(K[r], hk.data(), hk.size());
    w.put(V[r], hv.data(), hv.size());
  }
  tf_fd_shape sh{B, H, Hkv, d, L, p.scale, bf ? TF_BF16 : TF_F32, bf ? TF_BF16 : TF_F32};
  const std::uint64_t l0 = tf_launch_count(w.w);
  if (ps > 0) {
    const tf_fd_paged pl{ps, int(pps), int(npages), TF_PAGED_HND};
    b200::check(tf_flash_decode_paged(w.w, static_cast<tf_fd_variant>(variant), &sh, &pl,
                                      const_cast<const void* const*>(Q.data()),
                                      const_cast<const void* const*>(K.data()),
                                      const_cast<const void* const*>(V.data()),
                                      const_cast<const void* const*>(T.data()), O.data(), inbox.data(), nullptr));
  } else {
    b200::check(tf_flash_decode(w.w, static_cast<tf_fd_variant>(variant), &sh,
                                const_cast<const void* const*>(Q.data()), const_cast<const void* const*>(K.data()),
                                const_cast<const void* const*>(V.data()), O.data(), inbox.data(), nullptr));
  }
  FdRun out;
  out.launches = tf_launch_count(w.w) - l0;
  out.taxes = w.taxes();
  for (int r = 0; r < W; ++r) {
    std::vector<uint8_t> raw(esz * std::size_t(B) * H * d);
    w.put(raw.data(), O[r], raw.size());
    std::vector<float> o(std::size_t(B) * H * d);
    for (std::size_t i = 0; i < o.size(); ++i)
      o[i] = bf ? b200::from_bf16(reinterpret_cast<uint16_t*>(raw.data())[i]) : reinterpret_cast<float*>(raw.data())[i];
    out.out.push_back(std::move(o));
    std::vector<float> box(W * row);
    w.put(box.data(), inbox[r], box.size() * 4);
    out.inbox.push_back(std::move(box));
    if (variant != Variant::kBsp) {
      std::vector<std::uint64_t> f(W);
      std::size_t cnt = 0;
      b200::check(tf_fd_flag_counts(w.w, r, f.data(), f.size(), &cnt));
      f.resize(cnt);
      out.flag_counts.push_back(std::move(f));
    }
  }
  return out;
}

// :212 / :256 / :301 / :348
inline FdRun run_bsp(const DecodeProblem& p, const WorldConfig& cfg) { return run_fd(p, Variant::kBsp, cfg); }
inline FdRun run_independent_ag(const DecodeProblem& p, const WorldConfig& cfg) {
  return run_fd(p, Variant::kIndependentAg, cfg);
}
inline FdRun run_fine_waits(const DecodeProblem& p, const WorldConfig& cfg) {
  return run_fd(p, Variant::kFineWaits, cfg);
}
inline FdRun run_fused(const DecodeProblem& p, const WorldConfig& cfg, const FdOptions& opts = {}) {
  return run_fd(p, Variant::kFused, cfg, opts);
}

}  // namespace fd
}  // namespace tilefabric
