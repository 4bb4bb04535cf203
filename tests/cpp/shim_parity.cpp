// shim_parity.cpp -- the reference's own test bodies, run against the C++
// drop-in (include/tilefabric_b200/tilefabric.hpp) on the GPU.
//
// Each TEST mirrors a case of proj/tests/{ag_gemm,flash_decode}_test.cpp or
// acceptance_test.cpp (cited per test).  The checker is the CPU oracle
// (oracle/tf_oracle.c, pinned to the reference by tests/test_oracle_golden.py).
// Built by __graft_entry__.build(); run by tests/test_cpp_shim_gpu.py.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "tilefabric_b200/tilefabric.hpp"

extern "C" {
void tfo_gemm(const float* a, const float* b, size_t m, size_t n, size_t k, float* c);
void tfo_attention(const float* q, const float* k, const float* v, size_t heads, size_t d, size_t L,
                   float scale, float* out, float* scratch);
double tfo_max_head_relative_error(const float* a, const float* b, int heads, int d);
}

using namespace tilefabric;

static int g_fail = 0, g_checks = 0;
#define EXPECT_TRUE(c)                                                         \
  do {                                                                         \
    ++g_checks;                                                                \
    if (!(c)) {                                                                \
      ++g_fail;                                                                \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);             \
    }                                                                          \
  } while (0)
#define EXPECT_THROW(stmt, Exc)                                                \
  do {                                                                         \
    bool thrown = false;                                                       \
    try {                                                                      \
      stmt;                                                                    \
    } catch (const Exc&) {                                                     \
      thrown = true;                                                           \
    } catch (...) {                                                            \
    }                                                                          \
    EXPECT_TRUE(thrown);                                                       \
  } while (0)

static bool bitwise(const std::vector<float>& a, const std::vector<float>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 4) == 0;
}

static std::vector<float> oracle_gemm(const ag::AgGemmProblem& p) {
  std::vector<float> c(p.m * p.n);
  tfo_gemm(p.a.data(), p.b.data(), p.m, p.n, p.k, c.data());
  return c;
}

static std::vector<float> oracle_attention(const fd::DecodeProblem& p) {
  std::vector<float> out(std::size_t(p.heads) * p.head_dim), scratch(p.kv_len);
  tfo_attention(p.q.data(), p.k.data(), p.v.data(), p.heads, p.head_dim, p.kv_len, p.scale, out.data(),
                scratch.data());
  return out;
}

static WorldConfig quick_config(int w) {  // ag_gemm_test.cpp:34-39
  WorldConfig cfg;
  cfg.world_size = w;
  return cfg;
}

static void run_test(const char* name, const std::function<void()>& body) {
  const int before = g_fail;
  try {
    body();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("  EXCEPTION %s\n", e.what());
  }
  std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

int main() {
  // ag_gemm_test.cpp:42-48
  run_test("AgProblem.ValidatesShardability", [] {
    auto p = ag::make_problem(1, 4, 4, 12);
    p.validate(4);
    EXPECT_THROW(p.validate(5), ConfigError);
    p.m = 0;
    EXPECT_THROW(p.validate(4), ConfigError);
  });
  // ag_gemm_test.cpp:50-57
  run_test("AgProblem.SeedFullyDeterminesInputs", [] {
    const auto p1 = ag::make_problem(99, 3, 5, 8), p2 = ag::make_problem(99, 3, 5, 8);
    EXPECT_TRUE(p1.a == p2.a && p1.b == p2.b);
    EXPECT_TRUE(ag::make_problem(100, 3, 5, 8).a != p1.a);
  });
  // ag_gemm_test.cpp:62-83
  run_test("AgGemm.AllVariantsMatchNaiveGemmBitwise", [] {
    TileSpec tiles;
    tiles.bm = 4;
    tiles.bn = 5;
    tiles.bk = 3;
    const auto p = ag::make_problem(7, 13, 9, 16, tiles);
    const auto oracle = oracle_gemm(p);
    for (const int w : {1, 2, 4}) {
      const auto cfg = quick_config(w);
      const auto base = ag::run_baseline(p, cfg), pull = ag::run_pull(p, cfg), push = ag::run_push(p, cfg);
      for (int r = 0; r < w; ++r) {
        EXPECT_TRUE(bitwise(base.c[r], oracle));
        EXPECT_TRUE(bitwise(pull.c[r], oracle));
        EXPECT_TRUE(bitwise(push.c[r], oracle));
      }
    }
  });
  // ag_gemm_test.cpp:85-92
  run_test("AgGemm.SingleElementAndSingleRankEdges", [] {
    const auto p = ag::make_problem(3, 1, 1, 1);
    const auto oracle = oracle_gemm(p);
    const auto cfg = quick_config(1);
    EXPECT_TRUE(bitwise(ag::run_baseline(p, cfg).c[0], oracle));
    EXPECT_TRUE(bitwise(ag::run_pull(p, cfg).c[0], oracle));
    EXPECT_TRUE(bitwise(ag::run_push(p, cfg).c[0], oracle));
  });
  // ag_gemm_test.cpp:94-97
  run_test("AgGemm.RejectsNonDivisibleK", [] {
    const auto p = ag::make_problem(5, 4, 4, 10);
    EXPECT_THROW(ag::run_pull(p, quick_config(4)), ConfigError);
  });
  // cli_test.cpp:162-173 -- config 1: W=2, 8x8x8, seed 1, max_error == 0.0
  run_test("Cli.PullWorld2Verify", [] {
    const auto p = ag::make_problem(1, 8, 8, 8);
    const auto oracle = oracle_gemm(p);
    const auto run = ag::run_pull(p, quick_config(2));
    double max_error = 0.0;
    for (std::size_t i = 0; i < oracle.size(); ++i)
      max_error = std::max(max_error, double(std::fabs(run.c[0][i] - oracle[i])));
    EXPECT_TRUE(max_error == 0.0);
  });
  // ag_gemm_test.cpp:146-170 -- every push flag ends at exactly one signal.
  run_test("AgGemm.PushStructure", [] {
    const int w = 4;
    const auto p = ag::make_problem(13, 8, 8, 16);
    const auto run = ag::run_push(p, quick_config(w));
    const std::size_t kw = p.k / w, n_kb = (kw + p.tiles.bk - 1) / p.tiles.bk;
    EXPECT_TRUE(run.launches == std::uint64_t(2 * w));
    for (const auto& counts : run.flag_counts) {
      EXPECT_TRUE(counts.size() == w * n_kb);
      for (auto c : counts) EXPECT_TRUE(c == 1);
    }
    for (const auto& g : run.gathered) EXPECT_TRUE(bitwise(g, p.a));
  });
  // acceptance_test.cpp:90-135 -- the AG grid, bitwise.
  run_test("Acceptance.AgGridBitwise", [] {
    std::uint64_t seed = 1;
    for (int w : {1, 2, 4, 8})
      for (std::size_t m : {1, 16, 64})
        for (std::size_t n : {8, 32, 64})
          for (std::size_t k : {8, 32, 64}) {
            if (k % std::size_t(w)) continue;
            const auto p = ag::make_problem(seed++, m, n, k);
            const auto oracle = oracle_gemm(p);
            const auto run = (seed % 3 == 0) ? ag::run_push(p, quick_config(w))
                             : (seed % 3 == 1) ? ag::run_pull(p, quick_config(w))
                                               : ag::run_baseline(p, quick_config(w));
            for (const auto& c : run.c) EXPECT_TRUE(bitwise(c, oracle));
          }
  });
  // Extension (SPEC.md:265 leaves row sharding out): A sharded by rows gives the
  // K-sharded baseline's C and gathered operand bit for bit (bf16 path).
  run_test("Extension.AgRowShardedMatchesColumnShardedBaseline", [] {
    auto p = ag::make_problem(21, 256, 64, 128);
    p.dtype = Dtype::kBF16;
    const auto base = ag::run_baseline(p, quick_config(2));
    p.shard = ag::Shard::kM;
    for (auto* fn : {&ag::run_pull, &ag::run_baseline}) {
      const auto run = (*fn)(p, quick_config(2));
      for (int r = 0; r < 2; ++r) {
        EXPECT_TRUE(bitwise(run.c[r], base.c[r]));
        EXPECT_TRUE(bitwise(run.gathered[r], base.gathered[r]));
      }
    }
    auto q = ag::make_problem(21, 64, 64, 128);  // m not a multiple of 128 * W
    q.dtype = Dtype::kBF16;
    q.shard = ag::Shard::kM;
    EXPECT_THROW(ag::run_pull(q, quick_config(2)), ShapeError);
  });
  // Extension (SPEC.md:327 lists paged KV as a non-goal): a paged run is the
  // contiguous run of the same logical KV, bit for bit, every schedule.
  run_test("Extension.FdPagedEqualsContiguous", [] {
    const auto p = fd::make_problem(8, 2, 16, 200);
    for (const int w : {1, 2})
      for (auto v : {fd::Variant::kBsp, fd::Variant::kFineWaits, fd::Variant::kFused}) {
        fd::FdOptions paged;
        paged.page_size = 16;
        const auto base = fd::run_fd(p, v, quick_config(w)), pg = fd::run_fd(p, v, quick_config(w), paged);
        for (int r = 0; r < w; ++r) EXPECT_TRUE(bitwise(pg.out[r], base.out[r]));
      }
  });
  // flash_decode_test.cpp:45-56
  run_test("FdProblem.ValidatesShardabilityAndScale", [] {
    auto p = fd::make_problem(1, 2, 4, 64);
    p.validate(4);
    EXPECT_THROW(p.validate(3), ConfigError);
    p.scale = INFINITY;
    EXPECT_THROW(p.validate(4), ConfigError);
    EXPECT_TRUE(fd::make_problem(1, 2, 16, 8).scale == 0.25f);
  });
  // flash_decode_test.cpp:63-88
  run_test("FlashDecode.AllVariantsAgreeBitwiseAndMatchOracle", [] {
    const auto p = fd::make_problem(5, 2, 8, 96);
    const auto oracle = oracle_attention(p);
    for (const int w : {1, 2, 4}) {
      std::vector<float> first;
      for (auto v : {fd::Variant::kBsp, fd::Variant::kIndependentAg, fd::Variant::kFineWaits,
                     fd::Variant::kFused}) {
        const auto run = fd::run_fd(p, v, quick_config(w));
        EXPECT_TRUE(int(run.out.size()) == w);
        for (const auto& out : run.out) {
          if (first.empty()) first = out;
          EXPECT_TRUE(bitwise(out, first));
        }
        EXPECT_TRUE(tfo_max_head_relative_error(run.out[0].data(), oracle.data(), p.heads, p.head_dim) <= 1e-5);
      }
    }
  });
  // flash_decode_test.cpp:167-196 -- flags == 1, inbox identical on every rank.
  run_test("FlashDecode.FusedFlagsAndInbox", [] {
    const auto p = fd::make_problem(1, 2, 4, 64);
    const auto run = fd::run_fused(p, quick_config(4));
    for (const auto& counts : run.flag_counts) {
      EXPECT_TRUE(counts.size() == 4);
      for (auto c : counts) EXPECT_TRUE(c == 1);
    }
    for (const auto& box : run.inbox) EXPECT_TRUE(bitwise(box, run.inbox[0]));
    EXPECT_TRUE(run.launches == 1);  // one persistent launch per device
  });
  // acceptance_test.cpp:140-202 (sampled) -- oracle 1e-5, bitwise across ranks.
  run_test("Acceptance.FdGrid", [] {
    std::uint64_t seed = 1;
    for (int w : {1, 2, 4, 8})
      for (int h : {1, 2, 8})
        for (int d : {4, 16, 128})
          for (std::size_t kv : {64, 512, 4096}) {
            if (kv == 4096 && (h != 8 || d != 128)) continue;
            const auto p = fd::make_problem(seed++, h, d, kv);
            const auto oracle = oracle_attention(p);
            const auto run = fd::run_fused(p, quick_config(w));
            EXPECT_TRUE(tfo_max_head_relative_error(run.out[0].data(), oracle.data(), h, d) <= 1e-5);
            for (const auto& out : run.out) EXPECT_TRUE(bitwise(out, run.out[0]));
          }
  });
  // flash_decode.hpp:377-408: arrival-order fold -- same result up to
  // round-off (not bitwise reproducible), fused schedule only.
  run_test("FdOptions.FoldByArrival", [] {
    fd::FdOptions o;
    o.fold_by_arrival = true;
    const auto p = fd::make_problem(5, 2, 8, 96);
    const auto oracle = oracle_attention(p);
    for (int w : {1, 2, 4}) {
      const auto run = fd::run_fused(p, quick_config(w), o);
      for (const auto& out : run.out)
        EXPECT_TRUE(tfo_max_head_relative_error(out.data(), oracle.data(), p.heads, p.head_dim) <= 1e-5);
      for (const auto& counts : run.flag_counts)
        for (auto c : counts) EXPECT_TRUE(c == 1);
    }
    EXPECT_THROW(fd::run_fd(p, fd::Variant::kBsp, quick_config(2), o), ConfigError);
  });
  // flash_decode_test.cpp:250-286: a 50 ms straggler; rank 0 pays it as a
  // signal wait on source 1, nobody pays a barrier, the straggler barely waits.
  run_test("FlashDecode.FusedWaitsTargetTheStraggler", [] {
    auto cfg = quick_config(2);
    inject_skew(cfg, 1, std::chrono::milliseconds(50));
    const auto p = fd::make_problem(14, 2, 4, 64);
    const auto run = fd::run_fused(p, cfg);
    EXPECT_TRUE(run.taxes.size() == 2);
    EXPECT_TRUE(run.taxes[0].wait_idle_ns >= 45000000ull);
    EXPECT_TRUE(run.taxes[1].wait_idle_ns < 25000000ull);
    for (const auto& t : run.taxes) EXPECT_TRUE(t.bulk_sync_ns == 0 && t.barrier_waits == 0);
    EXPECT_THROW(inject_skew(cfg, 2, std::chrono::milliseconds(1)), ConfigError);
    EXPECT_THROW(inject_skew(cfg, 0, std::chrono::milliseconds(-1)), ConfigError);
  });
  // acceptance_test.cpp:207-243: barriers per rank -- bsp 2, fused 0.
  run_test("Acceptance.StructuralTaxCounts", [] {
    const auto p = fd::make_problem(7, 2, 8, 64);
    const auto bsp = fd::run_bsp(p, quick_config(4));
    const auto fused = fd::run_fused(p, quick_config(4));
    for (int r = 0; r < 4; ++r) {
      EXPECT_TRUE(bsp.taxes[r].barrier_waits == 2);
      EXPECT_TRUE(fused.taxes[r].barrier_waits == 0);
    }
    const auto agp = ag::make_problem(7, 8, 8, 16);
    for (const auto& t : ag::run_pull(agp, quick_config(4)).taxes)
      EXPECT_TRUE(t.barrier_waits == 0 && t.staged_bytes == 0);
  });
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
