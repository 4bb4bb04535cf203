// tilefabric_bench.cpp -- the reference's benchmark driver (proj/tools/bench.cpp,
// `tilefabric-bench`) on the B200 kernels: same flags, presets
// (tf/presets.hpp), CSV / JSON / gnuplot outputs and exit codes, so scripts
// written against the reference CLI run unchanged.
//
//   tilefabric-bench --pattern ag-pull --world-size 2 --m 8 --n 8 --k 8 --verify --iters 1
//   tilefabric-bench --preset desk-fd --verify --out results/fd
//   tilefabric-bench --patterns fd-bsp,fd-fused --sweep-kv 8192,131072 --dtype bf16
//
// What changes on the GPU:
//   * an iteration's makespan is host wall-clock from the launch of the
//     pattern to the sync of every rank's stream (SURVEY §8(d) methodology),
//     on inputs placed in HBM once per cell;
//   * bulk_sync_tax / wait_idle are the device-measured barrier and signal
//     wait times (tf_tax_report, summed over ranks); launch_tax stays the
//     reference's count x --launch-cost-us ledger (taxmeter.hpp:51);
//   * --skew delays the rank's first compute stage on the device;
//   * extensions: --dtype f32|bf16 (f32 = the exact-order path, bitwise equal
//     to the reference), --batch / --kv-heads (GQA decode), --devices.
// --verify checks against brute-force restatements of reference::gemm and
// reference::attention (reference.hpp:36-132) compiled into this tool.
//
// Exit codes: 0 success; 1 verification mismatch or runtime failure; 2
// invalid flags or constraint violations (bench.cpp:31-33).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "tilefabric_b200/tilefabric.hpp"

namespace tf = tilefabric;

namespace {

const std::vector<std::string> kAgPatterns = {"ag-baseline", "ag-pull", "ag-push"};
const std::vector<std::string> kFdPatterns = {"fd-bsp", "fd-ag", "fd-wait", "fd-fused", "fd-owner"};
constexpr const char* kAgBaseline = "ag-baseline";
constexpr const char* kFdBaseline = "fd-bsp";

bool contains(const std::vector<std::string>& v, const std::string& s) {
  return std::find(v.begin(), v.end(), s) != v.end();
}

tf_fd_variant fd_variant(const std::string& p, bool arrival) {
  if (p == "fd-bsp") return TF_FD_BSP;
  if (p == "fd-ag") return TF_FD_INDEPENDENT_AG;
  if (p == "fd-wait") return TF_FD_FINE_WAITS;
  if (p == "fd-owner") return TF_FD_FUSED_OWNER;  // GPU extension: owner-combine
  return arrival ? TF_FD_FUSED_BY_ARRIVAL : TF_FD_FUSED;
}

tf_ag_variant ag_variant(const std::string& p) {
  if (p == "ag-baseline") return TF_AG_BASELINE;
  if (p == "ag-pull") return TF_AG_PULL;
  return TF_AG_PUSH;
}

double percentile(std::vector<double> v, double q) {  // bench.cpp:82-93
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double pos = q * double(v.size() - 1);
  const auto lo = std::size_t(pos);
  const auto hi = std::min(lo + 1, v.size() - 1);
  return v[lo] + (pos - double(lo)) * (v[hi] - v[lo]);
}

std::string csv_escape(const std::string& s) {
  if (s.find_first_of(",\"\n") == std::string::npos) return s;
  std::string out = "\"";
  for (char c : s) {
    if (c == '"') out += '"';
    out += c;
  }
  return out + '"';
}

std::string json_str(const std::string& s) {
  std::string out = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') out += '\\';
    if (c == '\n') {
      out += "\\n";
      continue;
    }
    out += c;
  }
  return out + '"';
}

std::string num(double v) {
  std::ostringstream os;
  os.precision(17);
  os << v;
  return os.str();
}

// ---- presets (tf/presets.hpp) ----------------------------------------------
struct Preset {
  std::string name, family;
  int world_size = 8;
  std::vector<std::string> patterns;
  std::size_t n = 0, k = 0;
  std::vector<std::size_t> m_sweep;
  int heads = 0, head_dim = 0;
  std::vector<std::size_t> kv_sweep;
};

std::vector<std::size_t> powers_of_two(std::size_t lo, std::size_t hi) {
  std::vector<std::size_t> out;
  for (std::size_t v = lo; v <= hi; v *= 2) out.push_back(v);
  return out;
}

const std::vector<Preset>& presets() {
  static const std::vector<Preset> all = [] {
    std::vector<Preset> v;
    Preset ag{"paper-ag-gemm", "ag", 8, kAgPatterns, 28672, 8192, powers_of_two(1, 8192), 0, 0, {}};
    v.push_back(ag);
    Preset desk_ag = ag;
    desk_ag.name = "desk-ag-gemm";
    desk_ag.n = 448;
    desk_ag.k = 128;
    desk_ag.m_sweep = powers_of_two(1, 128);
    v.push_back(desk_ag);
    Preset fd{"paper-fd", "fd", 8, kFdPatterns, 0, 0, {}, 96, 128, powers_of_two(8192, 131072)};
    v.push_back(fd);
    Preset desk_fd = fd;
    desk_fd.name = "desk-fd";
    desk_fd.heads = 8;
    desk_fd.head_dim = 32;
    desk_fd.kv_sweep = powers_of_two(2048, 32768);
    v.push_back(desk_fd);
    return v;
  }();
  return all;
}

// ---- options (bench.cpp:131-152 + GPU extensions) ----------------------------
struct Options {
  std::vector<std::string> patterns;
  int world_size = 4;
  std::size_t m = 64, n = 64, k = 64;
  tf::TileSpec tiles;
  int heads = 8, head_dim = 32;
  std::size_t kv_len = 2048;
  std::vector<std::size_t> sweep_m, sweep_kv;
  std::vector<std::string> skew_specs;
  double launch_cost_us = 20.0;
  int iters = 500, warmup = 100;
  std::uint64_t seed = 1;
  bool verify = false, dry_run = false, fd_arrival_order = false;
  std::string out, preset;
  // GPU extensions
  std::string dtype = "f32";
  int batch = 1, kv_heads = 0;
  std::vector<int> devices;

  bool fd_family = false;
  std::vector<std::size_t> values;
  std::set<std::string> given;  // flags that appeared on the command line
  bool has(const std::string& f) const { return given.count(f) != 0; }
  bool bf16() const { return dtype == "bf16"; }
};

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct HelpRequested {};

const char* kUsage =
    "Fused communication/computation patterns over a symmetric heap on B200: "
    "all-gather GEMM and distributed decode, with per-pattern tax accounting.\n"
    "Usage: tilefabric-bench [OPTIONS]\n\n"
    "Options:\n"
    "  -h,--help                 Print this help message and exit\n"
    "  --pattern TEXT            One pattern: ag-baseline|ag-pull|ag-push|fd-bsp|fd-ag|fd-wait|fd-fused\n"
    "                            (GPU extension: fd-owner, fused with owner-combine)\n"
    "  --patterns TEXT,...       Comma-separated pattern list (sweep mode); excludes --pattern\n"
    "  --preset TEXT             Named configuration: paper-ag-gemm|desk-ag-gemm|paper-fd|desk-fd\n"
    "  --world-size INT          Ranks in the world\n"
    "  --m, --n, --k UINT        GEMM rows / cols / inner dim (K sharded over ranks)\n"
    "  --bm, --bn, --bk UINT     Tile extents\n"
    "  --heads INT               Attention (query) heads (fd family)\n"
    "  --head-dim INT            Head dimension (fd family)\n"
    "  --kv-len UINT             Key/value sequence length, sharded over ranks\n"
    "  --sweep-m UINT,...        Sweep over m values (ag)\n"
    "  --sweep-kv UINT,...       Sweep over kv-len values (fd)\n"
    "  --skew RANK:MILLIS        Straggler injection (repeatable)\n"
    "  --launch-cost-us FLOAT    Per-launch cost charged by the launch-tax ledger\n"
    "  --iters INT               Timed iterations per cell\n"
    "  --warmup INT              Untimed warmup iterations\n"
    "  --seed UINT               Input generator seed\n"
    "  --verify                  Check outputs against the brute-force references first\n"
    "  --dry-run                 Print the resolved configuration and exit\n"
    "  --fd-arrival-order        fd-fused only: fold partials in arrival order\n"
    "  --out TEXT                Output prefix: PREFIX.csv + PREFIX.json (single) or PREFIX.csv + PREFIX.dat (sweep)\n"
    "GPU extensions:\n"
    "  --dtype f32|bf16          f32: exact-order path (bitwise = reference); bf16: tensor-core path\n"
    "  --batch INT               Decode batch (fd family)\n"
    "  --kv-heads INT            KV heads for GQA (fd family; default = --heads)\n"
    "  --devices INT,...         GPU per rank (default: distinct GPUs when available, else all on GPU 0)\n";

template <class T>
T parse_num(const std::string& flag, const std::string& s) {
  try {
    std::size_t pos = 0;
    T v;
    if constexpr (std::is_same_v<T, double>) {
      v = std::stod(s, &pos);
    } else if constexpr (std::is_signed_v<T>) {
      const long long x = std::stoll(s, &pos);
      if (x < std::numeric_limits<T>::min() || x > std::numeric_limits<T>::max()) throw std::out_of_range(s);
      v = T(x);
    } else {
      if (!s.empty() && s[0] == '-') throw std::invalid_argument(s);
      v = T(std::stoull(s, &pos));
    }
    if (pos != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw ParseError(flag + ": Value " + s + " could not be converted");
  }
}

template <class T>
std::vector<T> parse_list(const std::string& flag, const std::string& s) {
  std::vector<T> out;
  std::string item;
  std::istringstream is(s);
  while (std::getline(is, item, ',')) {
    if constexpr (std::is_same_v<T, std::string>) out.push_back(item);
    else out.push_back(parse_num<T>(flag, item));
  }
  return out;
}

Options parse_args(int argc, char** argv) {
  Options o;
  static const std::set<std::string> flags = {"--verify", "--dry-run", "--fd-arrival-order"};
  static const std::set<std::string> valued = {
      "--pattern", "--patterns", "--preset", "--world-size", "--m", "--n", "--k", "--bm", "--bn", "--bk",
      "--heads", "--head-dim", "--kv-len", "--sweep-m", "--sweep-kv", "--skew", "--launch-cost-us",
      "--iters", "--warmup", "--seed", "--out", "--dtype", "--batch", "--kv-heads", "--devices"};
  std::string pattern;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i], val;
    if (a == "-h" || a == "--help") throw HelpRequested{};
    const auto eq = a.find('=');
    bool inline_val = false;
    if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
      val = a.substr(eq + 1);
      a = a.substr(0, eq);
      inline_val = true;
    }
    if (flags.count(a)) {
      if (inline_val) throw ParseError(a + ": flag takes no value");
      o.given.insert(a);
      if (a == "--verify") o.verify = true;
      if (a == "--dry-run") o.dry_run = true;
      if (a == "--fd-arrival-order") o.fd_arrival_order = true;
      continue;
    }
    if (!valued.count(a))
      throw ParseError("The following argument was not expected: " + std::string(argv[i]));
    if (!inline_val) {
      if (i + 1 >= argc) throw ParseError(a + ": 1 required TEXT missing");
      val = argv[++i];
    }
    if (a != "--skew" && o.given.count(a)) throw ParseError(a + ": option given more than once");
    o.given.insert(a);
    if (a == "--pattern") pattern = val;
    else if (a == "--patterns") o.patterns = parse_list<std::string>(a, val);
    else if (a == "--preset") o.preset = val;
    else if (a == "--world-size") o.world_size = parse_num<int>(a, val);
    else if (a == "--m") o.m = parse_num<std::size_t>(a, val);
    else if (a == "--n") o.n = parse_num<std::size_t>(a, val);
    else if (a == "--k") o.k = parse_num<std::size_t>(a, val);
    else if (a == "--bm") o.tiles.bm = parse_num<std::size_t>(a, val);
    else if (a == "--bn") o.tiles.bn = parse_num<std::size_t>(a, val);
    else if (a == "--bk") o.tiles.bk = parse_num<std::size_t>(a, val);
    else if (a == "--heads") o.heads = parse_num<int>(a, val);
    else if (a == "--head-dim") o.head_dim = parse_num<int>(a, val);
    else if (a == "--kv-len") o.kv_len = parse_num<std::size_t>(a, val);
    else if (a == "--sweep-m") o.sweep_m = parse_list<std::size_t>(a, val);
    else if (a == "--sweep-kv") o.sweep_kv = parse_list<std::size_t>(a, val);
    else if (a == "--skew") o.skew_specs.push_back(val);
    else if (a == "--launch-cost-us") o.launch_cost_us = parse_num<double>(a, val);
    else if (a == "--iters") o.iters = parse_num<int>(a, val);
    else if (a == "--warmup") o.warmup = parse_num<int>(a, val);
    else if (a == "--seed") o.seed = parse_num<std::uint64_t>(a, val);
    else if (a == "--out") o.out = val;
    else if (a == "--dtype") o.dtype = val;
    else if (a == "--batch") o.batch = parse_num<int>(a, val);
    else if (a == "--kv-heads") o.kv_heads = parse_num<int>(a, val);
    else if (a == "--devices") o.devices = parse_list<int>(a, val);
  }
  if (o.has("--pattern") && o.has("--patterns")) throw ParseError("--patterns excludes --pattern");
  if (o.has("--pattern")) o.patterns = {pattern};
  return o;
}

std::pair<int, tf::Duration> parse_skew(const std::string& spec) {  // bench.cpp:113-128
  const auto colon = spec.find(':');
  if (colon == std::string::npos || colon == 0 || colon + 1 == spec.size())
    throw tf::ConfigError("--skew expects RANK:MILLIS, got \"" + spec + "\"");
  try {
    std::size_t p1 = 0, p2 = 0;
    const int rank = std::stoi(spec.substr(0, colon), &p1);
    const double millis = std::stod(spec.substr(colon + 1), &p2);
    if (p1 != colon || p2 != spec.size() - colon - 1) throw std::invalid_argument(spec);
    return {rank, std::chrono::duration_cast<tf::Duration>(std::chrono::duration<double, std::milli>(millis))};
  } catch (const std::exception&) {
    throw tf::ConfigError("--skew expects RANK:MILLIS, got \"" + spec + "\"");
  }
}

// ---- brute-force checkers (reference.hpp:36-132, restated) ------------------
std::vector<float> check_gemm(const std::vector<float>& a, const std::vector<float>& b, std::size_t m,
                              std::size_t n, std::size_t k) {
  std::vector<float> c(m * n, 0.0f);
  for (std::size_t i = 0; i < m; ++i)
    for (std::size_t j = 0; j < n; ++j) {
      float acc = 0.0f;
      for (std::size_t p = 0; p < k; ++p) acc += a[i * k + p] * b[p * n + j];
      c[i * n + j] = acc;
    }
  return c;
}

// Two-pass softmax attention per (batch, q-head); q-head h reads kv head
// h / (Hq / Hkv) (GQA; MHA when Hkv == Hq is reference::attention exactly).
std::vector<float> check_attention(const std::vector<float>& q, const std::vector<float>& k,
                                   const std::vector<float>& v, int B, int Hq, int Hkv, int d, std::size_t L,
                                   float scale) {
  std::vector<float> out(std::size_t(B) * Hq * d, 0.0f), scores(L);
  const int gs = Hq / Hkv;
  for (int b = 0; b < B; ++b)
    for (int h = 0; h < Hq; ++h) {
      const float* qh = q.data() + (std::size_t(b) * Hq + h) * d;
      const float* kh = k.data() + (std::size_t(b) * Hkv + h / gs) * L * d;
      const float* vh = v.data() + (std::size_t(b) * Hkv + h / gs) * L * d;
      float mx = -std::numeric_limits<float>::infinity();
      for (std::size_t j = 0; j < L; ++j) {
        float s = 0.0f;
        for (int e = 0; e < d; ++e) s += qh[e] * kh[j * d + e];
        scores[j] = scale * s;
        mx = std::max(mx, scores[j]);
      }
      float den = 0.0f;
      for (std::size_t j = 0; j < L; ++j) {
        scores[j] = std::exp(scores[j] - mx);
        den += scores[j];
      }
      float* oh = out.data() + (std::size_t(b) * Hq + h) * d;
      for (std::size_t j = 0; j < L; ++j) {
        const float w = scores[j] / den;
        for (int e = 0; e < d; ++e) oh[e] += w * vh[j * d + e];
      }
    }
  return out;
}

double max_head_relative_error(const std::vector<float>& a, const std::vector<float>& b, std::size_t heads,
                               int d) {
  double worst = 0.0;
  for (std::size_t h = 0; h < heads; ++h) {
    double scale = 0.0, diff = 0.0;
    for (int e = 0; e < d; ++e) {
      const std::size_t i = h * d + e;
      scale = std::max(scale, double(std::max(std::fabs(a[i]), std::fabs(b[i]))));
      diff = std::max(diff, std::fabs(double(a[i]) - b[i]));
    }
    worst = std::max(worst, diff / std::max(scale, 1e-30));
  }
  return worst;
}

float round_bf16(float f) { return tf::b200::from_bf16(tf::b200::to_bf16(f)); }

// ---- one cell on the GPU ----------------------------------------------------
struct IterStats {
  double makespan_ms = 0, launch_tax_ms = 0, bulk_sync_ms = 0, wait_idle_ms = 0;
  std::uint64_t staged_bytes = 0;
};

struct LastTaxes {  // the TaxReport fields bench.cpp's JSON shows (taxmeter.hpp:144-157)
  std::vector<std::uint64_t> launch_count;
  std::uint64_t total_launches = 0;
  double launch_tax_ms = 0, bulk_sync_ms = 0, wait_idle_ms = 0, makespan_ms = 0;
  std::uint64_t staged_bytes = 0;
};

struct CellResult {
  std::string pattern;
  std::size_t value = 0;
  std::vector<IterStats> iters;
  LastTaxes last;
  std::optional<bool> verified;
  double max_err = 0.0;
  std::string error;
  double median_ms() const {
    std::vector<double> v;
    for (const auto& it : iters) v.push_back(it.makespan_ms);
    return percentile(v, 0.5);
  }
};

std::vector<int> device_list(const Options& o) {
  if (!o.devices.empty()) {
    if (int(o.devices.size()) != o.world_size)
      throw tf::ConfigError("--devices lists " + std::to_string(o.devices.size()) + " GPUs for world_size " +
                            std::to_string(o.world_size));
    return o.devices;
  }
  const int n = tf_device_count();
  const char* lb = std::getenv("TILEFABRIC_LOOPBACK");
  std::vector<int> d(std::size_t(o.world_size), 0);
  if (n >= o.world_size && !(lb && std::string(lb) == "1"))
    for (int r = 0; r < o.world_size; ++r) d[r] = r;
  return d;
}

struct GpuCell {
  const Options& o;
  tf::WorldConfig cfg;
  tf::b200::World* w = nullptr;
  std::vector<void*> a, bm, c, q, kk, vv, out;
  tf_ag_shape ag{};
  tf_fd_shape fd{};
  std::vector<float> host_a, host_b, host_q, host_k, host_v;  // for --verify
  std::size_t value = 0;

  GpuCell(const Options& opt, const tf::WorldConfig& c0) : o(opt), cfg(c0) {}
  ~GpuCell() { delete w; }

  std::size_t esz() const { return o.bf16() ? 2 : 4; }
  std::vector<uint8_t> pack(const float* src, std::size_t n) const {
    std::vector<uint8_t> outb(n * esz());
    if (o.bf16())
      for (std::size_t i = 0; i < n; ++i) reinterpret_cast<uint16_t*>(outb.data())[i] = tf::b200::to_bf16(src[i]);
    else
      std::memcpy(outb.data(), src, n * 4);
    return outb;
  }

  void setup(std::size_t val) {
    value = val;
    const int W = o.world_size;
    const auto devs = device_list(o);
    if (!o.fd_family) {
      const auto p = tf::ag::make_problem(o.seed, val, o.n, o.k, o.tiles);  // A then B (ag_gemm.hpp:71-83)
      const std::size_t kw = p.k / W;
      const std::size_t heap = esz() * (p.m * kw + 5 * p.m * p.k) + (64u << 20);
      w = new tf::b200::World(W, devs, heap, 0.0);
      w->apply(cfg);
      a = w->heap("ag.a", esz() * p.m * kw);
      const auto hb = pack(p.b.data(), p.b.size());
      for (int r = 0; r < W; ++r) {
        std::vector<float> shard(p.m * kw);  // fill_shard (ag_gemm.hpp:103-112)
        for (std::size_t i = 0; i < p.m; ++i)
          std::memcpy(&shard[i * kw], &p.a[i * p.k + r * kw], kw * 4);
        const auto hs = pack(shard.data(), shard.size());
        w->put(a[r], hs.data(), hs.size());
        bm.push_back(w->device(r, hb.size()));
        w->put(bm[r], hb.data(), hb.size());
        c.push_back(w->device(r, esz() * p.m * p.n));
      }
      ag = tf_ag_shape{p.m, p.n, p.k, o.tiles.bm, o.tiles.bn, o.tiles.bk, o.bf16() ? TF_BF16 : TF_F32};
      if (o.verify) {
        host_a = p.a;
        host_b = p.b;
      }
    } else {
      const int B = o.batch, Hq = o.heads, Hkv = o.kv_heads ? o.kv_heads : o.heads, d = o.head_dim;
      const std::size_t L = val, ln = L / W;
      // q, then K, then V from one stream (flash_decode.hpp:90-106).
      const std::size_t nq = std::size_t(B) * Hq * d, nkv = std::size_t(B) * Hkv * L * d;
      const auto all = tf::uniform_reals(o.seed, nq + 2 * nkv);
      std::vector<float> hq(all.begin(), all.begin() + nq), hk(all.begin() + nq, all.begin() + nq + nkv),
          hv(all.begin() + nq + nkv, all.end());
      const std::size_t row = std::size_t(B) * Hq * (d + 2);
      const std::size_t heap = 4 * W * row * 6 + 4 * std::size_t(B) * Hkv * 4096 * (d + 2) * 8 + (64u << 20);
      w = new tf::b200::World(W, devs, heap, 0.0);
      w->apply(cfg);
      const auto pq = pack(hq.data(), hq.size());
      for (int r = 0; r < W; ++r) {
        // slice_shard (flash_decode.hpp:140-160): positions [r*ln, (r+1)*ln).
        std::vector<float> sk(std::size_t(B) * Hkv * ln * d), sv(sk.size());
        for (std::size_t bh = 0; bh < std::size_t(B) * Hkv; ++bh) {
          std::memcpy(&sk[bh * ln * d], &hk[(bh * L + r * ln) * d], ln * d * 4);
          std::memcpy(&sv[bh * ln * d], &hv[(bh * L + r * ln) * d], ln * d * 4);
        }
        const auto pk = pack(sk.data(), sk.size()), pv = pack(sv.data(), sv.size());
        q.push_back(w->device(r, pq.size()));
        kk.push_back(w->device(r, pk.size()));
        vv.push_back(w->device(r, pv.size()));
        out.push_back(w->device(r, 4 * nq));  // fp32 output rows, as the reference returns
        w->put(q[r], pq.data(), pq.size());
        w->put(kk[r], pk.data(), pk.size());
        w->put(vv[r], pv.data(), pv.size());
      }
      fd = tf_fd_shape{B, Hq, Hkv, d, L, 1.0f / std::sqrt(float(d)), o.bf16() ? TF_BF16 : TF_F32, TF_F32};
      if (o.verify) {
        host_q = std::move(hq);
        host_k = std::move(hk);
        host_v = std::move(hv);
      }
    }
  }

  void launch(const std::string& pattern) {
    if (!o.fd_family)
      tf::b200::check(tf_ag_gemm_async(w->w, ag_variant(pattern), &ag, a.data(),
                                       const_cast<const void* const*>(bm.data()), c.data(), nullptr, nullptr));
    else
      tf::b200::check(tf_flash_decode_async(w->w, fd_variant(pattern, o.fd_arrival_order), &fd,
                                            const_cast<const void* const*>(q.data()),
                                            const_cast<const void* const*>(kk.data()),
                                            const_cast<const void* const*>(vv.data()), out.data(), nullptr,
                                            nullptr));
  }

  IterStats timed(const std::string& pattern, LastTaxes* last) {
    tf::b200::check(tf_tax_reset(w->w));
    const auto t0 = std::chrono::steady_clock::now();
    launch(pattern);
    tf::b200::check(tf_world_sync(w->w));
    const auto t1 = std::chrono::steady_clock::now();
    IterStats st;
    st.makespan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    const auto taxes = w->taxes();
    LastTaxes lt;
    for (const auto& t : taxes) {
      lt.bulk_sync_ms += double(t.bulk_sync_ns) / 1e6;
      lt.wait_idle_ms += double(t.wait_idle_ns) / 1e6;
      lt.staged_bytes += t.staged_bytes;
    }
    // tf_tax_report's launch count is the process' total since the reset:
    // shared by the ranks of a loopback device, so spread it evenly.
    const std::uint64_t total = taxes.empty() ? 0 : taxes[0].launches;
    lt.total_launches = total;
    for (std::size_t r = 0; r < taxes.size(); ++r)
      lt.launch_count.push_back(total / taxes.size() + (r < total % taxes.size() ? 1 : 0));
    lt.launch_tax_ms = double(total) * o.launch_cost_us / 1e3;
    lt.makespan_ms = st.makespan_ms;
    st.launch_tax_ms = lt.launch_tax_ms;
    st.bulk_sync_ms = lt.bulk_sync_ms;
    st.wait_idle_ms = lt.wait_idle_ms;
    st.staged_bytes = lt.staged_bytes;
    if (last) *last = lt;
    return st;
  }

  // One run, every rank's output against the brute-force checker.
  double verify(const std::string& pattern) {
    launch(pattern);
    tf::b200::check(tf_world_sync(w->w));
    const int W = o.world_size;
    double err = 0.0;
    auto unpack = [&](const void* dev, std::size_t n, bool bf) {
      std::vector<uint8_t> raw(n * (bf ? 2 : 4));
      w->put(raw.data(), dev, raw.size());
      std::vector<float> f(n);
      for (std::size_t i = 0; i < n; ++i)
        f[i] = bf ? tf::b200::from_bf16(reinterpret_cast<uint16_t*>(raw.data())[i])
                  : reinterpret_cast<float*>(raw.data())[i];
      return f;
    };
    if (!o.fd_family) {
      auto A = host_a, Bm = host_b;
      if (o.bf16()) {
        for (auto& x : A) x = round_bf16(x);
        for (auto& x : Bm) x = round_bf16(x);
      }
      const auto want = check_gemm(A, Bm, ag.m, ag.n, ag.k);
      double scale = 0.0;
      for (float x : want) scale = std::max(scale, double(std::fabs(x)));
      for (int r = 0; r < W; ++r) {
        const auto got = unpack(c[r], ag.m * ag.n, o.bf16());
        for (std::size_t i = 0; i < got.size(); ++i) {
          const double e = std::fabs(double(got[i]) - want[i]);
          err = std::max(err, o.bf16() ? e / std::max(scale, 1e-30) : e);
        }
      }
    } else {
      auto Q = host_q, K = host_k, V = host_v;
      if (o.bf16()) {
        for (auto* vec : {&Q, &K, &V})
          for (auto& x : *vec) x = round_bf16(x);
      }
      const auto want = check_attention(Q, K, V, fd.batch, fd.q_heads, fd.kv_heads, fd.head_dim, fd.kv_len,
                                        fd.scale);
      for (int r = 0; r < W; ++r) {
        const auto got = unpack(out[r], want.size(), false);
        err = std::max(err, max_head_relative_error(got, want, std::size_t(fd.batch) * fd.q_heads, fd.head_dim));
      }
    }
    return err;
  }
};

double verify_tol(const Options& o) {
  // bench.cpp:62-64: bitwise for the GEMM, 1e-5 head-relative for decode;
  // the bf16 path against bf16-rounded inputs: bf16 GEMM
  // output, fp32 decode output (hi/lo P on the tensor cores).
  if (o.bf16()) return o.fd_family ? 1e-4 : 4e-3;
  return o.fd_family ? 1e-5 : 0.0;
}

CellResult run_cell(const Options& o, const tf::WorldConfig& cfg, const std::string& pattern,
                    std::size_t value) {
  CellResult cell;
  cell.pattern = pattern;
  cell.value = value;
  GpuCell g(o, cfg);
  g.setup(value);
  if (o.verify) {
    cell.max_err = g.verify(pattern);
    const double tol = verify_tol(o);
    cell.verified = cell.max_err <= tol;
    if (!*cell.verified) {
      std::ostringstream msg;
      msg << "verify mismatch: max error " << cell.max_err << " exceeds " << tol;
      cell.error = msg.str();
      return cell;
    }
  }
  for (int i = 0; i < o.warmup; ++i) {
    g.launch(pattern);
    tf::b200::check(tf_world_sync(g.w->w));
  }
  for (int i = 0; i < o.iters; ++i) cell.iters.push_back(g.timed(pattern, &cell.last));
  return cell;
}

// ---- output writers (bench.cpp:272-418) ---------------------------------------
const char* kIterHeader =
    "pattern,world_size,m,n,k,heads,head_dim,kv_len,seed,iter,makespan_ms,"
    "launch_tax_ms,bulk_sync_tax_ms,wait_idle_ms,staged_bytes,verified";
const char* kSweepHeader =
    "pattern,world_size,m,n,k,heads,head_dim,kv_len,seed,iters,median_ms,"
    "p10_ms,p90_ms,launch_tax_ms,bulk_sync_tax_ms,wait_idle_ms,staged_bytes,"
    "verified,speedup_vs_baseline,error";

std::string shape_columns(const Options& o, std::size_t value) {
  std::ostringstream row;
  if (o.fd_family) row << ",,," << o.heads << "," << o.head_dim << "," << value;
  else row << value << "," << o.n << "," << o.k << ",,,";
  return row.str();
}

std::string verified_column(const std::optional<bool>& v) {
  if (!v.has_value()) return "";
  return *v ? "true" : "false";
}

void write_iteration_csv(std::ostream& os, const Options& o, const CellResult& cell) {
  os << kIterHeader << "\n";
  for (std::size_t i = 0; i < cell.iters.size(); ++i) {
    const auto& it = cell.iters[i];
    os << cell.pattern << "," << o.world_size << "," << shape_columns(o, cell.value) << "," << o.seed << ","
       << i << "," << it.makespan_ms << "," << it.launch_tax_ms << "," << it.bulk_sync_ms << ","
       << it.wait_idle_ms << "," << it.staged_bytes << "," << verified_column(cell.verified) << "\n";
  }
}

std::string summary_json(const Options& o, const CellResult& cell) {
  std::vector<double> ms, bulk, idle;
  for (const auto& it : cell.iters) {
    ms.push_back(it.makespan_ms);
    bulk.push_back(it.bulk_sync_ms);
    idle.push_back(it.wait_idle_ms);
  }
  std::ostringstream j;
  j << "{\n  \"pattern\": " << json_str(cell.pattern) << ",\n  \"world_size\": " << o.world_size << ",\n";
  if (o.fd_family) {
    j << "  \"heads\": " << o.heads << ",\n  \"head_dim\": " << o.head_dim << ",\n  \"kv_len\": " << cell.value
      << ",\n  \"batch\": " << o.batch << ",\n  \"kv_heads\": " << (o.kv_heads ? o.kv_heads : o.heads) << ",\n";
  } else {
    j << "  \"m\": " << cell.value << ",\n  \"n\": " << o.n << ",\n  \"k\": " << o.k << ",\n  \"tiles\": ["
      << o.tiles.bm << ", " << o.tiles.bn << ", " << o.tiles.bk << "],\n";
  }
  j << "  \"dtype\": " << json_str(o.dtype) << ",\n  \"seed\": " << o.seed << ",\n  \"iters\": " << o.iters
    << ",\n  \"warmup\": " << o.warmup << ",\n  \"launch_cost_us\": " << num(o.launch_cost_us)
    << ",\n  \"latency_ms\": {\"median\": " << num(percentile(ms, 0.5)) << ", \"p10\": "
    << num(percentile(ms, 0.1)) << ", \"p90\": " << num(percentile(ms, 0.9)) << "},\n";
  const auto& t = cell.last;
  j << "  \"taxes\": {\"world_size\": " << o.world_size << ", \"launch_cost_us\": " << num(o.launch_cost_us)
    << ", \"launch_count\": [";
  for (std::size_t r = 0; r < t.launch_count.size(); ++r) j << (r ? ", " : "") << t.launch_count[r];
  j << "], \"total_launches\": " << t.total_launches << ", \"launch_tax_ms\": " << num(t.launch_tax_ms)
    << ", \"bulk_sync_tax_ms\": " << num(t.bulk_sync_ms) << ", \"wait_idle_ms\": " << num(t.wait_idle_ms)
    << ", \"staged_bytes\": " << t.staged_bytes << ", \"makespan_ms\": " << num(t.makespan_ms)
    << ", \"bulk_sync_tax_ms_median\": " << num(percentile(bulk, 0.5))
    << ", \"wait_idle_ms_median\": " << num(percentile(idle, 0.5)) << "}";
  if (cell.verified.has_value())
    j << ",\n  \"verified\": " << (*cell.verified ? "true" : "false") << ",\n  \"max_error\": " << num(cell.max_err);
  j << "\n}";
  return j.str();
}

void write_sweep_row(std::ostream& os, const Options& o, const CellResult& cell, const std::string& speedup) {
  std::vector<double> ms, bulk, idle, launch;
  double staged = 0.0;
  for (const auto& it : cell.iters) {
    ms.push_back(it.makespan_ms);
    bulk.push_back(it.bulk_sync_ms);
    idle.push_back(it.wait_idle_ms);
    launch.push_back(it.launch_tax_ms);
    staged = double(it.staged_bytes);
  }
  os << cell.pattern << "," << o.world_size << "," << shape_columns(o, cell.value) << "," << o.seed << ","
     << cell.iters.size() << "," << percentile(ms, 0.5) << "," << percentile(ms, 0.1) << ","
     << percentile(ms, 0.9) << "," << percentile(launch, 0.5) << "," << percentile(bulk, 0.5) << ","
     << percentile(idle, 0.5) << "," << staged << "," << verified_column(cell.verified) << "," << speedup
     << "," << csv_escape(cell.error) << "\n";
}

void write_gnuplot_dat(std::ostream& os, const Options& o, const std::vector<CellResult>& cells) {
  const std::string baseline = o.fd_family ? kFdBaseline : kAgBaseline;
  os << "# median-makespan speedup vs " << baseline << " (ratio > 1: pattern is faster)\n";
  os << "# " << (o.fd_family ? "kv_len" : "m");
  for (const auto& p : o.patterns) os << " " << p;
  os << "\n";
  for (const std::size_t value : o.values) {
    double base_ms = 0.0;
    for (const auto& c : cells)
      if (c.value == value && c.pattern == baseline && c.error.empty()) base_ms = c.median_ms();
    os << value;
    for (const auto& p : o.patterns) {
      double ms = 0.0;
      for (const auto& c : cells)
        if (c.value == value && c.pattern == p && c.error.empty()) ms = c.median_ms();
      if (base_ms > 0.0 && ms > 0.0) os << " " << base_ms / ms;
      else os << " nan";
    }
    os << "\n";
  }
}

void print_dry_run(const Options& o) {
  std::string pats;
  for (const auto& p : o.patterns) pats += (pats.empty() ? "" : " ") + p;
  std::cout << "preset: " << (o.preset.empty() ? "(none)" : o.preset) << "\n"
            << "patterns: " << pats << "\n"
            << "world_size: " << o.world_size << "\n";
  if (o.fd_family) {
    std::cout << "heads: " << o.heads << "\n"
              << "head_dim: " << o.head_dim << "\n"
              << "kv_len:";
    for (const auto v : o.values) std::cout << " " << v;
    std::cout << "\nfold_by_arrival: " << (o.fd_arrival_order ? "true" : "false") << "\n"
              << "batch: " << o.batch << "\n"
              << "kv_heads: " << (o.kv_heads ? o.kv_heads : o.heads) << "\n";
  } else {
    std::cout << "m:";
    for (const auto v : o.values) std::cout << " " << v;
    std::cout << "\nn: " << o.n << "\n"
              << "k: " << o.k << "\n"
              << "tiles: " << o.tiles.bm << "x" << o.tiles.bn << "x" << o.tiles.bk << "\n";
  }
  std::cout << "dtype: " << o.dtype << "\n"
            << "launch_cost_us: " << o.launch_cost_us << "\n"
            << "iters: " << o.iters << "\n"
            << "warmup: " << o.warmup << "\n"
            << "seed: " << o.seed << "\n"
            << "verify: " << (o.verify ? "true" : "false") << "\n"
            << "skew:";
  if (o.skew_specs.empty()) std::cout << " (none)";
  for (const auto& s : o.skew_specs) std::cout << " " << s;
  std::cout << "\nout: " << (o.out.empty() ? "(stdout only)" : o.out) << std::endl;
}

std::ofstream open_or_throw(const std::string& path) {
  std::ofstream os(path);
  if (!os) throw tf::ConfigError("cannot open output file \"" + path + "\"");
  return os;
}

int run(Options o) {  // bench.cpp:476-693
  if (!o.preset.empty()) {
    const Preset* pre = nullptr;
    for (const auto& p : presets())
      if (p.name == o.preset) pre = &p;
    if (!pre) {
      std::string names;
      for (const auto& p : presets()) names += (names.empty() ? "" : ", ") + p.name;
      throw tf::ConfigError("unknown preset \"" + o.preset + "\" (available: " + names + ")");
    }
    if (!o.has("--pattern") && !o.has("--patterns")) o.patterns = pre->patterns;
    if (!o.has("--world-size")) o.world_size = pre->world_size;
    if (pre->family == "fd") {
      if (!o.has("--heads")) o.heads = pre->heads;
      if (!o.has("--head-dim")) o.head_dim = pre->head_dim;
      if (!o.has("--kv-len") && !o.has("--sweep-kv")) o.sweep_kv = pre->kv_sweep;
    } else {
      if (!o.has("--n")) o.n = pre->n;
      if (!o.has("--k")) o.k = pre->k;
      if (!o.has("--m") && !o.has("--sweep-m")) o.sweep_m = pre->m_sweep;
    }
  }
  if (o.patterns.empty()) throw tf::ConfigError("no pattern selected; pass --pattern, --patterns, or --preset");
  bool any_ag = false, any_fd = false;
  for (const auto& p : o.patterns) {
    if (contains(kAgPatterns, p)) {
      any_ag = true;
    } else if (contains(kFdPatterns, p)) {
      any_fd = true;
    } else {
      std::string names;
      for (const auto& n : kAgPatterns) names += (names.empty() ? "" : ", ") + n;
      for (const auto& n : kFdPatterns) names += ", " + n;
      throw tf::ConfigError("unknown pattern \"" + p + "\" (available: " + names + ")");
    }
  }
  if (any_ag && any_fd) throw tf::ConfigError("cannot mix ag-* and fd-* patterns in one run");
  o.fd_family = any_fd;
  if (o.iters < 1) throw tf::ConfigError("--iters must be >= 1");
  if (o.warmup < 0) throw tf::ConfigError("--warmup must be >= 0");
  if (!o.sweep_m.empty() && o.fd_family) throw tf::ConfigError("--sweep-m applies to ag-* patterns only");
  if (!o.sweep_kv.empty() && !o.fd_family) throw tf::ConfigError("--sweep-kv applies to fd-* patterns only");
  if (o.dtype != "f32" && o.dtype != "bf16") throw tf::ConfigError("--dtype must be f32 or bf16");
  if (o.batch < 1) throw tf::ConfigError("--batch must be >= 1");
  if (o.fd_arrival_order && o.fd_family)
    for (const auto& p : o.patterns)
      if (p != "fd-fused") throw tf::ConfigError("--fd-arrival-order applies to fd-fused only");
  o.values = o.fd_family ? (o.sweep_kv.empty() ? std::vector<std::size_t>{o.kv_len} : o.sweep_kv)
                         : (o.sweep_m.empty() ? std::vector<std::size_t>{o.m} : o.sweep_m);
  const bool sweep_mode = o.values.size() > 1 || o.patterns.size() > 1;
  if (o.dry_run) {
    print_dry_run(o);
    return 0;
  }

  tf::WorldConfig cfg;
  cfg.world_size = o.world_size;
  cfg.seed = o.seed;
  cfg.launch_cost = std::chrono::duration_cast<tf::Duration>(std::chrono::duration<double, std::micro>(o.launch_cost_us));
  for (const auto& spec : o.skew_specs) {
    const auto [rank, delay] = parse_skew(spec);
    tf::inject_skew(cfg, rank, delay);
  }
  cfg.validate();
  o.tiles.validate();
  // Divisibility is a flag error, not a cell error (bench.cpp:598-617).
  for (const std::size_t value : o.values) {
    if (o.fd_family) {
      tf::fd::DecodeProblem p;
      p.heads = o.heads;
      p.head_dim = o.head_dim;
      p.kv_len = value;
      p.scale = 1.0f;
      p.kv_heads = o.kv_heads;
      p.validate(o.world_size);
      if (o.kv_heads && (o.kv_heads < 1 || o.heads % o.kv_heads))
        throw tf::ConfigError("--heads must be a multiple of --kv-heads");
    } else {
      tf::ag::AgGemmProblem p;
      p.m = value;
      p.n = o.n;
      p.k = o.k;
      p.validate(o.world_size);
    }
  }

  if (!sweep_mode) {
    const CellResult cell = run_cell(o, cfg, o.patterns.front(), o.values.front());
    if (cell.verified.has_value() && !*cell.verified) {
      std::cerr << "verification FAILED for " << cell.pattern << ": " << cell.error << std::endl;
      return 1;
    }
    const auto j = summary_json(o, cell);
    std::cout << j << std::endl;
    if (!o.out.empty()) {
      auto csv = open_or_throw(o.out + ".csv");
      write_iteration_csv(csv, o, cell);
      auto js = open_or_throw(o.out + ".json");
      js << j << "\n";
    }
    return 0;
  }

  std::vector<CellResult> cells;
  for (const std::size_t value : o.values)
    for (const auto& pattern : o.patterns) {
      try {
        cells.push_back(run_cell(o, cfg, pattern, value));
      } catch (const std::exception& e) {  // a failed cell becomes a row; the sweep goes on
        CellResult cell;
        cell.pattern = pattern;
        cell.value = value;
        cell.error = e.what();
        cells.push_back(std::move(cell));
      }
    }
  std::ostringstream body;
  body << kSweepHeader << "\n";
  const std::string baseline = o.fd_family ? kFdBaseline : kAgBaseline;
  for (const auto& cell : cells) {
    std::string speedup;
    if (cell.error.empty())
      for (const auto& base : cells)
        if (base.value == cell.value && base.pattern == baseline && base.error.empty() && !base.iters.empty()) {
          std::ostringstream s;
          s << base.median_ms() / cell.median_ms();
          speedup = s.str();
        }
    write_sweep_row(body, o, cell, speedup);
  }
  std::cout << body.str();
  if (!o.out.empty()) {
    auto csv = open_or_throw(o.out + ".csv");
    csv << body.str();
    auto dat = open_or_throw(o.out + ".dat");
    write_gnuplot_dat(dat, o, cells);
  }
  for (const auto& cell : cells)
    if (!cell.error.empty() || (cell.verified.has_value() && !*cell.verified)) {
      std::cerr << "cell failed: " << cell.pattern << " @ " << cell.value << ": " << cell.error << std::endl;
      return 1;
    }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Options o;
  try {
    o = parse_args(argc, argv);
  } catch (const HelpRequested&) {
    std::cout << kUsage;
    return 0;
  } catch (const ParseError& e) {
    std::cerr << e.what() << "\nRun with --help for usage." << std::endl;
    return 2;
  }
  try {
    return run(std::move(o));
  } catch (const tf::ConfigError& e) {
    std::cerr << "error: " << e.what() << "\nRun with --help for usage." << std::endl;
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << std::endl;
    return 1;
  }
}
