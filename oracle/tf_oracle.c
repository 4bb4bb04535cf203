/*
 * tf_oracle.c -- CPU restatement of the reference ("tilefabric") arithmetic
 * for the two hot paths.  TEST INFRASTRUCTURE ONLY: imported by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the checker.
 * The product path (paper_2511_02168_b200/) never links or calls this.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function here
 * against (a) the golden values the reference's own code produced
 * (tests/golden/ fixtures) and (b) oracle/_ref, the
 * reference headers compiled as-is (oracle/Makefile).
 *
 * Build with -ffp-contract=off (as the reference does,
 * proj/CMakeLists.txt:12-16): the reference's GEMM/attention rely on
 * separate rounding of every multiply and add.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

/* ---- std::mt19937_64 (the engine behind uniform_reals,
 *      proj/include/tilefabric/common.hpp:132-140) ---------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} tfo_mt64;

static void mt64_seed(tfo_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) +
               (uint64_t)i;
  }
  s->idx = 312;
}

static uint64_t mt64_next(tfo_mt64* s) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  static const uint64_t MAG[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  if (s->idx >= 312) {
    int i = 0;
    for (; i < 312 - 156; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ MAG[x & 1ULL];
    }
    for (; i < 311; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ MAG[x & 1ULL];
    }
    uint64_t x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ MAG[x & 1ULL];
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* uniform_real_distribution<float>(-1, 1) over mt19937_64, as libstdc++
 * evaluates it: generate_canonical<float, 24> draws ONE 64-bit word
 * (24 bits needed <= 64 produced), converts it to float (round to
 * nearest), divides by 2^64 (exact power of two), clamps a result of 1.0
 * to nextafter(1, 0); the distribution then returns canon * (b - a) + a
 * in float.  common.hpp:132-140 is the call site. */
void tfo_uniform_reals(uint64_t seed, size_t n, float* out) {
  tfo_mt64 s;
  mt64_seed(&s, seed);
  const float two64 = 18446744073709551616.0f;
  for (size_t i = 0; i < n; ++i) {
    float c = (float)mt64_next(&s) / two64;
    if (c >= 1.0f) c = nextafterf(1.0f, 0.0f);
    float prod = c * 2.0f; /* (b - a) == 2.0f; no contraction */
    out[i] = prod + -1.0f;
  }
}

/* reference::gemm, proj/include/tilefabric/reference.hpp:36-49:
 * fp32, ascending k, one rounding per multiply and per add. */
void tfo_gemm(const float* a, const float* b, size_t m, size_t n, size_t k,
              float* c) {
  for (size_t i = 0; i < m; ++i) {
    for (size_t j = 0; j < n; ++j) {
      float acc = 0.0f;
      for (size_t p = 0; p < k; ++p) {
        float prod = a[i * k + p] * b[p * n + j];
        acc = acc + prod;
      }
      c[i * n + j] = acc;
    }
  }
}

/* Same chain over a row slice [row0, row0+rows): lets tests check sampled
 * rows of a full-size problem (SURVEY.md §8(c) parity item 3). */
void tfo_gemm_rows(const float* a, const float* b, size_t row0, size_t rows,
                   size_t n, size_t k, float* c) {
  tfo_gemm(a + row0 * k, b, rows, n, k, c);
}

/* reference::attention, reference.hpp:63-99: monolithic two-pass softmax.
 * q: heads x d; k, v: heads x L x d; out: heads x d. */
void tfo_attention(const float* q, const float* k, const float* v,
                   size_t heads, size_t d, size_t L, float scale, float* out,
                   float* scratch /* L floats */) {
  for (size_t h = 0; h < heads; ++h) {
    const float* qh = q + h * d;
    const float* kh = k + h * L * d;
    const float* vh = v + h * L * d;
    float mx = -INFINITY;
    for (size_t j = 0; j < L; ++j) {
      float s = 0.0f;
      for (size_t e = 0; e < d; ++e) {
        float prod = qh[e] * kh[j * d + e];
        s = s + prod;
      }
      scratch[j] = scale * s;
      mx = fmaxf(mx, scratch[j]);
    }
    float denom = 0.0f;
    for (size_t j = 0; j < L; ++j) {
      scratch[j] = expf(scratch[j] - mx);
      denom += scratch[j];
    }
    float* oh = out + h * d;
    for (size_t e = 0; e < d; ++e) oh[e] = 0.0f;
    for (size_t j = 0; j < L; ++j) {
      const float w = scratch[j] / denom;
      for (size_t e = 0; e < d; ++e) {
        float prod = w * vh[j * d + e];
        oh[e] = oh[e] + prod;
      }
    }
  }
}

/* attention_partial, proj/include/tilefabric/tilemath.hpp:145-181.
 * Writes wire rows [m | l | o[0..d)] per head (tilemath.hpp:244-258).
 * Returns 0, or 1 + (h * L + j) of the first non-finite score
 * (the NumericError case, tilemath.hpp:163-167). */
long long tfo_attention_partial_wire(const float* q, const float* k,
                                     const float* v, int heads, int d,
                                     size_t len, float scale, float* wire) {
  for (int h = 0; h < heads; ++h) {
    const float* qh = q + (size_t)h * d;
    const float* kh = k + (size_t)h * len * d;
    const float* vh = v + (size_t)h * len * d;
    float* row = wire + (size_t)h * (d + 2);
    float* oh = row + 2;
    float m = -INFINITY, l = 0.0f;
    for (int e = 0; e < d; ++e) oh[e] = 0.0f;
    for (size_t j = 0; j < len; ++j) {
      float s = 0.0f;
      for (int e = 0; e < d; ++e) {
        float prod = qh[e] * kh[j * d + e];
        s = s + prod;
      }
      s = s * scale;
      if (!isfinite(s)) return 1 + (long long)((size_t)h * len + j);
      const float mn = fmaxf(m, s);
      const float alpha = expf(m - mn);
      const float w = expf(s - mn);
      float la = l * alpha;
      l = la + w;
      for (int e = 0; e < d; ++e) {
        float oa = oh[e] * alpha;
        float wv = w * vh[j * d + e];
        oh[e] = oa + wv;
      }
      m = mn;
    }
    row[0] = m;
    row[1] = l;
  }
  return 0;
}

/* combine_partials, tilemath.hpp:186-220, on wire rows: acc <- acc (+) x. */
void tfo_combine_wire(float* acc, const float* x, int heads, int d) {
  for (int h = 0; h < heads; ++h) {
    float* a = acc + (size_t)h * (d + 2);
    const float* y = x + (size_t)h * (d + 2);
    if (a[1] == 0.0f) {
      memcpy(a, y, sizeof(float) * (size_t)(d + 2));
      continue;
    }
    if (y[1] == 0.0f) continue;
    const float m = fmaxf(a[0], y[0]);
    const float ax = expf(a[0] - m);
    const float ay = expf(y[0] - m);
    float l1 = a[1] * ax;
    float l2 = y[1] * ay;
    a[0] = m;
    a[1] = l1 + l2;
    for (int e = 0; e < d; ++e) {
      float o1 = a[2 + e] * ax;
      float o2 = y[2 + e] * ay;
      a[2 + e] = o1 + o2;
    }
  }
}

/* finalize, tilemath.hpp:225-239.  Returns 0, or 1 + head of the first
 * empty normalizer (EmptyAttentionError). */
int tfo_finalize_wire(const float* acc, int heads, int d, float* out) {
  for (int h = 0; h < heads; ++h) {
    const float* a = acc + (size_t)h * (d + 2);
    if (a[1] == 0.0f) return 1 + h;
    for (int e = 0; e < d; ++e) out[(size_t)h * d + e] = a[2 + e] / a[1];
  }
  return 0;
}

/* The neutral partial (tilemath.hpp:127-139) on the wire. */
void tfo_neutral_wire(float* acc, int heads, int d) {
  for (int h = 0; h < heads; ++h) {
    float* a = acc + (size_t)h * (d + 2);
    a[0] = -INFINITY;
    a[1] = 0.0f;
    for (int e = 0; e < d; ++e) a[2 + e] = 0.0f;
  }
}

/* fd::run_fused's math for one world (flash_decode.hpp:140-180, 348-423):
 * slice the KV sequence into W contiguous shards, one partial per shard,
 * ascending-source fold, finalize.  q: H x d; k, v: H x L x d.
 * wires: (W + 1) * H * (d+2) scratch (filled with each source's wire rows, i.e.
 * the inbox every rank ends up with).  Returns finalize's code. */
int tfo_fd_world(const float* q, const float* k, const float* v, int heads,
                 int d, size_t L, float scale, int world, float* wires,
                 float* shard_scratch /* 2 * H * (L/W) * d */, float* out) {
  const size_t len = L / (size_t)world;
  const size_t wire = (size_t)heads * (d + 2);
  float* ks = shard_scratch;
  float* vs = shard_scratch + (size_t)heads * len * d;
  for (int r = 0; r < world; ++r) {
    for (int h = 0; h < heads; ++h) {
      const size_t src = ((size_t)h * L + (size_t)r * len) * d;
      memcpy(ks + (size_t)h * len * d, k + src, sizeof(float) * len * d);
      memcpy(vs + (size_t)h * len * d, v + src, sizeof(float) * len * d);
    }
    long long bad = tfo_attention_partial_wire(q, ks, vs, heads, d, len, scale,
                                               wires + (size_t)r * wire);
    if (bad) return -1;
  }
  /* fold_rows (flash_decode.hpp:171-180): ascending source, then finalize;
   * the last wire slot-sized region past the W inbox rows is the fold acc. */
  float* acc = wires + (size_t)world * wire;
  tfo_neutral_wire(acc, heads, d);
  for (int s = 0; s < world; ++s) tfo_combine_wire(acc, wires + (size_t)s * wire, heads, d);
  return tfo_finalize_wire(acc, heads, d, out);
}

/* max_head_relative_error, reference.hpp:115-132. */
double tfo_max_head_relative_error(const float* a, const float* b, int heads,
                                   int d) {
  double worst = 0.0;
  for (int h = 0; h < heads; ++h) {
    double scale = 0.0, diff = 0.0;
    for (int e = 0; e < d; ++e) {
      const size_t i = (size_t)h * d + e;
      double aa = fabs((double)a[i]), bb = fabs((double)b[i]);
      double mx = aa > bb ? aa : bb;
      if (mx > scale) scale = mx;
      double df = fabs((double)a[i] - (double)b[i]);
      if (df > diff) diff = df;
    }
    double r = diff / (scale > 1e-30 ? scale : 1e-30);
    if (r > worst) worst = r;
  }
  return worst;
}

/* FNV-1a 64 over raw bytes (the hash SURVEY.md Appendix A quotes). */
uint64_t tfo_fnv1a64(const void* data, size_t bytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (size_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* bf16 round-to-nearest-even of an fp32 value, widened back to fp32: the
 * GPU path's inputs are RNE(uniform_reals) (BASELINE.md §2 "Inputs"). */
void tfo_round_bf16(const float* in, size_t n, float* out_f32,
                    uint16_t* out_bf16) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t u;
    memcpy(&u, &in[i], 4);
    uint32_t r;
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) {
      r = (u | 0x00400000u) & 0xffff0000u; /* quiet NaN */
    } else {
      r = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
    }
    if (out_bf16) out_bf16[i] = (uint16_t)(r >> 16);
    if (out_f32) memcpy(&out_f32[i], &r, 4);
  }
}
