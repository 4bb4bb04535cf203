// fd.cu -- multi-GPU Flash Decode (flash_decode.hpp), all four schedules.
//
// Work decomposition (every schedule shares it, so every schedule folds the
// same partial bits and outputs are bitwise identical across schedules and
// across ranks, as flash_decode.hpp:35-36 promises):
//   group  g = (b, kv_head): one KV stream [len][d] shared by gs = Hq/Hkv
//          q-heads (GQA; gs = 1 is the reference's MHA).
//   split  the rank's len = L/W positions are cut into S contiguous splits
//          (S from the shape only).  A CTA computes one (group, split)
//          attention partial for all gs heads (attention_partial,
//          tilemath.hpp:145-181) and the LAST split to finish (ticket)
//          folds the S split partials in ascending order into the rank's
//          partial for the group.
//   wire   the rank partial leaves as rows [m | l | o[d]] fp32
//          (tilemath.hpp:244-258), one per (b, q-head):
//          inbox[src][b][hq][d+2] (flash_decode.hpp:353-368).
//   fold   ascending source order, combine_partials (tilemath.hpp:186-220),
//          finalize (tilemath.hpp:225-239).
//
// Schedules:
//   bsp            attention(publish) | barrier | gather | barrier | fold
//   independent_ag attention(publish) | barrier | push+signal, wait-all |
//                  barrier | fold
//   fine_waits     attention(publish) | barrier | push+signal | fold with
//                  per-source waits
//   fused          ONE persistent launch: attention, split fold, push to
//                  every peer + red.release.sys flag per (src, group), then
//                  flag-gated ascending fold and finalize.  CTAs claim
//                  compute items dynamically and only wait once no compute
//                  item is left, so every push happens before any CTA
//                  blocks: deadlock-free without co-residency assumptions.
//
// Attention kernels:
//   fast     bf16 K/V, d = 128, gs = 8: register-only tensor-core decode.
//            S^T = K.Q^T with mma.m16n8k16 (16 keys x 8 heads, no padding),
//            P^T and V^T reach their MMA fragments through movmatrix
//            transposes of plain 16-byte row loads -- no shared memory in
//            the main loop, every KV byte read once with 128-bit
//            L1::no_allocate loads.
//   generic  any d <= 256, any gs <= 32, fp32 or bf16: one warp per q-head,
//            ascending keys, lanes split d.  Runs the reference's own test
//            shapes (d = 4, 8, 16; MHA).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "sm100.cuh"
#include "world.hpp"

namespace tfb {
namespace {

constexpr int kMaxLocal = 16;  // local ranks per launch (loopback worlds)
constexpr int kFoldRB = 16;    // rows per warp per load batch in the split folds
constexpr int kTraceSlots = 32;  // TFB_TRACE: %globaltimer stamps per CTA
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct FdRank {
  const void* q;
  const void* k;
  const void* v;
  void* out;
  float* pub;        // [B][Hq][d+2]: this rank's published partial (bsp/ag)
  float* inbox;      // [W][B][Hq][d+2] local inbox (fold source)
  uint64_t* flags;   // [W][G] local flag board
  int rank;          // global rank id
  uint64_t skew_ns;  // straggler delay before this rank's compute (fabric.hpp:59-62)
  const int* pages;  // paged KV: block table [B][pps] into this rank's pool (else null)
};

struct FdParams {
  int nlocal;
  int W, B, Hq, Hkv, gs, d;
  size_t len;        // positions per rank
  int S;             // splits per group
  size_t split_len;  // positions per split (last split may be shorter)
  float scale;
  int kv_bf16, out_bf16;
  uint64_t epoch;       // ticket epoch (per ticket buffer)
  uint64_t flag_epoch;  // flag-board epoch (per board geometry)
  uint64_t watchdog_ns;
  DevErr* err;
  int board;
  float* ws;                  // [nlocal][G][S][gs][d+4] split partials [m l - - o[d]]
  uint64_t* done;             // [nlocal][G] finished splits this launch (reset by the last CTA)
  uint64_t* gtick;            // [nlocal][G] split-folded sub-items this launch (reset by the last CTA)
  unsigned long long* claim;  // [nlocal][G] epoch-valued cross-rank fold claims
  unsigned int* ctr;          // [0] compute, [1] fold, [2] done
  unsigned int* sfc;          // [nlocal] split-fold sub-item counters
  int hc;                     // heads per split-fold sub-item
  int fold_once;              // every CTA's first split-fold claim covers all sub-items:
                              // a CTA folds at most one and skips the re-claim
  int interleave;             // fast split: the CTA's warps interleave 16-key tiles
  uint64_t local_dst;         // bit dst: dst's inbox/flags live on this launch's device
  int push;                   // push rank partials to every inbox (+ signal)
  int fold_inline;            // fused: fold after compute
  int direct;                 // fused, W = 1: the final split fold also finalizes out
  int by_arrival;             // fused: FdOptions::fold_by_arrival
  int owner;                  // fused, owner-combine: group g is folded by rank g % W only
  uint64_t oflag_epoch;       // owner-combine: epoch of the final-row flag board
  float* outbox_all[64];      // owner-combine: every rank's [B][Hq][d] fp32 final rows (this parity)
  unsigned long long* events_all[64];  // event log (tf_world_set_events): [W src][G] x {store, first load}
  uint64_t* oflags_all[64];   // owner-combine: every rank's [G] final-row flags
  unsigned long long* trace;  // TFB_TRACE: [grid][16] %globaltimer stamps per CTA (else null)
  float* inbox_all[64];       // every rank's inbox (this parity), this process' view
  uint64_t* flags_all[64];    // every rank's flag board
  // TMA-fed split kernel (fd_stream_kernel): host-built item table of ONE
  // rank, entry = {g, split j, first key, end key} (item i of the launch is
  // table entry i / nlocal of local rank i % nlocal); per group split count;
  // per (lr, g) fold claim state (0 free, 1 folded inline by the last
  // split's CTA, 2 taken by the fold phase; reset by the last CTA).
  // Device-resident epochs (fused schedules): when set, a launch reads its
  // flag / claim epochs from these cells (+1) and its last CTA stores them
  // back, so the launch is self-contained and a captured CUDA graph replays
  // with fresh epochs.  [0] fused flag board, [1] owner flag board, [2]
  // owner final-row flags, [3] fold claims.  inbox_all / outbox_all are then
  // the parity-0 halves; the launch adds epoch parity x *_pstride.
  uint64_t* depoch;
  size_t inbox_pstride, outbox_pstride;
  const uint4* items;
  unsigned nitems;
  const int* gS;
  unsigned* fstate;
  // Paged KV (tf_flash_decode_paged): k / v of each rank are page pools,
  // NHD [num_pages][1 << page_shift][Hkv][d] or (hnd) HND
  // [num_pages][Hkv][1 << page_shift][d]; key x of batch b sits in row
  // x & (page - 1) of page pages[b * pps + (x >> page_shift)].
  int paged, page_shift, pps, num_pages, hnd;
  FdRank r[kMaxLocal];
};

// Paged KV: the pool row (in units of d elements) of key x of batch b, KV
// head kvh.  An entry outside the pool raises TF_ERR_SHAPE (kPage) and reads
// page 0, so a bad table never faults the device.
__device__ __forceinline__ size_t paged_row_of(const FdParams& P, int pg, size_t x, int kvh, int b, int rank) {
  const size_t slot = x >> P.page_shift;
  if (unsigned(pg) >= unsigned(P.num_pages)) {
    raise_err(P.err, TF_ERR_SHAPE, kPage, rank, -1, b, int(slot), uint64_t(P.num_pages), uint64_t(unsigned(pg)), 0);
    pg = 0;
  }
  const size_t in_page = x & ((size_t(1) << P.page_shift) - 1);
  return P.hnd ? ((size_t(pg) * P.Hkv + kvh) << P.page_shift) + in_page
               : ((size_t(pg) << P.page_shift) + in_page) * size_t(P.Hkv) + kvh;
}
__device__ __forceinline__ size_t paged_row(const FdParams& P, const int* tbl, size_t x, int kvh, int b, int rank) {
  return paged_row_of(P, __ldg(tbl + (x >> P.page_shift)), x, kvh, b, rank);
}

__device__ __forceinline__ int split_count(const FdParams& P, int lr, int g) {
  (void)lr;  // every rank cuts the same splits
  return P.gS ? P.gS[g] : P.S;
}

// This launch's epochs (fd_epochs_begin): the device cells' values + 1, or
// the host's when the schedule is host-driven (P.depoch == nullptr).
__shared__ uint64_t s_fe, s_oe, s_ce;

__device__ __forceinline__ uint64_t fe(const FdParams& P) { return P.depoch ? s_fe : P.flag_epoch; }
__device__ __forceinline__ uint64_t oe(const FdParams& P) { return P.depoch ? s_oe : P.oflag_epoch; }
__device__ __forceinline__ uint64_t ce(const FdParams& P) { return P.depoch ? s_ce : P.epoch; }
// Inboxes / outboxes of this epoch's parity (peers are at most one run ahead).
__device__ __forceinline__ float* inbox_at(const FdParams& P, int dst) {
  return P.inbox_all[dst] + (P.depoch ? size_t(s_fe & 1) * P.inbox_pstride : 0);
}
__device__ __forceinline__ const float* rank_inbox(const FdParams& P, int lr) {
  return P.r[lr].inbox + (P.depoch ? size_t(s_fe & 1) * P.inbox_pstride : 0);
}
__device__ __forceinline__ float* outbox_at(const FdParams& P, int dst) {
  return P.outbox_all[dst] + (P.depoch ? size_t(s_oe & 1) * P.outbox_pstride : 0);
}
// Thread 0 at launch start (a __syncthreads follows in every kernel).
__device__ __forceinline__ void fd_epochs_begin(const FdParams& P) {
  if (!P.depoch) return;
  const volatile uint64_t* c = P.depoch;
  s_fe = c[P.owner ? 1 : 0] + 1;
  s_oe = c[2] + 1;
  s_ce = c[3] + 1;
}
// The launch's last CTA, after every CTA has passed its start.
__device__ __forceinline__ void fd_epochs_end(const FdParams& P) {
  if (!P.depoch) return;
  P.depoch[P.owner ? 1 : 0] = s_fe;
  if (P.owner) P.depoch[2] = s_oe;
  P.depoch[3] = s_ce;
}

__device__ __forceinline__ void consumer_bar() {  // the 8 consumer warps of fd_stream_kernel
  asm volatile("bar.sync 1, 256;" ::: "memory");
}
__device__ __forceinline__ void cta_bar(bool named) {
  if (named) consumer_bar();
  else __syncthreads();
}

// ---- combine monoid on wire rows (tilemath.hpp:186-220) -------------------
// One implementation for every fold so all schedules agree bit for bit.
// __fmul_rn/__fadd_rn keep the compiler from contracting to FMA, matching
// the reference's separately rounded arithmetic.
struct Part {
  float m, l;
};
__device__ __forceinline__ void combine_scalars(float am, float al, float bm, float bl,
                                                float* m, float* l, float* ax, float* ay,
                                                int* mode) {
  if (al == 0.0f) {
    *mode = 1;  // take b
    *m = bm;
    *l = bl;
    return;
  }
  if (bl == 0.0f) {
    *mode = 2;  // keep a
    *m = am;
    *l = al;
    return;
  }
  *mode = 0;
  const float mm = fmaxf(am, bm);
  *ax = expf(am - mm);
  *ay = expf(bm - mm);
  *m = mm;
  *l = __fadd_rn(__fmul_rn(al, *ax), __fmul_rn(bl, *ay));
}

__device__ __forceinline__ float combine_elem(int mode, float ao, float bo, float ax, float ay) {
  if (mode == 1) return bo;
  if (mode == 2) return ao;
  return __fadd_rn(__fmul_rn(ao, ax), __fmul_rn(bo, ay));
}

// acc (one wire row, in smem or registers per thread) <- acc (+) row.
// Cooperative over `nthreads` threads; each thread owns elements e = tid +
// k*nthreads of o.  Caller provides m/l in shared memory.
template <int MAXE>
__device__ __forceinline__ void fold_row(float& am, float& al, float* ao, const float* row,
                                         int d, int tid, int nthreads) {
  // Rows were written by other CTAs (or peers) during this launch: read them
  // through L2 (ld.cg).  L1 is not coherent, and a line shared with a
  // neighbouring row may already sit in this SM's L1 from an earlier fold.
  const float bm = __ldcg(row), bl = __ldcg(row + 1);
  float m, l, ax = 0.f, ay = 0.f;
  int mode;
  combine_scalars(am, al, bm, bl, &m, &l, &ax, &ay, &mode);
#pragma unroll
  for (int i = 0; i < MAXE; ++i) {
    const int e = tid + i * nthreads;
    if (e < d) ao[i] = combine_elem(mode, ao[i], __ldcg(row + 2 + e), ax, ay);
  }
  am = m;
  al = l;
}

__device__ __forceinline__ float load_kv(const void* p, size_t idx, int bf16) {
  return bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p)[idx])
              : static_cast<const float*>(p)[idx];
}

__device__ __forceinline__ void store_out(void* p, size_t idx, float v, int bf16) {
  if (bf16) static_cast<__nv_bfloat16*>(p)[idx] = __float2bfloat16_rn(v);
  else static_cast<float*>(p)[idx] = v;
}

// Split-partial workspace rows (internal, not the wire format): [m l - - o[d]]
// so o starts 16-byte aligned and the group fold reads it with 128-bit loads.
constexpr int kWsO = 4;
__host__ __device__ __forceinline__ int ws_row(int d) { return d + kWsO; }

// TFB_TRACE phase stamp (slot i of this CTA's 16), for tools/fd_trace.py.
__device__ __forceinline__ void trace_at(const FdParams& P, int i) {
  if (P.trace && threadIdx.x == 0) P.trace[size_t(blockIdx.x) * kTraceSlots + i] = globaltimer_ns();
}

// ---- generic split partial: one warp per q-head ----------------------------
// Writes ws rows [m | l | - - | o] (natural-log m) for the gs heads of the group.
__device__ void generic_split(const FdParams& P, int lr, int g, int sp, float* wsrow) {
  const FdRank& R = P.r[lr];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = g / P.Hkv, kvh = g % P.Hkv;
  const size_t k0 = size_t(sp) * P.split_len;
  const size_t k1 = min(P.len, k0 + P.split_len);
  const int d = P.d;
  const size_t kvbase = (size_t(b) * P.Hkv + kvh) * P.len * d;
  const int* tbl = P.paged ? R.pages + size_t(b) * P.pps : nullptr;
  for (int h = warp; h < P.gs; h += blockDim.x >> 5) {
    const int hq = kvh * P.gs + h;
    const size_t qbase = (size_t(b) * P.Hq + hq) * d;
    float q[8], o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = lane + 32 * i;
      q[i] = e < d ? load_kv(R.q, qbase + e, P.kv_bf16) : 0.0f;
      o[i] = 0.0f;
    }
    float m = -INFINITY, l = 0.0f;
    for (size_t j = k0; j < k1; ++j) {
      float part = 0.0f;
      const size_t kvj = tbl ? paged_row(P, tbl, j, kvh, b, R.rank) * d : kvbase + j * d;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = lane + 32 * i;
        if (e < d) part = __fadd_rn(part, __fmul_rn(q[i], load_kv(R.k, kvj + e, P.kv_bf16)));
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) part = __fadd_rn(part, __shfl_xor_sync(0xffffffffu, part, off));
      const float s = __fmul_rn(part, P.scale);
      if (!isfinite(s)) {
        if (lane == 0)
          raise_err(P.err, TF_ERR_NUMERIC, kNumeric, R.rank, -1, 0, 0, 0, 0,
                    (uint64_t(hq) << 32) | uint64_t(size_t(R.rank) * P.len + j));
        return;
      }
      const float mn = fmaxf(m, s);
      const float alpha = expf(m - mn);
      const float w = expf(s - mn);
      l = __fadd_rn(__fmul_rn(l, alpha), w);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = lane + 32 * i;
        if (e < d)
          o[i] = __fadd_rn(__fmul_rn(o[i], alpha), __fmul_rn(w, load_kv(R.v, kvj + e, P.kv_bf16)));
      }
      m = mn;
    }
    float* row = wsrow + size_t(h) * ws_row(d);
    if (lane == 0) {
      row[0] = m;
      row[1] = l;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = lane + 32 * i;
      if (e < d) row[kWsO + e] = o[i];
    }
  }
}

// ---- fast split partial: bf16, d = 128, gs = 8 -----------------------------
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t movtrans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ uint4 ldg_stream(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ uint32_t w4(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// 8 warps per CTA, 2 CTAs per SM at <= 128 registers: 16 streaming warps per
// SM keep ~128 KB of KV loads in flight (what HBM3e needs at ~2 us latency).
constexpr int kFastWarps = 8;
constexpr int kFastThreads = kFastWarps * 32;

// d index held by O^T accumulator row r of PV tile (i, j) (see header).
__device__ __forceinline__ int fast_d(int i, int j, int r) {
  return 32 * i + 8 * (r >> 1) + 2 * j + (r & 1);
}

// One warp: keys [kb, ke) of the group's stream; leaves its log2-domain
// partial for the 8 heads in smem (m2[8], l[8], o[8][128]).
// PAGED: K / V are the rank's page pools and every 16-key tile looks its
// two rows up in the batch's block table `tbl` (L1-resident; the rows of a
// tile may sit in two pages) -- the same keys in the same order, so a paged
// run is bitwise the contiguous run of the same logical KV.
template <bool HILO, bool PAGED>
__device__ void fast_warp_range(const FdParams& P, const __nv_bfloat16* K,
                                const __nv_bfloat16* V, const __nv_bfloat16* Q, size_t kb,
                                size_t ke, int stride, float* sm_m, float* sm_l, float* sm_o, int* bad,
                                const int* tbl = nullptr, int kvh = 0, int b = 0, int rank = 0) {
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, t = lane & 3;
  const float sl2 = P.scale * kLog2e;
  // Q^T fragments (head gq, d positions 8(t+4i) .. +8) are read from the
  // CTA's smem copy of the group's q each tile: 16 registers the KV software
  // pipeline needs more.
  const uint4* sq = reinterpret_cast<const uint4*>(Q);
  float o[8][4];
#pragma unroll
  for (int x = 0; x < 8; ++x) o[x][0] = o[x][1] = o[x][2] = o[x][3] = 0.0f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
  int badl = 0;
  const uint4 z = make_uint4(0, 0, 0, 0);
  uint64_t pol;  // K/V read once: L2 evict-first (see l2_evict_first_policy)
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint4 k_a[4], k_b[4], v_a[4], v_b[4];
  // Row a of each 16-key tile is key j0 + gq, row b is j0 + gq + 8: one
  // pointer per stream, lane slice folded in, tile/row/chunk offsets as
  // immediates (64-bit per-load addresses cost registers the loop needs).
  const __nv_bfloat16* kp = K + (kb + gq) * 128 + 8 * t;
  const __nv_bfloat16* vp = V + (kb + gq) * 128 + 8 * t;
  // (A one-tile-ahead register pipeline was measured: it spills at the
  //  128-register budget 16 warps/SM need and lost 10 %; the loads are issued
  //  at the top of each tile instead and the 16 resident warps overlap them.)
  // 16-key tiles kb, kb + stride, ... below ke.
  // PAGED: the block-table entries of the next tile's two rows are loaded
  // one tile ahead, so a tile's K/V loads never wait on a table lookup.
  int pg_a = 0, pg_b = 0;
  if (PAGED) {
    const int rem0 = int(ke - kb) - gq;
    if (rem0 > 0) pg_a = __ldg(tbl + ((ke - size_t(rem0)) >> P.page_shift));
    if (rem0 > 8) pg_b = __ldg(tbl + ((ke - size_t(rem0) + 8) >> P.page_shift));
  }
  for (int rem = int(ke - kb) - gq; rem > -gq; rem -= stride, kp += size_t(stride) * 128, vp += size_t(stride) * 128) {
    const bool va = rem > 0, vb = rem > 8;
    const __nv_bfloat16 *ka_p = kp, *kb_p = kp + 8 * 128, *va_p = vp, *vb_p = vp + 8 * 128;
    if (PAGED) {
      const size_t x = ke - size_t(rem);  // row a's key (row b: x + 8)
      const size_t oa = va ? paged_row_of(P, pg_a, x, kvh, b, rank) * 128 + 8 * t : 0;
      const size_t ob = vb ? paged_row_of(P, pg_b, x + 8, kvh, b, rank) * 128 + 8 * t : 0;
      const int rn = rem - stride;
      pg_a = rn > 0 ? __ldg(tbl + ((x + stride) >> P.page_shift)) : 0;
      pg_b = rn > 8 ? __ldg(tbl + ((x + stride + 8) >> P.page_shift)) : 0;
      ka_p = K + oa;
      kb_p = K + ob;
      va_p = V + oa;
      vb_p = V + ob;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      k_a[i] = va ? ldg_stream(ka_p + 32 * i, pol) : z;
      k_b[i] = vb ? ldg_stream(kb_p + 32 * i, pol) : z;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v_a[i] = va ? ldg_stream(va_p + 32 * i, pol) : z;
      v_b[i] = vb ? ldg_stream(vb_p + 32 * i, pol) : z;
    }
    // S^T = K . Q^T over 8 k-steps of 16 d.
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 qv = sq[gq * 16 + t + 4 * i];
#pragma unroll
      for (int h = 0; h < 2; ++h)
        mma_bf16(s, w4(k_a[i], 2 * h), w4(k_b[i], 2 * h), w4(k_a[i], 2 * h + 1),
                 w4(k_b[i], 2 * h + 1), w4(qv, 2 * h), w4(qv, 2 * h + 1));
    }
    // log2-domain scores; rows g (key ka) and g+8 (key kb8); cols 2t, 2t+1.
    float x0 = va ? s[0] * sl2 : -INFINITY, x1 = va ? s[1] * sl2 : -INFINITY;
    float x2 = vb ? s[2] * sl2 : -INFINITY, x3 = vb ? s[3] * sl2 : -INFINITY;
    badl |= (va && !(fabsf(x0) < INFINITY && fabsf(x1) < INFINITY)) ||
            (vb && !(fabsf(x2) < INFINITY && fabsf(x3) < INFINITY));
    float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    // HILO (fp32 output requested): the weights reach the tensor core as a
    // bf16 hi + lo pair (P = P_hi + P_lo to ~2^-16 relative) at one extra
    // MMA per PV step, which gives fp32-grade attention on bf16 K/V.  Else
    // (bf16 output, whose own rounding is 2^-9) a single bf16 P, with the
    // normalizer taken from the same rounded weights.
    const float e0 = exp2f(x0 - mn0), e1 = exp2f(x1 - mn1);
    const float e2 = exp2f(x2 - mn0), e3 = exp2f(x3 - mn1);
    const __nv_bfloat162 p01 = __floats2bfloat162_rn(e0, e1);
    const __nv_bfloat162 p23 = __floats2bfloat162_rn(e2, e3);
    __nv_bfloat162 r01, r23;
    if (HILO) {
      r01 = __floats2bfloat162_rn(e0 - __low2float(p01), e1 - __high2float(p01));
      r23 = __floats2bfloat162_rn(e2 - __low2float(p23), e3 - __high2float(p23));
      l0 = l0 * al0 + (e0 + e2);
      l1 = l1 * al1 + (e1 + e3);
    } else {
      l0 = l0 * al0 + (__low2float(p01) + __low2float(p23));
      l1 = l1 * al1 + (__high2float(p01) + __high2float(p23));
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      o[x][0] *= al0;
      o[x][1] *= al1;
      o[x][2] *= al0;
      o[x][3] *= al1;
    }
    const uint32_t pb0 = movtrans(*reinterpret_cast<const uint32_t*>(&p01));
    const uint32_t pb1 = movtrans(*reinterpret_cast<const uint32_t*>(&p23));
    uint32_t rb0 = 0, rb1 = 0;
    if (HILO) {
      rb0 = movtrans(*reinterpret_cast<const uint32_t*>(&r01));
      rb1 = movtrans(*reinterpret_cast<const uint32_t*>(&r23));
    }
    // O^T += V^T . P^T: tile (i, jp) covers d rows fast_d(i, 2jp, .) and
    // fast_d(i, 2jp+1, .).
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int jp = 0; jp < 2; ++jp) {
        const uint32_t a0 = movtrans(w4(v_a[i], 2 * jp));
        const uint32_t a1 = movtrans(w4(v_a[i], 2 * jp + 1));
        const uint32_t a2 = movtrans(w4(v_b[i], 2 * jp));
        const uint32_t a3 = movtrans(w4(v_b[i], 2 * jp + 1));
        mma_bf16(o[2 * i + jp], a0, a1, a2, a3, pb0, pb1);
        if (HILO) mma_bf16(o[2 * i + jp], a0, a1, a2, a3, rb0, rb1);
      }
    }
  }
  // Per-head normalizer: sum the per-lane partials over the 8 key rows.
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, off);
    l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  }
  if (gq == 0) {
    sm_m[2 * t] = m0;
    sm_m[2 * t + 1] = m1;
    sm_l[2 * t] = l0;
    sm_l[2 * t + 1] = l1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int jp = 0; jp < 2; ++jp) {
      const float* c = o[2 * i + jp];
      const int dA = fast_d(i, 2 * jp, gq), dB = fast_d(i, 2 * jp + 1, gq);
      sm_o[(2 * t) * 128 + dA] = c[0];
      sm_o[(2 * t + 1) * 128 + dA] = c[1];
      sm_o[(2 * t) * 128 + dB] = c[2];
      sm_o[(2 * t + 1) * 128 + dB] = c[3];
    }
  }
  if (badl) *bad = 1;
}

struct FastSmem {
  float m[kFastWarps][8];
  float l[kFastWarps][8];
  float o[kFastWarps][8 * 128];
  uint4 q[8 * 16];  // the group's 8 q heads x 128 d (bf16), fragment-ordered reads
  int bad;
  float wa[8][kFastWarps];  // per-head weight of each warp's partial, exp2(m_w - M)
  float hm[8], hl[8];       // per-head max M and weighted l
  unsigned long long wend[kFastWarps];  // TFB_TRACE: per-warp finish times
};

template <bool HILO, bool PAGED>
__device__ void fast_split(const FdParams& P, int lr, int g, int sp, float* wsrow,
                           FastSmem& sm) {
  const FdRank& R = P.r[lr];
  const int warp = threadIdx.x >> 5;
  const int b = g / P.Hkv, kvh = g % P.Hkv;
  const size_t k0 = size_t(sp) * P.split_len;
  const size_t k1 = min(P.len, k0 + P.split_len);
  // The CTA's warps interleave tile by tile over the split (warp w: tiles
  // w, w + 8, ...): contiguous per-warp ranges finished up to 13 us apart
  // inside a CTA (TFB_TRACE); interleaved, the warps share the same DRAM
  // pages and finish closer together (config 4: -1.7 %).  P.interleave = 0
  // (TFB_FD_CONTIGUOUS) restores contiguous ranges.
  size_t wb, we;
  int stride;
  if (P.interleave) {
    wb = min(k1, k0 + size_t(warp) * 16);
    we = k1;
    stride = 16 * kFastWarps;
  } else {
    const size_t per = ((k1 - k0 + kFastWarps - 1) / kFastWarps + 15) / 16 * 16;
    wb = min(k1, k0 + warp * per);
    we = min(k1, wb + per);
    stride = 16;
  }
  const __nv_bfloat16* K = static_cast<const __nv_bfloat16*>(R.k) + (size_t(b) * P.Hkv + kvh) * P.len * 128;
  const __nv_bfloat16* V = static_cast<const __nv_bfloat16*>(R.v) + (size_t(b) * P.Hkv + kvh) * P.len * 128;
  const __nv_bfloat16* Q = static_cast<const __nv_bfloat16*>(R.q) + (size_t(b) * P.Hq + kvh * 8) * 128;
  if (threadIdx.x == 0) sm.bad = 0;
  for (int i = threadIdx.x; i < 8 * 16; i += blockDim.x) sm.q[i] = reinterpret_cast<const uint4*>(Q)[i];
  __syncthreads();
  trace_at(P, 12);
  if (PAGED)
    fast_warp_range<HILO, true>(P, static_cast<const __nv_bfloat16*>(R.k), static_cast<const __nv_bfloat16*>(R.v),
                                reinterpret_cast<const __nv_bfloat16*>(sm.q), wb, we, stride, sm.m[warp], sm.l[warp],
                                sm.o[warp], &sm.bad, R.pages + size_t(b) * P.pps, kvh, b, R.rank);
  else
    fast_warp_range<HILO, false>(P, K, V, reinterpret_cast<const __nv_bfloat16*>(sm.q), wb, we, stride, sm.m[warp],
                                 sm.l[warp], sm.o[warp], &sm.bad);
  if (P.trace && (threadIdx.x & 31) == 0) sm.wend[warp] = globaltimer_ns();
  __syncthreads();
  trace_at(P, 13);
  if (P.trace && threadIdx.x == 0) {  // first / last warp of the CTA to finish streaming
    unsigned long long lo = ~0ull, hi = 0;
    for (int w = 0; w < kFastWarps; ++w) {
      lo = min(lo, sm.wend[w]);
      hi = max(hi, sm.wend[w]);
    }
    P.trace[size_t(blockIdx.x) * kTraceSlots + 10] = lo;
    P.trace[size_t(blockIdx.x) * kTraceSlots + 11] = hi;
    for (int w = 0; w < kFastWarps; ++w) P.trace[size_t(blockIdx.x) * kTraceSlots + 22 + w] = sm.wend[w];
  }
  if (sm.bad) {
    if (threadIdx.x == 0)
      raise_err(P.err, TF_ERR_NUMERIC, kNumeric, R.rank, -1, 0, 0, 0, 0,
                (uint64_t(kvh * 8) << 32) | uint64_t(size_t(R.rank) * P.len + k0));
    return;
  }
  // Fold of the warp partials (log2 domain), max first: the 8 weights of a
  // head, exp2(m_w - M), are computed once (64 exp2 per CTA) and every o
  // element is an ascending weighted sum -- the per-element online merge
  // this replaces spent 2 x 8 exp2 per element and ~2.5 us per item
  // (TFB_TRACE, config 3).  Then natural m.
  if (threadIdx.x < 8) {
    const int h = threadIdx.x;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kFastWarps; ++w)
      if (sm.l[w][h] != 0.0f) M = fmaxf(M, sm.m[w][h]);
    float L = 0.0f;
#pragma unroll
    for (int w = 0; w < kFastWarps; ++w) {
      const float bl = sm.l[w][h];
      const float a = bl != 0.0f ? exp2f(sm.m[w][h] - M) : 0.0f;
      sm.wa[h][w] = a;
      L = __fadd_rn(L, __fmul_rn(bl, a));
    }
    sm.hm[h] = M;
    sm.hl[h] = L;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 8 * 128; e += blockDim.x) {
    const int h = e >> 7, dd = e & 127;
    float o = 0.0f;
#pragma unroll
    for (int w = 0; w < kFastWarps; ++w) {  // a warp with no keys (weight 0) contributes nothing
      const float a = sm.wa[h][w];
      o = __fadd_rn(o, a != 0.0f ? __fmul_rn(sm.o[w][h * 128 + dd], a) : 0.0f);
    }
    float* row = wsrow + size_t(h) * ws_row(128);
    if (dd == 0) {
      row[0] = sm.hm[h] * kLn2;
      row[1] = sm.hl[h];
    }
    row[kWsO + dd] = o;
  }
}

// Ascending-order fold, batched (W <= 8, not fold_by_arrival): wait for the
// W sources in ascending order, then load every source's row of a head at
// once and combine them in ascending order in registers -- the same
// arithmetic as fold_group's wait-then-fold loop (bitwise), one L2 round
// trip per head instead of W dependent ones.  EL: d / 32 rounded up.
template <int EL>
__device__ __noinline__ bool fold_group_batched(const FdParams& P, int lr, int g, int& s_src) {
  const int G = P.B * P.Hkv, d = P.d, row_len = d + 2;
  const FdRank& R = P.r[lr];
  const int b = g / P.Hkv, kvh = g % P.Hkv;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // Ascending order, batched: wait for the W sources in ascending order,
    // then load every source's row of a head at once and combine them in
    // ascending order in registers -- the same arithmetic as the
    // wait-then-fold loop below (bitwise), one L2 round trip per head
    // instead of W dependent ones.
    if (threadIdx.x == 0) {
      int ok = 1;
      for (int i = 0; i < P.W && ok; ++i) {
        ok = wait_geq(R.flags + size_t(i) * G + g, fe(P), P.watchdog_ns, P.err, kWaitSignal, R.rank,
                      P.board, i, g, 0);
        if (ok && P.events_all[R.rank])  // first (only) read of source i's rows of g
          P.events_all[R.rank][(size_t(i) * G + g) * 2 + 1] = globaltimer_ns();
      }
      s_src = ok;
    }
    __syncthreads();
    const int ok = s_src;
    __syncthreads();
    if (!ok) return false;
    const size_t src_stride = size_t(P.B) * P.Hq * row_len;
    for (int h = warp; h < P.gs; h += nw) {
      const int hq = kvh * P.gs + h;
      const float* row0 = rank_inbox(P, lr) + (size_t(b) * P.Hq + hq) * row_len;
      float bm[8], bl[8], bo[8][EL];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < P.W) {
          const float* row = row0 + size_t(i) * src_stride;
          bm[i] = __ldcg(row);
          bl[i] = __ldcg(row + 1);
#pragma unroll
          for (int x = 0; x < EL; ++x) bo[i][x] = lane + 32 * x < d ? __ldcg(row + 2 + lane + 32 * x) : 0.0f;
        }
      }
      float m = -INFINITY, l = 0.0f, o[EL];
#pragma unroll
      for (int x = 0; x < EL; ++x) o[x] = 0.0f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < P.W) {
          float nm, nl, ax = 0.f, ay = 0.f;
          int mode;
          combine_scalars(m, l, bm[i], bl[i], &nm, &nl, &ax, &ay, &mode);
#pragma unroll
          for (int x = 0; x < EL; ++x) o[x] = combine_elem(mode, o[x], bo[i][x], ax, ay);
          m = nm;
          l = nl;
        }
      }
      if (l == 0.0f) {
        if (lane == 0) raise_err(P.err, TF_ERR_EMPTY_ATTENTION, kEmpty, R.rank, -1, 0, 0, 0, 0, uint64_t(hq));
        continue;
      }
      const size_t ooff = (size_t(b) * P.Hq + hq) * d;
#pragma unroll
      for (int x = 0; x < EL; ++x) {
        const int e = lane + 32 * x;
        if (e < d) {
          const float y = o[x] / l;
          store_out(R.out, ooff + e, y, P.out_bf16);
          if (P.owner)
            for (int dst = 0; dst < P.W; ++dst)
              if (dst != R.rank) outbox_at(P, dst)[ooff + e] = y;
        }
      }
    }
    if (P.owner) {
      __syncthreads();
      if (threadIdx.x < P.W && int(threadIdx.x) != R.rank) {
        uint64_t* f = P.oflags_all[threadIdx.x] + g;
        if ((P.local_dst >> threadIdx.x) & 1ull) {
          __threadfence();
          red_release_gpu(f, 1);
        } else {
          fence_sys();
          red_release_sys(f, 1);
        }
      }
    }
    return true;
  }

// d = 128 split fold, latency-lean: per warp, pass 1 reads its rows' (m, l)
// lane-parallel (one load per 32 rows) for the max, pass 2 streams the o
// rows as float4 per lane in batches of kFoldRB rows, every load of a batch
// in flight, weights broadcast from the lane that loaded the row.  The same
// arithmetic as fold_heads (wph warps per head, warp j of a head taking
// rows j, j + wph, ...; max first; ascending weighted sums; the wph warp
// partials combined in ascending warp order).  Eight warps work; the
// others only join the barriers.
__device__ __forceinline__ float4 ldcg_f4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }

__device__ __forceinline__ void emit_wire_row4(const FdParams& P, int lr, int g, int h, float M, float L, float4 O,
                                               int lane) {
  const int gs = P.gs, W = P.W, Hq = P.Hq, Hkv = P.Hkv, row_len = 130;
  const int rank = P.r[lr].rank;
  const int b = g / Hkv, kvh = g % Hkv;
  const size_t base_src = size_t(rank) * P.B * Hq * row_len;
  const size_t off = (size_t(b) * Hq + kvh * gs + h) * row_len;
  const int hq = kvh * gs + h;
  auto put = [&](float* r) {
    if (lane == 0) *reinterpret_cast<float2*>(r) = make_float2(M, L);
    reinterpret_cast<float2*>(r + 2 + 4 * lane)[0] = make_float2(O.x, O.y);
    reinterpret_cast<float2*>(r + 2 + 4 * lane)[1] = make_float2(O.z, O.w);
  };
  if (P.push) {
    for (int dst = 0; dst < W; ++dst) {
      if (P.owner && dst != g % W) continue;  // owner-combine: the group's owner only
      put(inbox_at(P, dst) + base_src + off);
    }
  } else {
    put(P.r[lr].pub + off);
  }
  if (P.direct) {
    if (L == 0.0f) {
      if (lane == 0) raise_err(P.err, TF_ERR_EMPTY_ATTENTION, kEmpty, rank, -1, 0, 0, 0, 0, uint64_t(hq));
      return;
    }
    const size_t ooff = (size_t(b) * Hq + hq) * 128 + 4 * lane;
    void* out = P.r[lr].out;
    store_out(out, ooff + 0, O.x / L, P.out_bf16);
    store_out(out, ooff + 1, O.y / L, P.out_bf16);
    store_out(out, ooff + 2, O.z / L, P.out_bf16);
    store_out(out, ooff + 3, O.w / L, P.out_bf16);
  }
}

__device__ __forceinline__ void fold_heads128(const FdParams& P, int lr, int g, int h0, int hc, float* s_wm,
                                              float* s_L, float* s_O) {
  const int G = P.B * P.Hkv, gs = P.gs, S = split_count(P, lr, g);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool act = warp < 8;
  const int wrl = ws_row(128);
  const float* grp = P.ws + ((size_t(lr) * G + g) * P.S) * gs * wrl;
  const int wph = hc >= 8 ? 1 : 8 / hc;
  auto rowp = [&](int h, int i) { return grp + (size_t(i) * gs + h) * wrl; };
  // Warp's rows j, j + wph, ... of head h -> (Mw, L, O[4 d of this lane]).
  // Rows are taken 32 at a time: lane u loads row u's (m, l) while the
  // first kFoldRB rows' o are already in flight; rows past the end load as
  // zeros with weight 0 (adding +0 leaves every sum's bits unchanged).
  auto fold_rows = [&](int h, int j, float& Mw, float& L, float4& O) {
    const int nr = j < S ? (S - j + wph - 1) / wph : 0;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    // pass 1: the max over every row of the warp (max is order-free)
    float2 ml0 = make_float2(0.f, 0.f);
    float4 v[kFoldRB];
#pragma unroll
    for (int x = 0; x < kFoldRB; ++x) v[x] = x < nr ? ldcg_f4(rowp(h, j + wph * x) + kWsO + 4 * lane) : z4;
    Mw = -INFINITY;
    for (int u0 = 0; u0 < nr; u0 += 32) {
      float2 ml = make_float2(0.f, 0.f);
      if (u0 + lane < nr) ml = __ldcg(reinterpret_cast<const float2*>(rowp(h, j + wph * (u0 + lane))));
      if (u0 == 0) ml0 = ml;
      float m = ml.y != 0.0f ? ml.x : -INFINITY;
#pragma unroll
      for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      Mw = fmaxf(Mw, m);
    }
    trace_at(P, 16);
    // pass 2: ascending weighted sums, kFoldRB rows per batch
    L = 0.0f;
    O = z4;
    for (int u0 = 0; u0 < nr; u0 += 32) {
      float2 ml = ml0;
      if (u0 > 0) {
        ml = make_float2(0.f, 0.f);
        if (u0 + lane < nr) ml = __ldcg(reinterpret_cast<const float2*>(rowp(h, j + wph * (u0 + lane))));
      }
      const float lw = ml.y, w = ml.y != 0.0f ? expf(ml.x - Mw) : 0.0f;
      for (int b0 = 0; b0 < 32 && u0 + b0 < nr; b0 += kFoldRB) {
        if (u0 + b0 > 0) {
#pragma unroll
          for (int x = 0; x < kFoldRB; ++x)
            v[x] = u0 + b0 + x < nr ? ldcg_f4(rowp(h, j + wph * (u0 + b0 + x)) + kWsO + 4 * lane) : z4;
        }
#pragma unroll
        for (int x = 0; x < kFoldRB; ++x) {
          const float wx = __shfl_sync(0xffffffffu, w, b0 + x), lx = __shfl_sync(0xffffffffu, lw, b0 + x);
          L = __fadd_rn(L, __fmul_rn(lx, wx));
          O.x = __fadd_rn(O.x, __fmul_rn(v[x].x, wx));
          O.y = __fadd_rn(O.y, __fmul_rn(v[x].y, wx));
          O.z = __fadd_rn(O.z, __fmul_rn(v[x].z, wx));
          O.w = __fadd_rn(O.w, __fmul_rn(v[x].w, wx));
        }
      }
    }
  };
  if (wph == 1) {
    if (!act) return;
    for (int hh = warp; hh < hc; hh += 8) {
      float M, L;
      float4 O;
      fold_rows(h0 + hh, 0, M, L, O);
      emit_wire_row4(P, lr, g, h0 + hh, M, L, O, lane);
    }
    return;
  }
  const int hh = warp / wph, j = warp % wph, h = h0 + hh;
  if (act) {
    float Mw, L;
    float4 O;
    fold_rows(h, j, Mw, L, O);
    trace_at(P, 17);
    if (lane == 0) {
      s_wm[warp] = Mw;
      s_L[warp] = L;
    }
    reinterpret_cast<float4*>(s_O + warp * 128)[lane] = O;
  }
  __syncthreads();
  trace_at(P, 18);
  if (act && j == 0) {
    float M = -INFINITY;
    for (int y = 0; y < wph; ++y)
      if (s_L[warp + y] != 0.0f) M = fmaxf(M, s_wm[warp + y]);
    float LL = 0.0f;
    float4 OO = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int y = 0; y < wph; ++y) {
      const float ly = s_L[warp + y];
      if (ly == 0.0f) continue;
      const float a = expf(s_wm[warp + y] - M);
      LL = __fadd_rn(LL, __fmul_rn(ly, a));
      const float4 oy = reinterpret_cast<const float4*>(s_O + (warp + y) * 128)[lane];
      OO.x = __fadd_rn(OO.x, __fmul_rn(oy.x, a));
      OO.y = __fadd_rn(OO.y, __fmul_rn(oy.y, a));
      OO.z = __fadd_rn(OO.z, __fmul_rn(oy.z, a));
      OO.w = __fadd_rn(OO.w, __fmul_rn(oy.w, a));
    }
    emit_wire_row4(P, lr, g, h, M, LL, OO, lane);
  }
  __syncthreads();
}

// ---- cross-rank fold of one (local rank, group) ---------------------------
// W inbox rows per q-head, folded in ascending source order with a
// per-source wait right before each fold (flash_decode.hpp:409-418) or --
// FdOptions::fold_by_arrival (:377-408) -- whichever source landed first,
// then finalized (tilemath.hpp:225-239) into out.  Returns false when a wait
// failed (the error is already raised).
__device__ __noinline__ bool fold_group(const FdParams& P, int lr, int g, int& s_src) {
  const int G = P.B * P.Hkv, d = P.d, row_len = d + 2;
  const FdRank& R = P.r[lr];
  const int b = g / P.Hkv, kvh = g % P.Hkv;
  constexpr int MAXH = 4;  // heads per warp (gs <= 32, 8 warps)
  float am[MAXH], al[MAXH], ao[MAXH][8];
#pragma unroll
  for (int j = 0; j < MAXH; ++j) {
    am[j] = -INFINITY;
    al[j] = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) ao[j][i] = 0.0f;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (!P.by_arrival && P.W <= 8)
    return d <= 128 ? fold_group_batched<4>(P, lr, g, s_src) : fold_group_batched<8>(P, lr, g, s_src);
  uint64_t folded = 0;
  for (int i = 0; i < P.W; ++i) {
    if (threadIdx.x == 0) {
      int src = -1;
      if (!P.by_arrival) {
        if (wait_geq(R.flags + size_t(i) * G + g, fe(P), P.watchdog_ns, P.err, kWaitSignal,
                     R.rank, P.board, i, g, 0))
          src = i;
      } else {
        const uint64_t t0 = globaltimer_ns();
        for (unsigned polls = 0; src < 0; ++polls) {
          for (int s = 0; s < P.W; ++s)
            if (!((folded >> s) & 1ull) && ld_acquire_sys(R.flags + size_t(s) * G + g) >= fe(P)) {
              src = s;
              break;
            }
          if (src < 0 && (polls & 63u) == 63u) {
            if (err_raised(P.err)) break;
            if (globaltimer_ns() - t0 > P.watchdog_ns) {
              raise_err(P.err, TF_ERR_DEADLOCK, kWaitSignal, R.rank, P.board, -1, g, fe(P), 0, 0);
              break;
            }
          }
        }
      }
      if (src >= 0 && P.events_all[R.rank]) P.events_all[R.rank][(size_t(src) * G + g) * 2 + 1] = globaltimer_ns();
      s_src = src;
    }
    __syncthreads();
    const int src = s_src;
    __syncthreads();
    if (src < 0) return false;
    folded |= 1ull << src;
    const float* base = rank_inbox(P, lr) + size_t(src) * P.B * P.Hq * row_len;
#pragma unroll
    for (int j = 0; j < MAXH; ++j) {
      const int h = warp + j * nw;
      if (h < P.gs)
        fold_row<8>(am[j], al[j], ao[j], base + (size_t(b) * P.Hq + kvh * P.gs + h) * row_len, d, lane, 32);
    }
  }
#pragma unroll
  for (int j = 0; j < MAXH; ++j) {
    const int h = warp + j * nw;
    if (h >= P.gs) continue;
    const int hq = kvh * P.gs + h;
    if (al[j] == 0.0f) {
      if (lane == 0) raise_err(P.err, TF_ERR_EMPTY_ATTENTION, kEmpty, R.rank, -1, 0, 0, 0, 0, uint64_t(hq));
      continue;
    }
    const size_t ooff = (size_t(b) * P.Hq + hq) * d;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = lane + 32 * i;
      if (e < d) {
        const float y = ao[j][i] / al[j];
        store_out(R.out, ooff + e, y, P.out_bf16);
        if (P.owner)  // owner-combine: the finalized row to every other rank
          for (int dst = 0; dst < P.W; ++dst)
            if (dst != R.rank) outbox_at(P, dst)[ooff + e] = y;
      }
    }
  }
  if (P.owner) {
    __syncthreads();
    if (threadIdx.x < P.W && int(threadIdx.x) != R.rank) {
      uint64_t* f = P.oflags_all[threadIdx.x] + g;
      if ((P.local_dst >> threadIdx.x) & 1ull) {
        __threadfence();
        red_release_gpu(f, 1);
      } else {
        fence_sys();
        red_release_sys(f, 1);
      }
    }
  }
  return true;
}

// Owner-combine, the receiving side: wait for group g's final rows from its
// owner, then copy them from the outbox into out (dtype of out).
__device__ __noinline__ bool take_group(const FdParams& P, int lr, int g) {
  const FdRank& R = P.r[lr];
  const int b = g / P.Hkv, kvh = g % P.Hkv, d = P.d, owner = g % P.W;
  __shared__ int s_ok;
  if (threadIdx.x == 0)
    s_ok = wait_geq(P.oflags_all[R.rank] + g, oe(P), P.watchdog_ns, P.err, kWaitSignal, R.rank,
                    P.board, owner, g, 0);
  __syncthreads();
  const int ok = s_ok;
  __syncthreads();
  if (!ok) return false;
  const size_t base = (size_t(b) * P.Hq + kvh * P.gs) * d;
  const float* src = outbox_at(P, R.rank) + base;
  for (int e = threadIdx.x; e < P.gs * d; e += blockDim.x) store_out(R.out, base + e, __ldcg(src + e), P.out_bf16);
  return true;
}

__device__ __forceinline__ float4 ldcg4(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}

// ---- split fold: the S split partials of a group -> the rank's wire rows --
// One sub-item = hc heads of one group (host-chosen so that a warp folds at
// most ~8 rows).  wph = 8 / hc warps share a head (hc <= 8), warp j of a
// head taking rows j, j + wph, ...; for hc > 8 every warp owns whole heads.
// Max-first and deterministic: per warp M = max m_i (over l_i != 0),
// w_i = exp(m_i - M), L = sum l_i w_i, O = sum o_i w_i (rows ascending),
// then the warps of a head combine the same way in ascending warp order --
// the monoid of combine_partials (tilemath.hpp:186-220) in two flat levels.  Every
// schedule runs this code, so schedules stay bitwise equal.  The first rows'
// o values are loaded before the m/l round trip: a sub-item costs about one
// L2 round trip.  Writes the wire rows [M | L | O] (every inbox when
// pushing, else the published partial) and, W = 1 fused (`direct`), the
// finalized output o / l (tilemath.hpp:225-239) -- bitwise what fold_group
// would compute from the single source.
// One head's rank partial [M | L | O] -> the wire rows (every inbox when
// pushing, else the published partial) and, W = 1 fused (direct), the
// finalized output O / L (tilemath.hpp:225-239, 244-258).  One warp.
template <int EL>
__device__ __forceinline__ void emit_wire_row(const FdParams& P, int lr, int g, int h, float M, float L,
                                              const float (&O)[EL], int lane) {
  const int d = P.d, gs = P.gs, W = P.W, Hq = P.Hq, Hkv = P.Hkv, row_len = d + 2;
  const int rank = P.r[lr].rank;
  const int b = g / Hkv, kvh = g % Hkv;
  const size_t base_src = size_t(rank) * P.B * Hq * row_len;
  const size_t off = (size_t(b) * Hq + kvh * gs + h) * row_len;
  const int hq = kvh * gs + h;
  if (P.push) {
    for (int dst = 0; dst < W; ++dst) {
      if (P.owner && dst != g % W) continue;  // owner-combine: the group's owner only
      float* r = inbox_at(P, dst) + base_src + off;
      if (lane == 0) {
        r[0] = M;
        r[1] = L;
      }
#pragma unroll
      for (int x = 0; x < EL; ++x)
        if (lane + 32 * x < d) r[2 + lane + 32 * x] = O[x];
    }
  } else {
    float* r = P.r[lr].pub + off;
    if (lane == 0) {
      r[0] = M;
      r[1] = L;
    }
#pragma unroll
    for (int x = 0; x < EL; ++x)
      if (lane + 32 * x < d) r[2 + lane + 32 * x] = O[x];
  }
  if (P.direct) {
    if (L == 0.0f) {
      if (lane == 0) raise_err(P.err, TF_ERR_EMPTY_ATTENTION, kEmpty, rank, -1, 0, 0, 0, 0, uint64_t(hq));
      return;
    }
    const size_t ooff = (size_t(b) * Hq + hq) * d;
#pragma unroll
    for (int x = 0; x < EL; ++x)
      if (lane + 32 * x < d) store_out(P.r[lr].out, ooff + lane + 32 * x, O[x] / L, P.out_bf16);
  }
}

// Eight warps do the work (a 10-warp fd_stream_kernel block: warps 8-9
// only join the barriers); `named`: the caller is the consumer warps alone.
template <int EL, int RB>
__device__ __forceinline__ void fold_heads(const FdParams& P, int lr, int g, int h0, int hc, float* s_wm,
                                        float* s_L, float* s_O, bool named = false) {
  const int G = P.B * P.Hkv;
  const int d = P.d, wrl = ws_row(d), gs = P.gs, S = split_count(P, lr, g), W = P.W, Hq = P.Hq, Hkv = P.Hkv,
            row_len = d + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool act = warp < 8;
  const int rank = P.r[lr].rank;
  const int direct = P.direct, push = P.push, out_bf16 = P.out_bf16;
  void* const out = P.r[lr].out;
  float* const pub = P.r[lr].pub;
  const int b = g / Hkv, kvh = g % Hkv;
  const float* grp = P.ws + ((size_t(lr) * G + g) * P.S) * gs * wrl;  // P.S: the layout's row stride
  const size_t base_src = size_t(rank) * P.B * Hq * row_len;
  const int wph = hc >= 8 ? 1 : 8 / hc;
  // Fold rows r0, r0 + step, ... of head h into (L, O[EL]) with max M.
  auto fold_rows = [&](int h, int r0, int step, float M, float& L, float (&O)[EL]) {
    L = 0.0f;
#pragma unroll
    for (int x = 0; x < EL; ++x) O[x] = 0.0f;
    for (int i0 = r0; i0 < S; i0 += RB * step) {
      float v[RB][EL];
      float2 ml[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int i = i0 + u * step;
        const float* row = grp + (size_t(i) * gs + h) * wrl;
        ml[u] = i < S ? make_float2(__ldcg(row), __ldcg(row + 1)) : make_float2(0.f, 0.f);
#pragma unroll
        for (int x = 0; x < EL; ++x) {
          const int e = lane + 32 * x;
          v[u][x] = (i < S && e < d) ? __ldcg(row + kWsO + e) : 0.0f;
        }
      }
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        if (i0 + u * step >= S) break;
        const float w = ml[u].y != 0.0f ? expf(ml[u].x - M) : 0.0f;
        L = __fadd_rn(L, __fmul_rn(ml[u].y, w));
#pragma unroll
        for (int x = 0; x < EL; ++x) O[x] = __fadd_rn(O[x], __fmul_rn(v[u][x], w));
      }
    }
  };
  auto row_max = [&](int h, int r0, int step) {
    float M = -INFINITY;
    for (int i = r0; i < S; i += step) {
      const float* row = grp + (size_t(i) * gs + h) * wrl;
      const float2 ml = make_float2(__ldcg(row), __ldcg(row + 1));
      if (ml.y != 0.0f) M = fmaxf(M, ml.x);
    }
    return M;
  };
  auto emit = [&](int h, float M, float L, const float (&O)[EL]) { emit_wire_row<EL>(P, lr, g, h, M, L, O, lane); };
  // One load batch (every row of this warp's share in flight at once, m/l
  // and o together): the common case, one L2 round trip per sub-item.
  auto one_batch = [&](int h, int r0, int step, float (&v)[RB][EL], float2 (&ml)[RB]) {
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int i = r0 + u * step;
      const float* row = grp + (size_t(i) * gs + h) * wrl;
      ml[u] = i < S ? make_float2(__ldcg(row), __ldcg(row + 1)) : make_float2(0.f, 0.f);
#pragma unroll
      for (int x = 0; x < EL; ++x) {
        const int e = lane + 32 * x;
        v[u][x] = (i < S && e < d) ? __ldcg(row + kWsO + e) : 0.0f;
      }
    }
  };
  auto sum_batch = [&](const float (&v)[RB][EL], const float2 (&ml)[RB], float M, float& L, float (&O)[EL]) {
    L = 0.0f;
#pragma unroll
    for (int x = 0; x < EL; ++x) O[x] = 0.0f;
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const float w = ml[u].y != 0.0f ? expf(ml[u].x - M) : 0.0f;  // rows past S carry l = 0
      L = __fadd_rn(L, __fmul_rn(ml[u].y, w));
#pragma unroll
      for (int x = 0; x < EL; ++x) O[x] = __fadd_rn(O[x], __fmul_rn(v[u][x], w));
    }
  };
  auto batch_max = [&](const float2 (&ml)[RB]) {
    float M = -INFINITY;
#pragma unroll
    for (int u = 0; u < RB; ++u)
      if (ml[u].y != 0.0f) M = fmaxf(M, ml[u].x);
    return M;
  };
  if (wph == 1) {
    // Whole heads per warp.
    if (!act) return;
    for (int hh = warp; hh < hc; hh += 8) {
      const int h = h0 + hh;
      float L, O[EL], M;
      if (S <= RB) {
        float v[RB][EL];
        float2 ml[RB];
        one_batch(h, 0, 1, v, ml);
        M = batch_max(ml);
        sum_batch(v, ml, M, L, O);
      } else {
        M = row_max(h, 0, 1);
        fold_rows(h, 0, 1, M, L, O);
      }
      emit(h, M, L, O);
    }
    return;
  }
  // wph warps per head: each warp folds its rows against its own max m_w
  // (nothing held across the barrier), then the head combines the wph warp
  // partials in ascending warp order: M = max m_w, L = sum L_w e^(m_w - M),
  // O = sum O_w e^(m_w - M).
  const int hh = warp / wph, j = warp % wph, h = h0 + hh;
  if (act) {
    float L, O[EL], Mw;
    if ((S + wph - 1) / wph <= RB) {
      float v[RB][EL];
      float2 ml[RB];
      one_batch(h, j, wph, v, ml);
      Mw = batch_max(ml);
      sum_batch(v, ml, Mw, L, O);
    } else {
      Mw = row_max(h, j, wph);
      fold_rows(h, j, wph, Mw, L, O);
    }
    if (lane == 0) {
      s_wm[warp] = Mw;
      s_L[warp] = L;
    }
#pragma unroll
    for (int x = 0; x < EL; ++x)
      if (lane + 32 * x < d) s_O[warp * d + lane + 32 * x] = O[x];
  }
  cta_bar(named);
  if (act && j == 0) {
    float M = -INFINITY;
    for (int y = 0; y < wph; ++y)
      if (s_L[warp + y] != 0.0f) M = fmaxf(M, s_wm[warp + y]);
    float LL = 0.0f, OO[EL];
#pragma unroll
    for (int x = 0; x < EL; ++x) OO[x] = 0.0f;
    for (int y = 0; y < wph; ++y) {
      const float ly = s_L[warp + y];
      if (ly == 0.0f) continue;
      const float a = expf(s_wm[warp + y] - M);
      LL = __fadd_rn(LL, __fmul_rn(ly, a));
#pragma unroll
      for (int x = 0; x < EL; ++x)
        if (lane + 32 * x < d) OO[x] = __fadd_rn(OO[x], __fmul_rn(s_O[(warp + y) * d + lane + 32 * x], a));
    }
    emit(h, M, LL, OO);
  }
  cta_bar(named);
}

// The phases after the splits are computed (both attention kernels):
// split-fold sub-items -> push + flags -> cross-rank fold (fused) ->
// owner-combine collection, then the last CTA resets the per-launch counts.
// Every thread of the block calls it; eight warps do fold work.
struct PostShared {
  unsigned* item;
  int* last;
  int* src;
  float *wm, *fL, *fO;
};
// Inlined into both kernels: as a separate (noinline) function it spilled
// (432 B of spill loads) on the latency-critical fold chain -- ~3 us per
// launch at config 3 (A/B against the round-1 build), ~2 us at config 4.
__device__ __forceinline__ void fd_post_phases_body(const FdParams& P, unsigned ranks_mask,
                                                    unsigned long long* tr, PostShared sh) {
  unsigned& s_item = *sh.item;
  int& s_last = *sh.last;
  int& s_src = *sh.src;
  float* s_wm = sh.wm;
  float* s_fL = sh.fL;
  float* s_fO = sh.fO;
  const int G = P.B * P.Hkv;
  auto stamp = [&](int i) {
    if (tr && threadIdx.x == 0) tr[i] = globaltimer_ns();
  };
  // direct + fold_once: a folding CTA counts itself out (ctr[2]) as soon as
  // its group's splits have landed -- its last read of any per-launch
  // counter -- and reads the ticket only after its fold, so the exit count's
  // round trip overlaps the fold instead of following it.
  unsigned exit_ticket = 0;  // thread 0: old ctr[2] + 1 (0: not counted yet)
  bool counted = false;
  // Split-fold phase: sub-items (group, hc heads) of every local rank this
  // CTA computed for, each waiting for its group's S splits.  Every compute
  // item has been claimed by a CTA that never blocks before publishing it,
  // so these waits always complete (no co-residency assumption), and every
  // rank's sub-items are claimed by CTAs that computed for it.  CTAs that ran
  // out of compute early fold finished groups while the others still
  // stream; in a loopback world a rank's CTAs never sit on another rank's
  // (straggling) groups -- they go on to the cross-rank fold, whose waits
  // are the ones the tax meter attributes (flash_decode_test.cpp:250-286).
  {
    const int nhc = P.gs / P.hc;
    const unsigned nsub = unsigned(G) * nhc;
    int lr = 0;
    bool folded = false;
    for (;;) {
      while (lr < P.nlocal && !((ranks_mask >> lr) & 1u)) ++lr;
      if (lr >= P.nlocal || (folded && P.fold_once)) break;  // fold_once: no claim round trip on the way out
      __syncthreads();
      if (threadIdx.x == 0) s_item = atomicAdd(&P.sfc[lr], 1u);
      __syncthreads();
      const unsigned item = s_item;
      __syncthreads();
      if (item >= nsub) {
        ++lr;
        continue;
      }
      const int hb = item % nhc, g = item / nhc;
      folded = true;
      stamp(13);
      if (threadIdx.x == 0) {
        // Intra-rank completion counter: a local spin, not a fabric signal
        // (not counted as a signal wait in the tax meter).
        const uint64_t* c = P.done + size_t(lr) * G + g;
        const uint64_t want = uint64_t(split_count(P, lr, g));
        const uint64_t t0 = globaltimer_ns();
        int ok = 1;
        for (unsigned polls = 0; ld_acquire_gpu(c) < want; ++polls) {
          if ((polls & 255u) == 255u) {
            if (err_raised(P.err)) {
              ok = 0;
              break;
            }
            if (globaltimer_ns() - t0 > P.watchdog_ns) {  // never silent: a DeadlockError
              raise_err(P.err, TF_ERR_DEADLOCK, kWaitSignal, P.r[lr].rank, -1, g, 0, want, ld_acquire_gpu(c), 0);
              ok = 0;
              break;
            }
          }
        }
        // A group the stream kernel already folded inline (its last split's
        // CTA, while compute items remained) is skipped here.
        if (ok && P.fstate && atomicCAS(&P.fstate[size_t(lr) * G + g], 0u, 2u) == 1u) ok = 2;
        s_last = ok;
      }
      __syncthreads();
      if (s_last == 2) continue;
      if (!s_last) break;  // an error elsewhere (e.g. NumericError) ends the launch
      stamp(9);
      if (P.direct && P.fold_once) {
        if (threadIdx.x == 0) exit_ticket = atomicAdd(&P.ctr[2], 1u) + 1u;
        counted = true;
      }
      if (P.d == 128) fold_heads128(P, lr, g, hb * P.hc, P.hc, s_wm, s_fL, s_fO);
      else if (P.d <= 128) fold_heads<4, 8>(P, lr, g, hb * P.hc, P.hc, s_wm, s_fL, s_fO);
      else fold_heads<8, 4>(P, lr, g, hb * P.hc, P.hc, s_wm, s_fL, s_fO);
      stamp(8);
      // The last sub-item of a group releases its flags to every rank
      // (push).  Every schedule counts, so the epoch-valued count stays in
      // step with the ticket epoch.
      const FdRank& R = P.r[lr];
      __syncthreads();
      if (threadIdx.x == 0) {
        // This sub-item's rows before the count (system scope only when a
        // destination inbox is on another device).
        // direct (W = 1): the rows are the final output, read only after the
        // launch retires, so the count and flags need no ordering.
        if (P.push && !P.direct) {
          if (P.local_dst == (P.W >= 64 ? ~0ull : ((1ull << P.W) - 1))) __threadfence();
          else __threadfence_system();
        }
        unsigned long long* gt = reinterpret_cast<unsigned long long*>(P.gtick + size_t(lr) * G + g);
        // direct (W = 1): the flag only records "the group landed" for the
        // flag snapshot -- nobody waits on it -- so head block 0 raises it
        // without a round trip on the ticket.
        s_last = P.direct ? hb == 0 : atom_add_acq_rel_gpu(gt, 1ull) == uint64_t(nhc) - 1;
      }
      __syncthreads();
      stamp(15);
      if (!P.push || !s_last) continue;
      stamp(7);
      if (threadIdx.x < P.W && (!P.owner || int(threadIdx.x) == g % P.W)) {
        uint64_t* f = P.flags_all[threadIdx.x] + size_t(R.rank) * G + g;
        if (P.events_all[threadIdx.x])  // this source's rows of g are in dst's inbox
          P.events_all[threadIdx.x][(size_t(R.rank) * G + g) * 2] = globaltimer_ns();
        if (P.direct) atomicAdd(reinterpret_cast<unsigned long long*>(f), 1ull);
        else if ((P.local_dst >> threadIdx.x) & 1ull) red_release_gpu(f, 1);
        else red_release_sys(f, 1);
      }
      stamp(3);
      if (P.fold_inline && !P.direct) {
        // Early fold: when every source of this group has already landed
        // (the last rank to push) fold it here instead of handing it to the
        // fold phase.  Non-blocking check.  Owner-combine: owners only.
        __syncthreads();
        if (threadIdx.x == 0) s_src = 0;
        if (threadIdx.x == 0 && (!P.owner || g % P.W == R.rank)) {
          bool all = true;
          for (int i = 0; i < P.W && all; ++i) all = ld_acquire_sys(R.flags + size_t(i) * G + g) >= fe(P);
          s_src = all && atomicMax(&P.claim[size_t(lr) * G + g], (unsigned long long)ce(P)) < ce(P);
        }
        __syncthreads();
        const int mine = s_src;
        __syncthreads();
        if (mine) fold_group(P, lr, g, s_src);
      }
    }
  }
  stamp(4);
  if (P.fold_inline && !P.direct) {
    // Fold phase: every compute item has been claimed by a CTA that never
    // blocks before pushing, so these waits always complete.
    const unsigned nfold = unsigned(P.nlocal) * G;
    for (;;) {
      __syncthreads();
      if (threadIdx.x == 0) {
        s_item = atomicAdd(&P.ctr[1], 1u);
        s_src = s_item < nfold && atomicMax(&P.claim[s_item], (unsigned long long)ce(P)) < ce(P);
      }
      __syncthreads();
      const unsigned item = s_item;
      const int mine = s_src;
      __syncthreads();
      if (item >= nfold) break;
      if (!mine) continue;  // folded early by its group's last CTA
      if (P.owner && int(item % G) % P.W != P.r[item / G].rank) continue;  // another rank's group
      stamp(5);
      if (!fold_group(P, item / G, item % G, s_src)) break;
    }
    if (P.owner) {
      // Owner-combine, last phase: collect the groups other ranks own.  Every
      // fold item was claimed before any CTA gets here, by CTAs whose waits
      // depend only on pushes that never wait -- these waits complete.
      for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_item = atomicAdd(&P.ctr[3], 1u);
        __syncthreads();
        const unsigned item = s_item;
        __syncthreads();
        if (item >= nfold) break;
        const int lr = item / G, g = item % G;
        if (g % P.W == P.r[lr].rank) continue;
        if (!take_group(P, lr, g)) break;
      }
    }
  }
  stamp(6);
  // Last CTA out resets the work counters and the per-launch completion
  // counts (done / gtick) for the next launch.  Plain per-launch counts,
  // not epoch-valued: the fused schedule keeps every local rank's counts in
  // one launch's buffer while the other schedules launch per rank, so an
  // epoch-valued count would fall behind when schedules are mixed.
  __syncthreads();
  if (threadIdx.x == 0) {
    if (counted) {
      s_last = exit_ticket == gridDim.x;
    } else {
      __threadfence();
      s_last = atomicAdd(&P.ctr[2], 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (s_last) {
    const int n = P.nlocal * G;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      P.done[i] = 0;
      P.gtick[i] = 0;
      if (P.fstate) P.fstate[i] = 0;
    }
    if (threadIdx.x == 0) {
      P.ctr[0] = 0;
      P.ctr[1] = 0;
      P.ctr[2] = 0;
      P.ctr[3] = 0;
      for (int i = 0; i < P.nlocal; ++i) P.sfc[i] = 0;
      fd_epochs_end(P);
    }
    __threadfence();
  }
}

// ---- the persistent kernel ------------------------------------------------
// MODE: 0 generic split, 1 fast split with bf16 P, 2 fast split with hi/lo P,
// 3 / 4 the same over a paged KV cache (own instances: the contiguous
// kernels keep their register allocation).
template <int MODE>
__global__ void __launch_bounds__(kFastThreads, 2) fd_attention_kernel(const __grid_constant__ FdParams P) {
  pdl_begin();
  __shared__ unsigned int s_item;
  __shared__ int s_last, s_src;
  __shared__ FastSmem fsm;
  __shared__ float s_wm[8], s_fL[8];
  __shared__ __align__(16) float s_fO[8 * 256];  // float4 rows (fold_heads128)
  const int G = P.B * P.Hkv;
  const unsigned total = unsigned(P.nlocal) * G * P.S;
  const int d = P.d, row_len = d + 2, wrl = ws_row(d);
  unsigned long long* tr = P.trace ? P.trace + size_t(blockIdx.x) * kTraceSlots : nullptr;
  auto stamp = [&](int i) {
    if (tr && threadIdx.x == 0) tr[i] = globaltimer_ns();
  };
  stamp(0);
  unsigned ranks_mask = 0;  // local ranks this CTA computed for
  __shared__ unsigned long long s_t0;  // CTA entry time (straggler model)
  // Device epochs: loads issued now, consumed only by the post phases, so
  // their L2 round trip overlaps the first item's claim and stream instead
  // of delaying both (measured: ~1 us per launch at config 3).
  uint64_t ep[3] = {0, 0, 0};
  if (threadIdx.x == 0) {
    s_t0 = globaltimer_ns();
    if (P.depoch) {
      const volatile uint64_t* c = P.depoch;
      ep[0] = c[P.owner ? 1 : 0];
      ep[1] = c[2];
      ep[2] = c[3];
    }
  }
  if (tr && threadIdx.x == 0)
    for (int i = 1; i < kTraceSlots; ++i)
      if (i != 12 && i != 13) tr[i] = 0;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(&P.ctr[0], 1u);
    __syncthreads();
    const unsigned item = s_item;
    __syncthreads();
    if (item >= total) break;
    const int sp = item % P.S;
    const int g = (item / P.S) % G;
    const int lr = item / (unsigned(P.S) * G);
    ranks_mask |= 1u << lr;
    if (P.r[lr].skew_ns) {  // straggler model: this rank's compute starts late
      if (threadIdx.x == 0)
        while (globaltimer_ns() - s_t0 < P.r[lr].skew_ns) __nanosleep(1000);
      __syncthreads();
    }
    float* grp = P.ws + ((size_t(lr) * G + g) * P.S) * P.gs * wrl;
    float* wsrow = grp + size_t(sp) * P.gs * wrl;
    if (MODE == 2) fast_split<true, false>(P, lr, g, sp, wsrow, fsm);
    else if (MODE == 1) fast_split<false, false>(P, lr, g, sp, wsrow, fsm);
    else if (MODE == 4) fast_split<true, true>(P, lr, g, sp, wsrow, fsm);
    else if (MODE == 3) fast_split<false, true>(P, lr, g, sp, wsrow, fsm);
    else generic_split(P, lr, g, sp, wsrow);
    stamp(1);
    if (tr && threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[14] = smid;
      tr[15] = item;
    }
    // Publish the split: bar.sync orders every thread's ws stores before
    // thread 0's release (cumulative), which the split-fold acquires.
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();  // every thread's ws rows (ordered by the barrier) before the count
      red_release_gpu(P.done + size_t(lr) * G + g, 1);
    }
  }
  stamp(2);
  if (P.depoch) {
    if (threadIdx.x == 0) {
      s_fe = ep[0] + 1;
      s_oe = ep[1] + 1;
      s_ce = ep[2] + 1;
    }
    __syncthreads();
  }
  fd_post_phases_body(P, ranks_mask, tr, PostShared{&s_item, &s_last, &s_src, s_wm, s_fL, s_fO});
}

// ---- TMA-fed split partials (bf16 K/V, d = 128, 8 q-heads per KV head) ----
// One CTA per SM, 10 warps:
//   warp 8  producer (one lane): walks the items this CTA claims (its first
//           item is blockIdx.x, the rest come from a global counter, each
//           claim issued one item ahead so its latency hides behind the
//           streaming) and streams every item's K and V through a
//           kStreamStages-deep smem ring with TMA (cp.async.bulk.tensor, 64
//           keys x 128 d of K and of V per stage, 128-byte swizzle), plus
//           the group's 8 q rows (1-D bulk copy) on the item's first stage.
//   warps 0-7  consumers: warp c takes 16-key tile (c & 3) of the stages
//           whose index inside their item has parity c >> 2 -- a function
//           of the item alone, so an item's partial is the same bits on any
//           CTA.  The math is the register decode of fast_warp_range fed from
//           smem: S^T = K.Q^T with mma.m16n8k16 on ldmatrix'd K, exp2-domain
//           online softmax with warp-shuffle max/sum, O^T += V^T.P^T on
//           ldmatrix.trans'd V.  At an item boundary each warp drops its
//           partial into one of two merge slots and goes straight on.
//   warp 9  merger: folds the 8 warp partials of each finished item (max
//           first, ascending warp order) into the item's split row, frees
//           the slot, then publishes the row (release onto the group's
//           completion count).  The fold phase folds the groups' split rows.
constexpr int kStreamStages = 5;
constexpr int kStageKeys = 64;                  // keys per stage (one 32 KB TMA box of K, one of V)
constexpr int kTPS = kStageKeys / 16;            // 16-key tiles per stage
constexpr int kStreamConsumers = 8;
constexpr int kProducerWarp = kStreamConsumers;
constexpr int kStreamThreads = 32 * (kStreamConsumers + 1);
constexpr int kStageKV = 2 * kStageKeys * 128 * 2;  // K + V of a stage, bf16
constexpr int kORow = 132;                   // padded merge row (conflict-free stores)
constexpr int kPubMax = 64;                  // merged rows the merger counts in per fence

struct FdMaps {
  CUtensorMap k[kMaxLocal];  // per local rank: [B*Hkv*len keys][2 halves][64 d] bf16 view, box 64 x 64 x 2
  CUtensorMap v[kMaxLocal];
};

struct StreamSmem {
  uint8_t kv[kStreamStages][kStageKV];  // 1024-aligned: [K half0 | K half1 | V half0 | V half1], kStageKeys x 128 B each
  uint8_t q[kStreamStages][8 * 128 * 2];
  float mo[kStreamConsumers][8 * kORow];  // the item merge: per warp o[head][d]
  float mm[kStreamConsumers][8], ml[kStreamConsumers][8], wa[8][kStreamConsumers];
  float hm[8], hl[8];
  int bad;
  int meta[kStreamStages][4];  // item (-1: end), keys | stage-in-item << 9, lr << 24 | g, split j
  uint64_t full[kStreamStages], empty[kStreamStages];
  unsigned ranks_mask;
  int npub, pub[kPubMax];  // merged split rows not yet counted in (lr << 24 | g)
};

// K/V are read once: stream them with an L2 evict-first policy, so the
// half-gigabyte pass does not flush what the tail needs from L2 (the split
// rows, the item table, the kernel's own code).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(sm100::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(sm100::smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4, %5}], [%6], %7;" ::"r"(sm100::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sm100::smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sm100::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(sm100::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
// Zero the bf16 halves of a V^T fragment register whose key is >= n.
__device__ __forceinline__ uint32_t mask_keys(uint32_t x, int key_lo, int n) {
  return (key_lo < n ? (x & 0xffffu) : 0u) | (key_lo + 1 < n ? (x & 0xffff0000u) : 0u);
}

__device__ __forceinline__ uint4 stream_item(const FdParams& P, unsigned it) {
  uint4 e = P.items[it / unsigned(P.nlocal)];
  e.x |= (it % unsigned(P.nlocal)) << 24;
  return e;
}

// Producer: lane 0 of kProducerWarp.
__device__ void stream_producer(const FdParams& P, const FdMaps& M, StreamSmem& sm) {
  unsigned seq = 0, skewed = 0;
  const uint64_t t0 = globaltimer_ns();
  const uint64_t pol = l2_evict_first_policy();
  // First item static (blockIdx.x); later ones claimed two items ahead so
  // that both the claim and the table-entry load of the next item have
  // long landed when the current item's last stage is issued.  Claims only
  // increase, so stopping at the first claim >= nitems loses no item.
  unsigned it = blockIdx.x;
  uint4 e = it < P.nitems ? stream_item(P, it) : make_uint4(0, 0, 0, 0);
  unsigned next = it < P.nitems ? gridDim.x + atomicAdd(&P.ctr[0], 1u) : ~0u;
  for (;;) {
    const bool end = it >= P.nitems;
    uint4 e_next = make_uint4(0, 0, 0, 0);
    unsigned next2 = ~0u;
    const int lr = int(e.x >> 24), g = int(e.x & 0xffffffu);
    const int b = g / P.Hkv, kvh = g % P.Hkv;
    const unsigned row0 = unsigned(g) * unsigned(P.len);  // [B][Hkv][len] rows: (b * Hkv + kvh) * len
    if (!end && P.r[lr].skew_ns && !((skewed >> lr) & 1u)) {  // straggler model: the rank starts late
      while (globaltimer_ns() - t0 < P.r[lr].skew_ns) __nanosleep(1000);
      skewed |= 1u << lr;
    }
    // Paged KV (page_size >= 64, so a 64-key stage never crosses a page):
    // the stage's page comes from the batch's block table; the next slot's
    // entry is loaded when a slot is entered, so the table read is off the
    // issue chain except at an item's first stage.
    const int* tbl = P.paged && !end ? P.r[lr].pages + size_t(b) * P.pps : nullptr;
    int cslot = -1, cpg = 0, nslot = -1, npg = 0;
    for (unsigned key = e.z;; key += kStageKeys) {
      if (!end && key >= e.w) break;
      const int st = int(seq % kStreamStages);
      sm100::mbar_wait(&sm.empty[st], ((seq / kStreamStages) & 1u) ^ 1u);
      volatile int* mt = sm.meta[st];
      mt[0] = end ? -1 : int(it);
      mt[1] = end ? 0 : int(min(unsigned(kStageKeys), e.w - key)) | int(((key - e.z) / kStageKeys) << 9);
      mt[2] = int(e.x);
      mt[3] = int(e.y);
      ++seq;
      if (end) {
        sm100::mbar_arrive(&sm.full[st]);
        return;
      }
      const bool first = key == e.z;
      sm100::mbar_arrive_expect_tx(&sm.full[st], kStageKV + (first ? 2048u : 0u));
      if (tbl) {
        const int slot = int(key >> P.page_shift);
        if (slot != cslot) {
          cpg = slot == nslot ? npg : __ldg(tbl + slot);
          cslot = slot;
          nslot = slot + 1;
          npg = nslot < P.pps ? __ldg(tbl + nslot) : 0;
          if (unsigned(cpg) >= unsigned(P.num_pages)) {
            raise_err(P.err, TF_ERR_SHAPE, kPage, P.r[lr].rank, -1, b, slot, uint64_t(P.num_pages),
                      uint64_t(unsigned(cpg)), 0);
            cpg = 0;
          }
        }
        const int in_page = int(key & ((1u << P.page_shift) - 1u));
        if (P.hnd) {  // [pages][Hkv][page][d]: one row range per (page, kv head)
          const int row = ((cpg * P.Hkv + kvh) << P.page_shift) + in_page;
          tma_load_3d(sm.kv[st], &M.k[lr], &sm.full[st], 0, row, 0, pol);
          tma_load_3d(sm.kv[st] + kStageKV / 2, &M.v[lr], &sm.full[st], 0, row, 0, pol);
        } else {  // [pages][page][Hkv][d]: key rows Hkv * 256 B apart
          const int krow = (cpg << P.page_shift) + in_page;
          tma_load_4d(sm.kv[st], &M.k[lr], &sm.full[st], 0, krow, kvh, 0, pol);
          tma_load_4d(sm.kv[st] + kStageKV / 2, &M.v[lr], &sm.full[st], 0, krow, kvh, 0, pol);
        }
      } else {
        tma_load_3d(sm.kv[st], &M.k[lr], &sm.full[st], 0, int(row0 + key), 0, pol);
        tma_load_3d(sm.kv[st] + kStageKV / 2, &M.v[lr], &sm.full[st], 0, int(row0 + key), 0, pol);
      }
      if (first) {
        bulk_load(sm.q[st], static_cast<const __nv_bfloat16*>(P.r[lr].q) + (size_t(b) * P.Hq + kvh * 8) * 128, 2048,
                  &sm.full[st]);
        // The item after next: claimed now, its successor's table entry
        // loaded now -- neither is waited on before this item is issued.
        if (next < P.nitems) {
          e_next = stream_item(P, next);
          next2 = gridDim.x + atomicAdd(&P.ctr[0], 1u);
        }
      }
    }
    it = next;
    e = e_next;
    next = next2;
  }
}

// Consumer thread 0: fence once (after the barrier that ordered every
// consumer's row stores), then count every merged split row in.
__device__ __forceinline__ void stream_publish(const FdParams& P, StreamSmem& sm) {
  const int G = P.B * P.Hkv;
  __threadfence();  // every consumer's row stores (ordered by the preceding barrier) before the counts
  for (int i = 0; i < sm.npub; ++i)
    atomicAdd(reinterpret_cast<unsigned long long*>(P.done + size_t(sm.pub[i] >> 24) * G + (sm.pub[i] & 0xffffff)), 1ull);
  sm.npub = 0;
}

// The 8 consumer warps' partials of one item -> its split row (the fold of
// fast_split: per head M = max m_w over warps with l_w != 0, weights
// exp2(m_w - M), ascending-warp sums).  Three named barriers; the row's
// completion count is added at the end of the compute (stream_publish), so
// nothing here waits on the memory system -- the producer keeps filling
// the ring meanwhile.
__device__ __forceinline__ void stream_merge_item(const FdParams& P, StreamSmem& sm, int lrg, int j, float m0,
                                                  float m1, float l0, float l1, const float (&o)[8][4], int badl) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, t = lane & 3;
  const int G = P.B * P.Hkv;
  const int lr = lrg >> 24, g = lrg & 0xffffff;
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, off);
    l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  }
  if (gq == 0) {
    sm.mm[warp][2 * t] = m0;
    sm.mm[warp][2 * t + 1] = m1;
    sm.ml[warp][2 * t] = l0;
    sm.ml[warp][2 * t + 1] = l1;
  }
  float* ow = sm.mo[warp];
#pragma unroll
  for (int db = 0; db < 8; ++db) {
    const int dA = 16 * db + gq;
    ow[(2 * t) * kORow + dA] = o[db][0];
    ow[(2 * t + 1) * kORow + dA] = o[db][1];
    ow[(2 * t) * kORow + dA + 8] = o[db][2];
    ow[(2 * t + 1) * kORow + dA + 8] = o[db][3];
  }
  if (__any_sync(0xffffffffu, badl) && lane == 0) sm.bad = 1;
  consumer_bar();
  if (threadIdx.x < 8) {
    const int h = threadIdx.x;
    float Mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kStreamConsumers; ++w)
      if (sm.ml[w][h] != 0.0f) Mx = fmaxf(Mx, sm.mm[w][h]);
    float L = 0.0f;
#pragma unroll
    for (int w = 0; w < kStreamConsumers; ++w) {
      const float bl = sm.ml[w][h];
      const float a = bl != 0.0f ? exp2f(sm.mm[w][h] - Mx) : 0.0f;
      sm.wa[h][w] = a;
      L = __fadd_rn(L, __fmul_rn(bl, a));
    }
    sm.hm[h] = Mx;
    sm.hl[h] = L;
  }
  consumer_bar();
  // 256 threads x 4 consecutive d (float4) = 8 heads x 128 d.
  const int wrl = ws_row(128);
  float* wsrow = P.ws + ((size_t(lr) * G + g) * P.S + j) * 8 * wrl;
  {
    const int h = threadIdx.x >> 5, dd = 4 * lane;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < kStreamConsumers; ++w) {
      const float a = sm.wa[h][w];
      const float4 x = *reinterpret_cast<const float4*>(&sm.mo[w][h * kORow + dd]);
      acc.x = __fadd_rn(acc.x, a != 0.0f ? __fmul_rn(x.x, a) : 0.0f);
      acc.y = __fadd_rn(acc.y, a != 0.0f ? __fmul_rn(x.y, a) : 0.0f);
      acc.z = __fadd_rn(acc.z, a != 0.0f ? __fmul_rn(x.z, a) : 0.0f);
      acc.w = __fadd_rn(acc.w, a != 0.0f ? __fmul_rn(x.w, a) : 0.0f);
    }
    float* row = wsrow + size_t(h) * wrl;
    *reinterpret_cast<float4*>(row + kWsO + dd) = acc;
    if (lane == 0) *reinterpret_cast<float2*>(row) = make_float2(sm.hm[h] * kLn2, sm.hl[h]);
  }
  consumer_bar();  // the smem merge area is free again
  if (threadIdx.x == 0) {
    if (sm.bad) {
      raise_err(P.err, TF_ERR_NUMERIC, kNumeric, P.r[lr].rank, -1, 0, 0, 0, 0,
                (uint64_t((g % P.Hkv) * 8) << 32) | uint64_t(size_t(P.r[lr].rank) * P.len));
      sm.bad = 0;
    }
    sm.ranks_mask |= 1u << lr;
    sm.pub[sm.npub++] = lrg;
    if (sm.npub == kPubMax) stream_publish(P, sm);
  }
}

template <bool HILO>
__device__ void stream_consumer(const FdParams& P, StreamSmem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t = lane & 3;
  // Warp c takes 16-key tile c % kTPS of the stages whose index inside
  // their item is c / kTPS modulo 8 / kTPS.
  constexpr int kSel = kStreamConsumers / kTPS;
  const int tl = warp % kTPS;
  const unsigned sel = unsigned(warp / kTPS);
  const float sl2 = P.scale * kLog2e;
  // Lane-constant parts of the ldmatrix addresses (128-byte swizzle: the
  // 16-byte chunk index is XORed with the key row's low 3 bits).
  const uint32_t krow = uint32_t(tl * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * 128;
  const uint32_t vrow = uint32_t(tl * 16 + (lane & 7) + ((lane >> 4) & 1) * 8) * 128;
  const int khi = lane >> 4, vhi = (lane >> 3) & 1, sw = lane & 7;
  int cur = -1, cur_lrg = 0, cur_j = 0;
  float o[8][4];
  uint32_t qb[8][2];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
  int badl = 0;
  for (unsigned seq = 0;; ++seq) {
    const int st = int(seq % kStreamStages);
    sm100::mbar_wait(&sm.full[st], (seq / kStreamStages) & 1u);
    if (seq == 0 && P.trace && threadIdx.x == 0) P.trace[size_t(blockIdx.x) * kTraceSlots + 10] = globaltimer_ns();
    const volatile int* mt = sm.meta[st];
    const int item = mt[0], nk = mt[1] & 0x1ff, sidx = mt[1] >> 9, lrg = mt[2], j = mt[3];
    if (item != cur) {
      if (cur >= 0) {
        const uint64_t tm = P.trace ? globaltimer_ns() : 0;
        stream_merge_item(P, sm, cur_lrg, cur_j, m0, m1, l0, l1, o, badl);
        if (P.trace && threadIdx.x == 0) {
          unsigned long long* tr = P.trace + size_t(blockIdx.x) * kTraceSlots;
          tr[11] += 1;
          tr[12] += globaltimer_ns() - tm;
        }
      }
      if (item < 0) {
        if (threadIdx.x == 0) stream_publish(P, sm);
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&sm.empty[st]);
        break;
      }
      cur = item;
      cur_lrg = lrg;
      cur_j = j;
      const uint32_t* qs = reinterpret_cast<const uint32_t*>(sm.q[st]);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        qb[kk][0] = qs[gq * 64 + 8 * kk + t];
        qb[kk][1] = qs[gq * 64 + 8 * kk + 4 + t];
      }
#pragma unroll
      for (int x = 0; x < 8; ++x) o[x][0] = o[x][1] = o[x][2] = o[x][3] = 0.0f;
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.0f;
      badl = 0;
    }
    const int n = nk - tl * 16;  // valid keys of this warp's tile
    if ((unsigned(sidx) % kSel) == sel && n > 0) {
      const uint32_t kb = sm100::smem_u32(sm.kv[st]), vb = kb + kStageKV / 2;
      // S^T over 8 k-steps of 16 d as four independent accumulator chains
      // (k-steps c, c + 4), summed in a fixed order: half the dependent
      // MMA latency per tile of one 8-step chain.
      float sc[4][4];
#pragma unroll
      for (int c = 0; c < 4; ++c) sc[c][0] = sc[c][1] = sc[c][2] = sc[c][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4(kb + (kk >> 2) * (kStageKeys * 128) + krow + ((((2 * kk + khi) & 7) ^ sw) << 4), a0, a1, a2, a3);
        mma_bf16(sc[kk & 3], a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
      }
      float s[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) s[r] = (sc[0][r] + sc[1][r]) + (sc[2][r] + sc[3][r]);
      const bool va = gq < n, vbk = gq + 8 < n;
      const float x0 = va ? s[0] * sl2 : -INFINITY, x1 = va ? s[1] * sl2 : -INFINITY;
      const float x2 = vbk ? s[2] * sl2 : -INFINITY, x3 = vbk ? s[3] * sl2 : -INFINITY;
      badl |= (va && !(fabsf(x0) < INFINITY && fabsf(x1) < INFINITY)) ||
              (vbk && !(fabsf(x2) < INFINITY && fabsf(x3) < INFINITY));
      float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
      }
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      const float e0 = exp2f(x0 - mn0), e1 = exp2f(x1 - mn1);
      const float e2 = exp2f(x2 - mn0), e3 = exp2f(x3 - mn1);
      const __nv_bfloat162 p01 = __floats2bfloat162_rn(e0, e1);
      const __nv_bfloat162 p23 = __floats2bfloat162_rn(e2, e3);
      __nv_bfloat162 r01, r23;
      if (HILO) {
        r01 = __floats2bfloat162_rn(e0 - __low2float(p01), e1 - __high2float(p01));
        r23 = __floats2bfloat162_rn(e2 - __low2float(p23), e3 - __high2float(p23));
        l0 = l0 * al0 + (e0 + e2);
        l1 = l1 * al1 + (e1 + e3);
      } else {
        l0 = l0 * al0 + (__low2float(p01) + __low2float(p23));
        l1 = l1 * al1 + (__high2float(p01) + __high2float(p23));
      }
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        o[x][0] *= al0;
        o[x][1] *= al1;
        o[x][2] *= al0;
        o[x][3] *= al1;
      }
      const uint32_t pb0 = movtrans(*reinterpret_cast<const uint32_t*>(&p01));
      const uint32_t pb1 = movtrans(*reinterpret_cast<const uint32_t*>(&p23));
      uint32_t rb0 = 0, rb1 = 0;
      if (HILO) {
        rb0 = movtrans(*reinterpret_cast<const uint32_t*>(&r01));
        rb1 = movtrans(*reinterpret_cast<const uint32_t*>(&r23));
      }
#pragma unroll
      for (int db = 0; db < 8; ++db) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(vb + (db >> 2) * (kStageKeys * 128) + vrow + ((((2 * db + vhi) & 7) ^ sw) << 4), a0, a1, a2, a3);
        if (n < 16) {  // keys past the item: P is 0 there, and V must not be Inf/NaN either
          a0 = mask_keys(a0, 2 * t, n);
          a1 = mask_keys(a1, 2 * t, n);
          a2 = mask_keys(a2, 8 + 2 * t, n);
          a3 = mask_keys(a3, 8 + 2 * t, n);
        }
        mma_bf16(o[db], a0, a1, a2, a3, pb0, pb1);
        if (HILO) mma_bf16(o[db], a0, a1, a2, a3, rb0, rb1);
      }
    }
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(&sm.empty[st]);
  }
}

template <bool HILO>
__global__ void __launch_bounds__(kStreamThreads, 1)
    fd_stream_kernel(const __grid_constant__ FdParams P, const __grid_constant__ FdMaps M) {
  pdl_begin();
  extern __shared__ uint8_t fd_smem_raw[];
  StreamSmem& sm = *reinterpret_cast<StreamSmem*>((reinterpret_cast<uintptr_t>(fd_smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ unsigned int s_item;
  __shared__ int s_last, s_src;
  __shared__ float s_wm[8], s_fL[8];
  __shared__ __align__(16) float s_fO[8 * 256];  // float4 rows (fold_heads128)
  unsigned long long* tr = P.trace ? P.trace + size_t(blockIdx.x) * kTraceSlots : nullptr;
  if (tr && threadIdx.x == 0) {
    tr[0] = globaltimer_ns();
    for (int i = 1; i < kTraceSlots; ++i) tr[i] = 0;
  }
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStreamStages; ++i) {
      sm100::mbar_init(&sm.full[i], 1);
      sm100::mbar_init(&sm.empty[i], kStreamConsumers);
    }
    sm.bad = 0;
    sm.ranks_mask = 0;
    sm.npub = 0;
    fd_epochs_begin(P);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x == 32 * kProducerWarp) {
    for (int i = 0; i < P.nlocal; ++i) {
      sm100::tma_prefetch(&M.k[i]);
      sm100::tma_prefetch(&M.v[i]);
    }
  }
  __syncthreads();
  if (warp == kProducerWarp) {
    if ((threadIdx.x & 31) == 0) stream_producer(P, M, sm);
  } else {
    stream_consumer<HILO>(P, sm);
    if (tr && threadIdx.x == 0) tr[1] = globaltimer_ns();
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[14] = smid;
    tr[2] = globaltimer_ns();
  }
  fd_post_phases_body(P, sm.ranks_mask, tr, PostShared{&s_item, &s_last, &s_src, s_wm, s_fL, s_fO});
}

// Push this rank's published rows into every inbox slot `self` and signal
// (dst, row=self, slot=0); block 0 then optionally waits for every source
// (independent_ag's collective-internal wait-all, flash_decode.hpp:277-284).
__global__ void fd_push_kernel(const float* pub, size_t row_floats, int self, int W,
                               FdParams P, int wait_all) {
  const int dst = blockIdx.x;
  float* ib = P.inbox_all[dst] + size_t(self) * row_floats;
  for (size_t e = threadIdx.x; e < row_floats; e += blockDim.x) ib[e] = pub[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_sys();
    red_release_sys(P.flags_all[dst] + self, 1);
  }
  if (wait_all && dst == 0 && threadIdx.x == 0) {
    for (int s = 0; s < W; ++s)
      if (!wait_geq(P.r[0].flags + s, P.flag_epoch, P.watchdog_ns, P.err, kWaitSignal, self, P.board, s,
                    0, 0))
        return;
  }
}

// BSP gather (flash_decode.hpp:234-241): copy every source's published row
// into the local stage [W][B][Hq][d+2].
__global__ void fd_gather_kernel(float* stage, size_t row_floats, FdParams P, int W) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < size_t(W) * row_floats;
       e += size_t(gridDim.x) * blockDim.x) {
    const int s = int(e / row_floats);
    stage[e] = P.inbox_all[s][e % row_floats];  // inbox_all carries the pubs here
  }
}

// Fold kernel (bsp / independent_ag / fine_waits): one CTA per (b, hq) row,
// optional per-source waits right before each fold (fine_waits,
// flash_decode.hpp:333-338).
__global__ void fd_fold_kernel(const float* src_rows, void* out, FdParams P, int self,
                               const uint64_t* flags, int wait) {
  const int row = blockIdx.x;  // b * Hq + hq
  const int d = P.d, row_len = d + 2;
  __shared__ int ok;
  if (threadIdx.x == 0) ok = 1;
  __syncthreads();
  float am = -INFINITY, al = 0.0f, ao[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) ao[i] = 0.0f;
  const size_t stride = size_t(P.B) * P.Hq * row_len;
  for (int s = 0; s < P.W; ++s) {
    if (wait) {
      if (threadIdx.x == 0 &&
          !wait_geq(flags + s, P.flag_epoch, P.watchdog_ns, P.err, kWaitSignal, self, P.board, s, 0, 0))
        ok = 0;
      __syncthreads();
      if (!ok) return;
    }
    fold_row<8>(am, al, ao, src_rows + size_t(s) * stride + size_t(row) * row_len, d,
                threadIdx.x, 32);
  }
  if (al == 0.0f) {
    if (threadIdx.x == 0)
      raise_err(P.err, TF_ERR_EMPTY_ATTENTION, kEmpty, self, -1, 0, 0, 0, 0, uint64_t(row % P.Hq));
    return;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = threadIdx.x + 32 * i;
    if (e < d) store_out(out, size_t(row) * d + e, ao[i] / al, P.out_bf16);
  }
}

}  // namespace

static bool fast_ok(const tf_fd_shape& s) {
  if (std::getenv("TFB_FD_GENERIC")) return false;  // debugging aid
  return s.kv_dtype == TF_BF16 && s.head_dim == 128 && s.q_heads / s.kv_heads == 8;
}

// Split count: enough (group, split) items to cover the SMs a few times,
// never fewer than 64 positions per split.  Shape-only, so every schedule
// and every rank cuts identically.
static int choose_splits(const tf_fd_shape& s, size_t len, int sms) {
  const long groups = long(s.batch) * s.kv_heads;
  // ~2 items per SM: enough CTAs to saturate HBM, few enough splits that the
  // group fold (S rows per head) stays short (measured sweep, profiles/).
  // Rounded down: a few extra items would start a mostly idle second wave
  // (measured, config 4: S = 1 -> 625 us, S = 2 -> 639 us).
  long want = std::max(1L, long(sms) * 2 / groups);
  long maxs = long((len + 63) / 64);
  long S = std::max(1L, std::min(want, maxs));
  if (const char* e = std::getenv("TFB_FD_SPLITS")) S = std::max(1L, std::min(std::atol(e), maxs));
  return int(S);
}

// ---- fd_stream_kernel host side ------------------------------------------
using FdEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static FdEncodeFn fd_encode_fn() {
  static std::atomic<FdEncodeFn> fn{nullptr};
  FdEncodeFn f = fn.load();
  if (!f) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<FdEncodeFn>(p);
    fn.store(f);
  }
  return f;
}

// K or V of one rank, [rows = B * Hkv * len][128] bf16, viewed as
// (64 d, rows, 2 halves) with strides (2 B, 256 B, 128 B): a box of
// (64, 64, 2) lands in smem as [half][64 keys][128 B], swizzled by 128 B, so
// ldmatrix reads 8 key rows of one 16-byte d chunk conflict-free.
static tf_status fd_kv_map(CUtensorMap* m, const void* base, size_t rows) {
  FdEncodeFn enc = fd_encode_fn();
  if (!enc) return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, rows, 2};
  cuuint64_t strides[2] = {256, 128};
  cuuint32_t box[3] = {64, uint32_t(kStageKeys), 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled (flash decode K/V) failed (" + std::to_string(int(r)) + ")");
  return TF_OK;
}

// Paged NHD pool [pages][page][Hkv][d] as [key rows][Hkv][2 halves][64 d]
// with the key dimension second, so a box lands in smem exactly like the
// contiguous map's [2 halves][64 keys][64 d].
static tf_status fd_kv_map_nhd(CUtensorMap* m, const void* base, size_t key_rows, int hkv) {
  FdEncodeFn enc = fd_encode_fn();
  if (!enc) return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {64, key_rows, cuuint64_t(hkv), 2};
  cuuint64_t strides[3] = {cuuint64_t(hkv) * 256, 256, 128};
  cuuint32_t box[4] = {64, uint32_t(kStageKeys), 1, 2};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled (paged NHD K/V) failed (" + std::to_string(int(r)) + ")");
  return TF_OK;
}

// Item table of fd_stream_kernel: a fixed function of the shape and the
// grid, so every run cuts the same splits (bitwise-reproducible partials
// whatever CTA computes them).  Guided sizes: each item takes
// remaining / (div * grid) keys (rounded up to 64, at least min_keys), the
// groups taking turns, so items shrink as the work runs out and CTAs that
// claim dynamically finish within about one small item of each other.
struct FdPlan {
  std::vector<uint4> items;
  std::vector<int> gS;
  int S_max = 1;
};
static FdPlan fd_plan(int G, size_t len, unsigned grid) {
  const int nlocal = 1;
  FdPlan pl;
  size_t min_keys = 256;
  if (const char* e = std::getenv("TFB_FD_MINKEYS")) min_keys = std::max<size_t>(64, std::strtoull(e, nullptr, 10));
  const bool group_major = std::getenv("TFB_FD_GROUP_MAJOR") != nullptr;
  // Items are remaining / (div * grid): half a CTA's fair share at most, so
  // a CTA streaming ~15 % slower than the rest (measured spread) is still
  // rebalanced by the items after its first.  Config 4: div 1/2/3/4/6 ->
  // 677/620/622/628/640 us (each item pays ~1.5 us of merge and refill).
  int div = 2;
  if (const char* e = std::getenv("TFB_FD_CHUNKDIV")) div = std::max(1, std::atoi(e));
  const size_t ng = size_t(nlocal) * G;
  pl.gS.assign(ng, 0);
  std::vector<size_t> pos(ng, 0);
  size_t rem = ng * len;
  size_t gi = 0;
  while (rem > 0) {
    if (pos[gi] < len) {
      size_t sz = (rem + size_t(div) * grid - 1) / (size_t(div) * grid);
      sz = std::max(min_keys, (sz + 63) / 64 * 64);
      sz = std::min(sz, len - pos[gi]);
      const unsigned lr = unsigned(gi / G), g = unsigned(gi % G);
      pl.items.push_back(make_uint4((lr << 24) | g, unsigned(pl.gS[gi]++), unsigned(pos[gi]), unsigned(pos[gi] + sz)));
      pos[gi] += sz;
      rem -= sz;
      if (group_major && pos[gi] < len) continue;
    }
    gi = (gi + 1) % ng;
  }
  for (int v : pl.gS) pl.S_max = std::max(pl.S_max, v);
  return pl;
}

// Which tensor-core kernel runs a fast-path shape (tools/fd_ab.py, one
// process, profiles/r2_fd_ab.log).  The TMA-fed stream kernel balances the
// work dynamically and wins on many long KV streams (config 4 at W = 1:
// 256 groups x 32K keys, 632 vs 643 us); everywhere else the register-
// streaming kernel's static splits over two CTAs per SM are faster (config
// 3: 100 vs 112 us; per-rank W = 8 shapes: 33 vs 38 us and 100 vs 118 us),
// because the stream kernel's fold tail costs ~5 us per sub-item round.
// Shape-only, so every schedule and rank of a problem runs the same kernel
// (bitwise-equal partials).  TFB_FD_STREAM=1/0 forces it (TFB_FD_LEGACY=1
// is the old spelling of 0).
static bool fd_stream_ok(const tf_fd_shape& s, World* w, const void* const* q, const void* const* k,
                         const void* const* v) {
  if (std::getenv("TFB_FD_LEGACY")) return false;
  if (!fast_ok(s)) return false;
  const char* force = std::getenv("TFB_FD_STREAM");
  if (force && std::atoi(force) == 0) return false;
  if (!force && (long(s.batch) * s.kv_heads < 64 ||
                 double(s.batch) * s.kv_heads * double(s.kv_len / size_t(w->W)) < 4.0 * 1024 * 1024))
    return false;
  const size_t len = s.kv_len / size_t(w->W);
  if (size_t(s.batch) * s.kv_heads * len >= (size_t(1) << 31)) return false;
  for (int r = 0; r < w->W; ++r)
    if (w->ranks[r].local &&
        ((reinterpret_cast<uintptr_t>(q[r]) | reinterpret_cast<uintptr_t>(k[r]) | reinterpret_cast<uintptr_t>(v[r])) & 15))
      return false;  // TMA needs 16-byte aligned bases
  return true;
}

static tf_status fd_validate(World* w, const tf_fd_shape* s, const void* const* q,
                             const void* const* k, const void* const* v, void* const* out) {
  if (!s || !q || !k || !v || !out) return set_error(TF_ERR_CONFIG, "tf_flash_decode: NULL argument");
  if (s->q_heads < 1 || s->head_dim < 1 || s->kv_len < 1 || s->batch < 1 || s->kv_heads < 1)
    return set_error(TF_ERR_CONFIG, "flash_decode: heads, head_dim, kv_len must be >= 1");
  if (s->kv_len % size_t(w->W) != 0)
    return set_error(TF_ERR_CONFIG, "flash_decode: kv_len = " + std::to_string(s->kv_len) +
                                        " must be divisible by world_size = " +
                                        std::to_string(w->W));
  if (!std::isfinite(s->scale)) return set_error(TF_ERR_CONFIG, "flash_decode: scale must be finite");
  if (s->q_heads % s->kv_heads != 0)
    return set_error(TF_ERR_CONFIG, "flash_decode: q_heads must be a multiple of kv_heads");
  if (s->head_dim > 256 || s->q_heads / s->kv_heads > 32)
    return set_error(TF_ERR_SHAPE, "flash_decode: head_dim <= 256 and q_heads/kv_heads <= 32");
  for (int r = 0; r < w->W; ++r)
    if (w->ranks[r].local && (!q[r] || !k[r] || !v[r] || !out[r]))
      return set_error(TF_ERR_CONFIG, "flash_decode: NULL tensor for rank " + std::to_string(r));
  return TF_OK;
}

void fd_preload() {  // see ag_exact_preload
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, fd_attention_kernel<0>);
  cudaFuncGetAttributes(&a, fd_attention_kernel<1>);
  cudaFuncGetAttributes(&a, fd_attention_kernel<2>);
  cudaFuncGetAttributes(&a, fd_attention_kernel<3>);
  cudaFuncGetAttributes(&a, fd_attention_kernel<4>);
  cudaFuncGetAttributes(&a, fd_stream_kernel<false>);
  cudaFuncGetAttributes(&a, fd_stream_kernel<true>);
  cudaFuncGetAttributes(&a, fd_push_kernel);
  cudaFuncGetAttributes(&a, fd_gather_kernel);
  cudaFuncGetAttributes(&a, fd_fold_kernel);
}

}  // namespace tfb

using namespace tfb;

// Every Flash Decode entry point.  rows_out != NULL: the attention stage
// only (the BSP schedule's first kernel), each local rank's partial wire
// rows [B][Hq][d+2] landing in rows_out[r] instead of the heap.
static tf_status fd_async(tf_world* tw, tf_fd_variant variant, const tf_fd_shape* shape, const void* const* q,
                          const void* const* k_shard, const void* const* v_shard, void* const* out,
                          void* const* inbox_opt, void* const* streams, void* const* rows_out,
                          const tf_fd_paged* paged = nullptr, const void* const* tables = nullptr) {
  if (!tw) return set_error(TF_ERR_CONFIG, "tf_flash_decode: NULL world");
  World* w = &tw->impl;
  TFB_CHECK(fd_validate(w, shape, q, k_shard, v_shard, rows_out ? rows_out : out));
  int page_shift = 0;
  if (paged) {
    const size_t len_r = shape->kv_len / size_t(w->W);
    const int ps = paged->page_size;
    if (ps < 1 || ps > (1 << 20) || (ps & (ps - 1)))
      return set_error(TF_ERR_CONFIG, "flash_decode_paged: page_size must be a power of two in [1, 2^20]");
    while ((1 << page_shift) < ps) ++page_shift;
    if (paged->layout != TF_PAGED_NHD && paged->layout != TF_PAGED_HND)
      return set_error(TF_ERR_CONFIG, "flash_decode_paged: layout must be TF_PAGED_NHD or TF_PAGED_HND");
    if (paged->num_pages < 1)
      return set_error(TF_ERR_CONFIG, "flash_decode_paged: num_pages must be >= 1");
    if (size_t(paged->pages_per_seq) * size_t(ps) < len_r)
      return set_error(TF_ERR_SHAPE, "flash_decode_paged: pages_per_seq * page_size = " +
                                         std::to_string(size_t(paged->pages_per_seq) * size_t(ps)) +
                                         " < kv_len / world_size = " + std::to_string(len_r));
    if (!tables) return set_error(TF_ERR_CONFIG, "flash_decode_paged: NULL block tables");
    for (int r = 0; r < w->W; ++r)
      if (w->ranks[r].local && !tables[r])
        return set_error(TF_ERR_CONFIG, "flash_decode_paged: NULL block table for rank " + std::to_string(r));
  }
  if (variant < TF_FD_BSP || variant > TF_FD_FUSED_OWNER)
    return set_error(TF_ERR_CONFIG, "run_fd: unknown variant");
  const tf_fd_shape& sh = *shape;
  auto st = resolve_streams(w, streams);
  const bool fused_v = variant == TF_FD_FUSED || variant == TF_FD_FUSED_BY_ARRIVAL || variant == TF_FD_FUSED_OWNER;
  // The fused schedules keep their epochs on the device (FdParams::depoch):
  // one self-contained launch per device, capturable into a CUDA graph in
  // any world.  The multi-kernel schedules' epochs are host state.
  const bool dev_epochs = fused_v && !rows_out && !w->events;
  if (!dev_epochs) TFB_CHECK(refuse_multi_rank_capture(w, st, "tf_flash_decode"));
  TFB_CHECK(order_after_legacy(w, streams));
  const int W = w->W, d = sh.head_dim, G = sh.batch * sh.kv_heads, gs = sh.q_heads / sh.kv_heads;
  const size_t len = sh.kv_len / W;
  const size_t row_floats = size_t(sh.batch) * sh.q_heads * (d + 2);
  const bool fast = fast_ok(sh);
  // TMA-fed kernel (fd_stream_kernel) with a guided item table, else the
  // register-streaming kernel with S equal splits per group.
  // Paged KV streams through the TMA kernel when a 64-key stage stays in one
  // page (page_size >= 64) and the pool's rows fit int32 coordinates;
  // smaller pages use the register kernel's per-tile lookups.
  const bool paged_stream_ok =
      !paged || (paged->page_size >= int(kStageKeys) &&
                 size_t(paged->num_pages) * size_t(paged->page_size) * size_t(sh.kv_heads) < (size_t(1) << 31) &&
                 !std::getenv("TFB_FD_PAGED_REGISTER"));
  const bool stream = paged_stream_ok && fd_stream_ok(sh, w, q, k_shard, v_shard);
  // The plan is a function of (G, len, grid, knobs): built and uploaded
  // once per geometry; later calls only need its size and split count.
  FdPlan plan;
  size_t plan_items = 0;
  std::string plan_key;
  if (stream) {
    plan_key = std::to_string(G) + "x" + std::to_string(len) + "@" + std::to_string(w->sm_count);
    for (const char* k : {"TFB_FD_MINKEYS", "TFB_FD_CHUNKDIV", "TFB_FD_GROUP_MAJOR"})
      if (const char* e = std::getenv(k)) plan_key += std::string(",") + k + "=" + e;
    uint64_t& n = w->epochs["fd.plan.items:" + plan_key];
    uint64_t& smax = w->epochs["fd.plan.smax:" + plan_key];
    if (!n) {
      plan = fd_plan(G, len, unsigned(w->sm_count));
      n = plan.items.size();
      smax = uint64_t(plan.S_max);
    }
    plan_items = size_t(n);
    plan.S_max = int(smax);
  }
  const int S = stream ? plan.S_max : choose_splits(sh, len, w->sm_count);
  const size_t split_len = (len + S - 1) / S;
  const int S_eff = stream ? plan.S_max : int((len + split_len - 1) / split_len);

  // Boards: per (src, group) for fused, per src otherwise (fd.flags is
  // W x 1 in the reference, flash_decode.hpp:357).
  const bool fused = variant == TF_FD_FUSED || variant == TF_FD_FUSED_BY_ARRIVAL || variant == TF_FD_FUSED_OWNER;
  const bool owner = variant == TF_FD_FUSED_OWNER && W > 1;
  if (fused) {
    // The fused schedule runs every co-located rank in ONE persistent grid
    // (its waits need every local producer resident): at most kMaxLocal
    // ranks per device fit in a launch's parameters.
    std::map<int, int> per_dev;
    for (int r = 0; r < W; ++r)
      if (w->ranks[r].local && ++per_dev[w->ranks[r].device] > kMaxLocal)
        return set_error(TF_ERR_CONFIG, "run_fused: at most " + std::to_string(kMaxLocal) +
                                            " ranks may share a device (loopback world)");
  }
  BoardEntry fb;
  // Only schedules that signal advance the board's epoch: every rank (every
  // process, in an IPC world) must agree on "run e waits for >= e".
  if (variant == TF_FD_BSP) {
    TFB_CHECK(board_get(w, "fd.flags[" + std::to_string(W) + "x1]", W, 1, &fb));
    fb.epoch = w->boards["fd.flags[" + std::to_string(W) + "x1]"].epoch;
  } else if (owner) {
    // Owner-combine keeps its own boards and inbox: only the owner's cells
    // advance, so sharing them with the all-gather schedules would leave
    // their epochs behind.
    TFB_CHECK(board_next_epoch(w, "fd.flags.owner", W, G, &fb));
  } else {
    TFB_CHECK(board_next_epoch(w, "fd.flags", W, fused ? G : 1, &fb));
    w->fd_flags = FlagSnapshot{w->board_names[fb.id], size_t(W) * (fused ? G : 1), fb.epoch};
  }
  BoardEntry ob{};
  size_t outbox_off = 0;
  const size_t out_floats = size_t(sh.batch) * sh.q_heads * d;
  if (owner) {
    TFB_CHECK(board_next_epoch(w, "fd.oflags", 1, G, &ob));
    TFB_CHECK(heap_get(w, "fd.outbox[" + std::to_string(out_floats) + "]", sizeof(float) * out_floats * 2,
                       &outbox_off));
  }
  // Inbox / pubs / stage in the symmetric heap.  The internal inbox is
  // double-buffered by epoch parity: a fast peer's next push can never land
  // in the buffer a slow rank is still folding.
  size_t inbox_off = 0, pub_off = 0, ws_off = 0, tick_off = 0, ctr_off = 0;
  const std::string geo = "[" + std::to_string(row_floats) + "]";
  // The fused schedules own their inboxes (device-epoch parity); the others
  // share one (host-counted parity).
  TFB_CHECK(heap_get(w, (owner ? "fd.inbox.owner" : fused ? "fd.inbox.fused" : "fd.inbox") + geo,
                     sizeof(float) * W * row_floats * 2, &inbox_off));
  size_t depoch_off = 0;
  if (dev_epochs) {
    TFB_CHECK(heap_get(w, "fd.depoch", sizeof(uint64_t) * 4, &depoch_off));
    if (!owner) {
      w->fd_flags.dev = true;
      w->fd_flags.dev_off = depoch_off;
      w->fd_flags.dev_idx = 0;
    }
  }
  TFB_CHECK(heap_get(w, "fd.partials" + geo, sizeof(float) * row_floats, &pub_off));
  const int nlocal_max = std::min(w->n_local, kMaxLocal);
  const size_t ws_floats = size_t(nlocal_max) * G * S_eff * gs * ws_row(d);
  TFB_CHECK(heap_get(w, "fd.ws[" + std::to_string(ws_floats) + "]", sizeof(float) * ws_floats, &ws_off));
  // Split-fold granularity: hc heads per sub-item, a power of two dividing
  // gs, as many as keep a warp's share at <= kFoldRB rows (one load batch).
  int hc = 1;
  while (hc * 2 <= 32 && gs % (hc * 2) == 0 && S_eff * hc * 2 <= 8 * kFoldRB) hc *= 2;
  TFB_CHECK(heap_get(w, "fd.tickets[" + std::to_string(G) + "x" + std::to_string(S_eff) + "]",
                     sizeof(unsigned long long) * (nlocal_max * G * 3 + kMaxLocal), &tick_off));  // done | gtick | claims | sfc
  TFB_CHECK(heap_get(w, "fd.ctr", 64, &ctr_off));
  // Stream kernel tables: the item plan (uploaded once per geometry, before
  // any launch uses it) and the per-(rank, group) fold claims.
  size_t items_off = 0, fstate_off = 0;
  if (stream) {
    const size_t tbytes = plan_items * sizeof(uint4) + size_t(G) * sizeof(int);
    TFB_CHECK(heap_get(w, "fd.items[" + plan_key + "]", tbytes, &items_off));
    TFB_CHECK(heap_get(w, "fd.fstate[" + std::to_string(G) + "]", sizeof(unsigned) * kMaxLocal * G, &fstate_off));
    uint64_t& up = w->epochs["fd.items.uploaded@" + std::to_string(items_off)];
    if (!up) {
      if (plan.items.empty()) plan = fd_plan(G, len, unsigned(w->sm_count));  // heap was reset
      std::vector<uint8_t> host(tbytes);
      std::memcpy(host.data(), plan.items.data(), plan.items.size() * sizeof(uint4));
      std::memcpy(host.data() + plan.items.size() * sizeof(uint4), plan.gS.data(), size_t(G) * sizeof(int));
      for (int r = 0; r < W; ++r) {
        if (!w->ranks[r].local) continue;
        TFB_CUDA(cudaSetDevice(w->ranks[r].device));
        TFB_CUDA(cudaMemcpy(w->ptr(r, items_off), host.data(), tbytes, cudaMemcpyHostToDevice));
      }
      up = 1;
    }
  }
  // Tickets are epoch-valued per (group, split-count) geometry.
  const uint64_t tepoch = ++w->epochs["fd.tickets@" + std::to_string(tick_off)];
  // Inbox parity: one counter per inbox shared by every schedule that
  // writes it (the fused and the per-source boards have separate epochs, so
  // keying the parity on either let a fused run and a following
  // fine-waits run land in the same buffer).  Every rank issues the same
  // call sequence, so every rank agrees on it; consecutive pushing runs
  // alternate buffers, and a peer is at most one run ahead.
  int parity = 0;
  if (variant != TF_FD_BSP && !dev_epochs)
    parity = int(++w->epochs[std::string(owner ? "fd.inbox.owner" : "fd.inbox") + "@" + std::to_string(inbox_off)] & 1);

  auto inbox_of = [&](int r) -> float* {
    if (inbox_opt && inbox_opt[r]) return static_cast<float*>(inbox_opt[r]);
    return reinterpret_cast<float*>(w->ptr(r, inbox_off)) + size_t(parity) * W * row_floats;
  };
  // Device-epoch launches add the parity themselves (a caller's inbox is a
  // single buffer: no parity).
  const bool caller_inbox = inbox_opt != nullptr;

  FdParams P{};
  P.W = W;
  P.B = sh.batch;
  P.Hq = sh.q_heads;
  P.Hkv = sh.kv_heads;
  P.gs = gs;
  if (paged) {
    P.paged = 1;
    P.page_shift = page_shift;
    P.pps = paged->pages_per_seq;
    P.num_pages = paged->num_pages;
    P.hnd = paged->layout == TF_PAGED_HND;
  }
  P.d = d;
  P.len = len;
  P.S = S_eff;
  P.split_len = split_len;
  P.scale = sh.scale;
  P.kv_bf16 = sh.kv_dtype == TF_BF16;
  P.out_bf16 = sh.out_dtype == TF_BF16;
  P.watchdog_ns = w->watchdog_ns;
  P.err = nullptr;  // set per launch (per device)
  P.board = fb.id;
  for (int r = 0; r < W; ++r) {
    P.inbox_all[r] = inbox_of(r);
    P.flags_all[r] = reinterpret_cast<uint64_t*>(w->ptr(r, fb.offset));
  }

  // Group local ranks by device: one attention launch per device.
  std::map<int, std::vector<int>> by_dev;
  for (int r = 0; r < W; ++r)
    if (w->ranks[r].local) by_dev[w->ranks[r].device].push_back(r);

  P.epoch = tepoch;
  P.flag_epoch = fb.epoch;
  if (w->events && fused && !owner && W > 1) {
    // Event log (debug, untimed): ~0-filled synchronously before any launch.
    size_t ev_off = 0;
    const size_t bytes = size_t(W) * G * 2 * sizeof(unsigned long long);
    TFB_CHECK(heap_get(w, "fd.events[" + std::to_string(W) + "x" + std::to_string(G) + "]", bytes, &ev_off));
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      cudaSetDevice(w->ranks[r].device);
      TFB_CUDA(cudaDeviceSynchronize());
      TFB_CUDA(cudaMemset(w->ptr(r, ev_off), 0xFF, bytes));
      TFB_CUDA(cudaDeviceSynchronize());
    }
    for (int r = 0; r < W; ++r) P.events_all[r] = reinterpret_cast<unsigned long long*>(w->ptr(r, ev_off));
    w->fd_events_off = ev_off;
    w->fd_events_n = size_t(W) * G * 2;
  }
  if (owner) {
    P.oflag_epoch = ob.epoch;
    for (int r = 0; r < W; ++r) {
      P.outbox_all[r] = reinterpret_cast<float*>(w->ptr(r, outbox_off)) + (dev_epochs ? 0 : size_t(ob.epoch & 1) * out_floats);
      P.oflags_all[r] = reinterpret_cast<uint64_t*>(w->ptr(r, ob.offset));
    }
  }
  // One attention launch per device (a loopback device runs all its ranks
  // in one persistent grid, so the fused waits can never starve a producer).
  // The fused schedule shares one launch per device (its waits need every
  // local producer resident); the others never wait inside the attention
  // kernel, so each rank gets its own launch on its own stream, as in the
  // reference (a straggling rank then delays only its own stage).
  auto launch_attention = [&](int push, int fold_inline) -> tf_status {
    const size_t per_launch = fold_inline ? size_t(kMaxLocal) : 1;
    for (auto& kv : by_dev) {
      const std::vector<int>& rs = kv.second;
      for (size_t c0 = 0; c0 < rs.size(); c0 += per_launch) {
        FdParams Q = P;
        Q.nlocal = int(std::min(rs.size() - c0, per_launch));
        const int lead = rs[c0];
        for (int i = 0; i < Q.nlocal; ++i) {
          const int r = rs[c0 + i];
          Q.r[i] = FdRank{q[r], k_shard[r], v_shard[r], out ? out[r] : nullptr,
                          rows_out ? static_cast<float*>(rows_out[r]) : reinterpret_cast<float*>(w->ptr(r, pub_off)),
                          inbox_of(r),
                          reinterpret_cast<uint64_t*>(w->ptr(r, fb.offset)), r, w->skew_of(r),
                          paged ? static_cast<const int*>(tables[r]) : nullptr};
        }
        Q.err = w->err_of(lead);
        Q.ws = reinterpret_cast<float*>(w->ptr(lead, ws_off));
        if (dev_epochs && fold_inline) {
          Q.depoch = reinterpret_cast<uint64_t*>(w->ptr(lead, depoch_off));
          Q.inbox_pstride = caller_inbox ? 0 : size_t(W) * row_floats;
          Q.outbox_pstride = out_floats;
        }
        if (std::getenv("TFB_TRACE")) {
          size_t toff;
          TFB_CHECK(heap_get(w, "fd.trace", sizeof(unsigned long long) * kTraceSlots * 4096, &toff));
          Q.trace = reinterpret_cast<unsigned long long*>(w->ptr(lead, toff));
        }
        Q.done = reinterpret_cast<uint64_t*>(w->ptr(lead, tick_off));
        Q.gtick = Q.done + size_t(nlocal_max) * G;
        Q.claim = reinterpret_cast<unsigned long long*>(Q.gtick + size_t(nlocal_max) * G);
        Q.sfc = reinterpret_cast<unsigned int*>(Q.claim + size_t(nlocal_max) * G);
        Q.hc = hc;
        Q.interleave = !std::getenv("TFB_FD_CONTIGUOUS");
        Q.local_dst = 0;
        for (int r = 0; r < W; ++r)
          if (w->ranks[r].local && w->ranks[r].device == kv.first) Q.local_dst |= 1ull << r;
        Q.ctr = reinterpret_cast<unsigned int*>(w->ptr(lead, ctr_off));
        Q.push = push;
        Q.fold_inline = fold_inline;
        Q.direct = fold_inline && W == 1;
        Q.by_arrival = variant == TF_FD_FUSED_BY_ARRIVAL;
        Q.owner = owner;
        if (stream) {
          Q.items = reinterpret_cast<const uint4*>(w->ptr(lead, items_off));
          Q.gS = reinterpret_cast<const int*>(Q.items + plan_items);
          Q.nitems = unsigned(plan_items) * unsigned(Q.nlocal);
        }
        cudaSetDevice(kv.first);
        // Every co-located rank's inputs may come from its own stream: the
        // shared launch on st[lead] is ordered after all of them.
        for (int i = 1; i < Q.nlocal; ++i) {
          const int r = rs[c0 + i];
          if (st[r] == st[lead]) continue;
          cudaEvent_t ev;
          TFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
          TFB_CUDA(cudaEventRecord(ev, st[r]));
          TFB_CUDA(cudaStreamWaitEvent(st[lead], ev, 0));
          cudaEventDestroy(ev);
        }
        // Tensor-core split with bf16 P for bf16 output, hi/lo P when the
        // caller asked for fp32 output; the generic split otherwise.
        // P reaches the PV product as a bf16 hi + lo pair for every output
        // dtype: attention accurate to ~1e-5 whatever the output, so a bf16
        // output's only error is its own rounding (<= 2^-8 of the head's
        // max).  Measured cost < 1 % (HBM-bound).  TFB_FD_HILO=0: one bf16 P.
        const char* hl = std::getenv("TFB_FD_HILO");
        const bool hilo = sh.out_dtype == TF_F32 || !hl || std::atoi(hl) != 0;
        if (stream) {
          FdMaps maps{};
          for (int i = 0; i < Q.nlocal; ++i) {
            const int r = rs[c0 + i];
            if (paged && paged->layout == TF_PAGED_NHD) {
              const size_t krows = size_t(paged->num_pages) * size_t(paged->page_size);
              TFB_CHECK(fd_kv_map_nhd(&maps.k[i], k_shard[r], krows, sh.kv_heads));
              TFB_CHECK(fd_kv_map_nhd(&maps.v[i], v_shard[r], krows, sh.kv_heads));
            } else {
              const size_t rows = paged ? size_t(paged->num_pages) * size_t(paged->page_size) * sh.kv_heads
                                        : size_t(sh.batch) * sh.kv_heads * len;
              TFB_CHECK(fd_kv_map(&maps.k[i], k_shard[r], rows));
              TFB_CHECK(fd_kv_map(&maps.v[i], v_shard[r], rows));
            }
          }
          const void* kfn = hilo ? reinterpret_cast<const void*>(fd_stream_kernel<true>)
                                 : reinterpret_cast<const void*>(fd_stream_kernel<false>);
          const size_t smem = sizeof(StreamSmem) + 1024;
          static std::atomic<bool> attr[2][64];
          if (!attr[hilo][kv.first & 63].load()) {
            TFB_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr[hilo][kv.first & 63].store(true);
          }
          const unsigned grid = std::max(1u, std::min(Q.nitems, unsigned(w->sm_count)));
          Q.fold_once = Q.nlocal == 1 && Q.nitems >= grid && unsigned(G) * unsigned(Q.gs / Q.hc) <= grid &&
                        !std::getenv("TFB_FD_REFOLD");
          cudaLaunchConfig_t lc{};
          cudaLaunchAttribute la[1];
          lc.gridDim = dim3(grid);
          lc.blockDim = dim3(kStreamThreads);
          lc.dynamicSmemBytes = smem;
          lc.stream = st[lead];
          lc.attrs = la;
          lc.numAttrs = unsigned(pdl_attrs(la));
          if (hilo) TFB_CUDA(cudaLaunchKernelEx(&lc, fd_stream_kernel<true>, Q, maps));
          else TFB_CUDA(cudaLaunchKernelEx(&lc, fd_stream_kernel<false>, Q, maps));
          TFB_CUDA(cudaGetLastError());
          ++w->launches;
          for (int i = 1; i < Q.nlocal; ++i) {
            const int r = rs[c0 + i];
            if (st[r] == st[lead]) continue;
            cudaEvent_t ev;
            TFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            TFB_CUDA(cudaEventRecord(ev, st[lead]));
            TFB_CUDA(cudaStreamWaitEvent(st[r], ev, 0));
            cudaEventDestroy(ev);
          }
          continue;
        }
        const unsigned items = unsigned(Q.nlocal) * G * S_eff;
        const int mode = !fast ? 0 : (hilo ? 2 : 1) + (paged ? 2 : 0);
        const void* kfn = mode == 0 ? reinterpret_cast<const void*>(fd_attention_kernel<0>)
                        : mode == 1 ? reinterpret_cast<const void*>(fd_attention_kernel<1>)
                        : mode == 2 ? reinterpret_cast<const void*>(fd_attention_kernel<2>)
                        : mode == 3 ? reinterpret_cast<const void*>(fd_attention_kernel<3>)
                                    : reinterpret_cast<const void*>(fd_attention_kernel<4>);
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kFastThreads, 0);
        const unsigned grid =
            std::max(1u, std::min(items, unsigned(std::max(per_sm, 1) * w->sm_count)));
        // Every CTA computes an item (items >= grid), so every CTA enters the
        // split fold and the first claims cover all nsub sub-items.
        Q.fold_once = Q.nlocal == 1 && items >= grid && unsigned(G) * unsigned(Q.gs / Q.hc) <= grid &&
                      !std::getenv("TFB_FD_REFOLD");
        cudaLaunchConfig_t lc{};
        cudaLaunchAttribute la[1];
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(kFastThreads);
        lc.stream = st[lead];
        lc.attrs = la;
        lc.numAttrs = unsigned(pdl_attrs(la));
        if (mode == 0) TFB_CUDA(cudaLaunchKernelEx(&lc, fd_attention_kernel<0>, Q));
        else if (mode == 1) TFB_CUDA(cudaLaunchKernelEx(&lc, fd_attention_kernel<1>, Q));
        else if (mode == 2) TFB_CUDA(cudaLaunchKernelEx(&lc, fd_attention_kernel<2>, Q));
        else if (mode == 3) TFB_CUDA(cudaLaunchKernelEx(&lc, fd_attention_kernel<3>, Q));
        else TFB_CUDA(cudaLaunchKernelEx(&lc, fd_attention_kernel<4>, Q));
        TFB_CUDA(cudaGetLastError());
        ++w->launches;
        // Ranks sharing the launch are complete when it is: order their streams.
        for (int i = 1; i < Q.nlocal; ++i) {
          const int r = rs[c0 + i];
          if (st[r] == st[lead]) continue;
          cudaEvent_t ev;
          TFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
          TFB_CUDA(cudaEventRecord(ev, st[lead]));
          TFB_CUDA(cudaStreamWaitEvent(st[r], ev, 0));
          cudaEventDestroy(ev);
        }
      }
    }
    return TF_OK;
  };

  if (rows_out) return launch_attention(0, 0);  // attention stage only: rows to the caller
  // Every schedule lands W wire rows per rank in an inbox / stage
  // (flash_decode_test.cpp:167-196: W*W*wire*4 bytes world-wide).
  for (int r = 0; r < W; ++r)
    if (w->ranks[r].local) {
      // Owner-combine lands the partial rows of the groups this rank owns
      // (W sources x 1/W of the rows) plus the finished rows of the others.
      if (owner) w->stage(r, sizeof(float) * (row_floats + (W - 1) * out_floats / W));
      else w->stage(r, sizeof(float) * W * row_floats);
    }
  if (fused) return launch_attention(/*push=*/1, /*fold_inline=*/1);
  // Everything the later stages allocate exists before the first launch.
  TFB_CHECK(ensure_barrier(w));
  size_t stage_off = 0;
  if (variant == TF_FD_BSP)
    TFB_CHECK(heap_get(w, "fd.stage" + geo, sizeof(float) * W * row_floats, &stage_off));
  TFB_CHECK(launch_attention(0, 0));
  TFB_CHECK(world_barrier(w, st));
  FdParams PP = P;
  auto with_err = [&](int r) {
    FdParams x = PP;
    x.err = w->err_of(r);
    return x;
  };
  if (variant == TF_FD_BSP) {
    FdParams G2 = PP;
    for (int r = 0; r < W; ++r) G2.inbox_all[r] = reinterpret_cast<float*>(w->ptr(r, pub_off));
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      cudaSetDevice(w->ranks[r].device);
      float* stage = (inbox_opt && inbox_opt[r]) ? static_cast<float*>(inbox_opt[r])
                                                 : reinterpret_cast<float*>(w->ptr(r, stage_off));
      const unsigned blocks = unsigned(std::min<size_t>((W * row_floats + 255) / 256, 1024));
      fd_gather_kernel<<<blocks, 256, 0, st[r]>>>(stage, row_floats, G2, W);
      TFB_CUDA(cudaGetLastError());
      ++w->launches;
    }
    TFB_CHECK(world_barrier(w, st));
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      cudaSetDevice(w->ranks[r].device);
      float* stage = (inbox_opt && inbox_opt[r]) ? static_cast<float*>(inbox_opt[r])
                                                 : reinterpret_cast<float*>(w->ptr(r, stage_off));
      fd_fold_kernel<<<sh.batch * sh.q_heads, 32, 0, st[r]>>>(stage, out[r], with_err(r), r, nullptr, 0);
      TFB_CUDA(cudaGetLastError());
      ++w->launches;
    }
    return TF_OK;
  }
  // independent_ag / fine_waits: push kernel per rank.
  const int wait_all = variant == TF_FD_INDEPENDENT_AG;
  for (int r = 0; r < W; ++r) {
    if (!w->ranks[r].local) continue;
    cudaSetDevice(w->ranks[r].device);
    FdParams Q = with_err(r);
    Q.r[0].flags = reinterpret_cast<uint64_t*>(w->ptr(r, fb.offset));
    fd_push_kernel<<<W, 256, 0, st[r]>>>(reinterpret_cast<float*>(w->ptr(r, pub_off)), row_floats,
                                         r, W, Q, wait_all);
    TFB_CUDA(cudaGetLastError());
    ++w->launches;
  }
  if (wait_all) TFB_CHECK(world_barrier(w, st));
  for (int r = 0; r < W; ++r) {
    if (!w->ranks[r].local) continue;
    cudaSetDevice(w->ranks[r].device);
    fd_fold_kernel<<<sh.batch * sh.q_heads, 32, 0, st[r]>>>(
        inbox_of(r), out[r], with_err(r), r, reinterpret_cast<uint64_t*>(w->ptr(r, fb.offset)),
        wait_all ? 0 : 1);
    TFB_CUDA(cudaGetLastError());
    ++w->launches;
  }
  return TF_OK;
}

extern "C" tf_status tf_flash_decode_async(tf_world* tw, tf_fd_variant variant,
                                           const tf_fd_shape* shape, const void* const* q,
                                           const void* const* k_shard,
                                           const void* const* v_shard, void* const* out,
                                           void* const* inbox_opt, void* const* streams) {
  return fd_async(tw, variant, shape, q, k_shard, v_shard, out, inbox_opt, streams, nullptr);
}

// Paged KV cache (an extension beyond the reference API: its SPEC lists
// paged KV as a non-goal).  Same schedules, wire format and
// fold as tf_flash_decode; the K/V of each rank are page pools addressed
// through per-rank block tables.
extern "C" tf_status tf_flash_decode_paged_async(tf_world* tw, tf_fd_variant variant, const tf_fd_shape* shape,
                                                 const tf_fd_paged* paged, const void* const* q,
                                                 const void* const* k_pool, const void* const* v_pool,
                                                 const void* const* block_tables, void* const* out,
                                                 void* const* inbox_opt, void* const* streams) {
  if (!paged) return set_error(TF_ERR_CONFIG, "flash_decode_paged: NULL paged layout");
  return fd_async(tw, variant, shape, q, k_pool, v_pool, out, inbox_opt, streams, nullptr, paged, block_tables);
}

extern "C" tf_status tf_flash_decode_paged(tf_world* tw, tf_fd_variant variant, const tf_fd_shape* shape,
                                           const tf_fd_paged* paged, const void* const* q, const void* const* k_pool,
                                           const void* const* v_pool, const void* const* block_tables,
                                           void* const* out, void* const* inbox_opt, void* const* streams) {
  TFB_CHECK(tf_flash_decode_paged_async(tw, variant, shape, paged, q, k_pool, v_pool, block_tables, out, inbox_opt,
                                        streams));
  return sync_and_check(&tw->impl, resolve_streams(&tw->impl, streams));
}

// attention_partial + serialize_partial of every (b, q-head) for each local
// rank (tilemath.hpp:145-181, 244-258; flash_decode.hpp:162-167): the
// rank's wire rows [B][Hq][d+2] fp32 into rows[r] -- the BSP schedule's
// attention kernel alone, so callers can exchange the rows with their own
// collective (NCCL all-gather) and fold them with tf_fd_combine_async.
extern "C" tf_status tf_fd_partial_async(tf_world* tw, const tf_fd_shape* shape, const void* const* q,
                                         const void* const* k_shard, const void* const* v_shard,
                                         void* const* rows, void* const* streams) {
  if (!rows) return set_error(TF_ERR_CONFIG, "tf_fd_partial: NULL rows");
  return fd_async(tw, TF_FD_BSP, shape, q, k_shard, v_shard, nullptr, nullptr, streams, rows);
}

// fold_rows + finalize (flash_decode.hpp:171-180, tilemath.hpp:186-239):
// rows[r] holds W sources' wire rows [W][B][Hq][d+2] (an all-gather of
// every rank's tf_fd_partial_async rows), folded in ascending source order
// into out[r] -- the BSP schedule's fold kernel, bitwise every schedule's
// output.
extern "C" tf_status tf_fd_combine_async(tf_world* tw, const tf_fd_shape* shape, const void* const* rows,
                                         void* const* out, void* const* streams) {
  if (!tw || !shape || !rows || !out) return set_error(TF_ERR_CONFIG, "tf_fd_combine: NULL argument");
  World* w = &tw->impl;
  const tf_fd_shape& sh = *shape;
  if (sh.head_dim < 1 || sh.head_dim > 256 || sh.batch < 1 || sh.q_heads < 1)
    return set_error(TF_ERR_CONFIG, "fd_combine: bad shape");
  auto st = resolve_streams(w, streams);
  TFB_CHECK(refuse_multi_rank_capture(w, st, "tf_fd_combine"));
  TFB_CHECK(order_after_legacy(w, streams));
  FdParams P{};
  P.W = w->W;
  P.B = sh.batch;
  P.Hq = sh.q_heads;
  P.Hkv = sh.kv_heads;
  P.gs = sh.kv_heads > 0 ? sh.q_heads / sh.kv_heads : 1;
  P.d = sh.head_dim;
  P.out_bf16 = sh.out_dtype == TF_BF16;
  P.watchdog_ns = w->watchdog_ns;
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local) continue;
    if (!rows[r] || !out[r]) return set_error(TF_ERR_CONFIG, "fd_combine: NULL buffer for rank " + std::to_string(r));
    cudaSetDevice(w->ranks[r].device);
    P.err = w->err_of(r);
    fd_fold_kernel<<<sh.batch * sh.q_heads, 32, 0, st[r]>>>(static_cast<const float*>(rows[r]), out[r], P, r,
                                                              nullptr, 0);
    TFB_CUDA(cudaGetLastError());
    ++w->launches;
  }
  return TF_OK;
}

extern "C" tf_status tf_flash_decode(tf_world* tw, tf_fd_variant variant,
                                     const tf_fd_shape* shape, const void* const* q,
                                     const void* const* k_shard, const void* const* v_shard,
                                     void* const* out, void* const* inbox_opt,
                                     void* const* streams) {
  TFB_CHECK(tf_flash_decode_async(tw, variant, shape, q, k_shard, v_shard, out, inbox_opt, streams));
  return sync_and_check(&tw->impl, resolve_streams(&tw->impl, streams));
}

extern "C" tf_status tf_fd_flag_counts(tf_world* tw, int rank, uint64_t* out, size_t cap,
                                       size_t* count) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  const FlagSnapshot& f = w->fd_flags;
  if (count) *count = f.cells ? size_t(w->W) : 0;
  if (f.cells == 0 || !out) return TF_OK;
  if (rank < 0 || rank >= w->W) return set_error(TF_ERR_BOUNDS, "fd_flag_counts: bad rank");
  auto it = w->boards.find(f.board);
  if (it == w->boards.end()) return TF_OK;
  std::vector<uint64_t> v(f.cells);
  TFB_CUDA(cudaMemcpy(v.data(), w->ptr(rank, it->second.offset), sizeof(uint64_t) * f.cells,
                      cudaMemcpyDefault));
  uint64_t epoch = f.epoch;
  if (f.dev && w->ranks[rank].local) {
    // The epoch the rank's launch left in its device's lead cell.
    int lead = rank;
    for (int r = 0; r < w->W; ++r)
      if (w->ranks[r].local && w->ranks[r].device == w->ranks[rank].device) {
        lead = r;
        break;
      }
    TFB_CUDA(cudaMemcpy(&epoch, reinterpret_cast<uint64_t*>(w->ptr(lead, f.dev_off)) + f.dev_idx, sizeof(uint64_t),
                        cudaMemcpyDefault));
  }
  const size_t per = f.cells / size_t(w->W);
  for (int s = 0; s < w->W && size_t(s) < cap; ++s) {
    uint64_t mn = UINT64_MAX;
    for (size_t g = 0; g < per; ++g) mn = std::min(mn, v[size_t(s) * per + g]);
    out[s] = mn - (epoch - 1);
  }
  return TF_OK;
}

extern "C" tf_status tf_fd_events(tf_world* tw, int rank, uint64_t* out, size_t cap, size_t* count) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  if (rank < 0 || rank >= w->W) return set_error(TF_ERR_BOUNDS, "fd_events: bad rank");
  if (count) *count = w->fd_events_n;
  if (!out || w->fd_events_n == 0) return TF_OK;
  const size_t n = cap < w->fd_events_n ? cap : w->fd_events_n;
  TFB_CUDA(cudaDeviceSynchronize());
  TFB_CUDA(cudaMemcpy(out, w->ptr(rank, w->fd_events_off), n * sizeof(uint64_t), cudaMemcpyDefault));
  return TF_OK;
}
