// ag_sm100.cu -- the bf16 All-Gather+GEMM path on 5th-generation tensor cores.
//
// One persistent, warp-specialised kernel per rank (ag_gemm.hpp:185-305
// re-designed for sm_100a):
//   warp 0      TMA producer.  Streams A (128 x 64 per CTA, SWIZZLE_128B,
//               K-major) and B (64 x 256 per CTA as four 64 x 64 boxes,
//               MN-major -- B is used in the caller's k x n layout, no
//               transpose pass) into a 4-deep smem ring.  A k-block owned by
//               this rank comes straight from its shard; a k-block owned by
//               rank s comes from the local gathered buffer ("inbox", the
//               reference's ag.inbox, m x k) once ready[m_blk][s] reaches
//               this run's epoch (ld.acquire.sys spin, then
//               fence.proxy.async so the TMA sees the generic-proxy bytes).
//               The k loop starts at the rank's own shard, so the first
//               K/W of every tile never waits on the network.
//   warp 1      MMA issuer (one thread): tcgen05.mma.kind::f16, fp32
//               accumulators in TMEM; tcgen05.commit releases smem stages.
//   warps 2-5   epilogue: tcgen05.ld 32x32b -> bf16 -> global C.
//   warps 6-9   gather (PULL): claim (m_blk, src) chunks from a global
//               counter, copy them from the owner's shard over NVLink
//               (128-bit peer loads) into the local inbox at column src*kw,
//               then release ready[m_blk][src].  Each remote A byte crosses
//               NVLink exactly once per rank (the reference re-pulls every
//               A tile once per N tile, ag_gemm_test.cpp:134-143).
//
// Tile shapes (the L2->SM crossbar, ~9.5 TB/s measured, is what a B200 GEMM
// must economise, profiles/r1_*):
//   CG = 2  a CTA pair (cluster of 2, tcgen05.mma.cta_group::2) owns a
//           256 x 512 tile: each CTA stages its 128 rows of A and 256 of the
//           512 B columns per k-block (48 KB), the leader issues two
//           M=256 N=256 K=16 MMAs per k-step (one per 256-column half), and
//           each CTA's whole TMEM (512 columns) holds its 128 x 512
//           accumulator.  5.9 bytes per kFLOP -- cuBLAS's own tile.
//   CG = 1  skinny M (< 256 rows): 128 x 256 tiles, two TMEM accumulators so
//           the epilogue overlaps the next tile.
// PUSH replaces the gather warps with a producer kernel on every rank that
// stores its shard chunks into every peer's inbox and raises the peer's
// ready cell (red.release.sys) -- the same consumer gate.
// BASELINE gathers with copy engines between two world barriers and runs
// the same kernel ungated.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>

#include "ag_internal.hpp"
#include "sm100.cuh"

namespace tfb {
namespace {

using namespace sm100;

constexpr int BM = 128, BK = 64;  // BM: A rows staged per CTA
constexpr int GROUP_M = 16;       // tile-rows per raster group (L2 reuse of B)
constexpr int NUM_THREADS = 320;    // 6 role warps + 4 gather warps
constexpr int GATHER_T = NUM_THREADS - 192;  // gather threads (PULL)
constexpr int TMEM_COLS = 512;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB

template <int CG, int NH_, int BK_ = 64>
struct Cfg {
  static constexpr int NH = NH_;                        // 256-column MMA halves per tile
  static constexpr int BN_TILE = 256 * NH;              // tile width
  static constexpr int ACC_BUFS = NH == 2 ? 1 : 2;      // accumulators in 512 TMEM columns
  static constexpr int BK = BK_;                        // k-block depth (64, or 128 for narrow pair tiles)
  static constexpr int A_BYTES = BM * BK_ * 2;          // 16 / 32 KB: BK / 64 A boxes of 64 columns
  // Narrow pair tiles (32 KB stages) fit six in flight: the skinny main loop is load-latency bound.
  // With 128-deep k-blocks (64 KB stages) three: the same bytes in flight, half the ring rounds.
  static constexpr int STAGES = (CG == 2 && NH_ == 1) ? (BK_ == 128 ? 3 : 6) : 4;
  static constexpr int CPH = 4 / CG;                    // 64-column B chunks per half per CTA
  static constexpr int B_BYTES = NH * CPH * BK * 128;   // 32 KB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES; // 48 KB
  static constexpr uint32_t IDESC = idesc_bf16(BM * CG, 256, /*A K-major*/ 0, /*B MN-major*/ 1);
  static constexpr int EPI_BYTES = 4 * 2 * 4096;         // C staging for TMA stores
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + EPI_BYTES + 1024 + 256;
};

struct AgTcParams {
  int M, N, K, kw, W;
  int own;          // rank whose shard map serves its own k-range; -1: all from inbox
  int num_m, num_n, num_tiles, kb_total, kbw;  // num_m: 128-row blocks; num_n: tile columns
  __nv_bfloat16* C;
  const uint64_t* ready;  // [num_m][W] local board; nullptr: ungated
  uint64_t epoch;
  int gather;             // gather warps active (PULL)
  int gather_own;         // PULL into a caller's gathered buffer: also place the own shard (placement check)
  __nv_bfloat16* inbox;   // local inbox, m x k
  uint64_t* ready_w;      // writable view of `ready` (gather)
  unsigned long long* events;  // event log (tf_world_set_events): [num_m][W] x {store, first load} %globaltimer
  unsigned int* ctr;      // [0] gather chunk counter, [1] done counter
  uint64_t watchdog_ns;
  DevErr* err;
  int board;
  int xchg_lsu;  // split-K L2 exchange: outgoing slices stored by every thread (else one TMA bulk store each)
  int dbg;  // TFB_DEBUG knobs: 1 skip C stores, 2 skip MMAs, 8 force CG=1, 16 skip the split-K reduce,
           // 32 poll-wait the epilogue, 64 skip the epilogue, 256 skip A loads, 512 skip B loads,
           // 4096 print CTA 0's phase stamps (profiling aids)
  int ksplit;  // > 1: skinny-M split-K across a cluster of ksplit CTAs (pairs), reduced through DSMEM
  int full_items;   // items [0, full_items) are whole tiles (x k-splits)
  int q_tail;       // > 1: the tiles after them run as q_tail column slices each (last-wave balance)
  int total_items;
  int ldc;     // row pitch of C (elements)
  int b4;      // whole tiles load B with ONE 4-D box per stage (tmB4) instead of NH * CPH 2-D boxes
  uint8_t* ws;  // split-K exchange through L2: [grid CTAs][NH][128 rows x 1 KB]; nullptr: through DSMEM
  // M-sharded A (TF_SHARD_M): rank s owns m-blocks [s*mpr, (s+1)*mpr) (all
  // of K); k runs ascending and the tile rows rotate by mt_rot so a rank's
  // own rows come first (they never wait on the network).
  int msharded, mpr, mt_rot;
  int l2hint;  // TMA L2 policies: 1 A evict_last, 2 B evict_first (TFB_L2HINT)
  int one_producer;  // TFB_ONE_PRODUCER: warp 0 issues A and B boxes (no B producer warp)
  const __nv_bfloat16* peer_shard[64];
};

__constant__ int g_group_m;  // raster group (tile-rows); GROUP_M unless overridden

// Tile raster: g tile-rows at a time, column-major inside the group, so
// concurrently running CTAs share B panels in L2.
__device__ __forceinline__ void tile_coords(int num_mt, int num_n, int t, int& mt, int& nb) {
  const int gm = g_group_m > 0 ? g_group_m : GROUP_M;
  const int per_group = gm * num_n;
  const int group = t / per_group;
  const int first_m = group * gm;
  const int gsize = min(num_mt - first_m, gm);
  const int r = t % per_group;
  mt = first_m + r % gsize;
  nb = r / gsize;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (a local smem object) in CTA `rank`.
// Explicit shared-window accesses for the split-K dump and sum: through a
// generic pointer (the 1 KB-aligned dynamic smem base loses its state
// space) they compiled to generic LD.E / ST.E.
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// Remote arrive.  Deliberately without .release.cluster: that form fences
// the whole cluster on every call and was measured to halve the pipeline
// rate; the data it orders is written by TMA and tracked by the barrier.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

template <int CG>
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                         int c1, uint64_t pol = 0) {
  if (pol) {  // with an L2 cache policy (createpolicy)
    if (CG == 2)
      asm volatile(
          "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
          "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
          "l"(map), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(pol)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
          "{%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
          "l"(map), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(pol)
          : "memory");
    return;
  }
  if (CG == 2)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
}

// 4-D box: this CTA's whole B slice of a k-block (NH halves x CPH 64-column
// chunks x BK rows, 32 KB) in one instruction.  A TMA box costs the issuing
// CTA a roughly fixed time whatever its size (tools/micro_tma_req.cu: 8 KB
// boxes stream at ~31 GB/s per CTA, 32 KB boxes at ~125), so fewer, larger
// boxes is what raises the L2->SM rate.
template <int CG>
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c1,
                                            int c2, int c3, uint64_t pol = 0) {
  if (pol) {
    if (CG == 2)
      asm volatile(
          "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
          "[%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
          "l"(map), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(bar_cluster), "l"(pol)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
          "{%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
          "l"(map), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(bar_cluster), "l"(pol)
          : "memory");
    return;
  }
  if (CG == 2)
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(bar_cluster)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(bar_cluster)
        : "memory");
}

template <int CG>
__device__ __forceinline__ void mma_issue(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  if (CG == 2)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    mma_bf16_ss(d_tmem, a_desc, b_desc, idesc, accumulate);
}

// tcgen05.commit: arrive on `bar` in every CTA of the pair (cluster ranks in
// pair_mask) once the issued MMAs retired.
template <int CG>
__device__ __forceinline__ void mma_commit_all(uint64_t* bar, uint16_t pair_mask) {
  if (CG == 2)
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;" ::"r"(smem_u32(bar)),
        "h"(pair_mask)
        : "memory");
  else
    mma_commit(bar);
}

template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* slot) {
  if (CG == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  } else {
    tmem_alloc(slot, TMEM_COLS);
  }
}

template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr) {
  if (CG == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(TMEM_COLS)
                 : "memory");
  else
    tmem_dealloc(taddr, TMEM_COLS);
}

// Split-K sum (see the kernel): CTA ks owns rows [ks*rows_per, +rows_per)
// of the tile's 128; sibling s2's partial of them sits in R's slice s2
// (L2 route) or in sibling s2's own R (DSMEM route, cluster rank
// prank + CG * s2).  Task (row, g): 16-byte chunks g and g + 32 of the
// row (columns 4g..4g+3, 128+4g..), so a quarter-warp reads 8 consecutive
// chunks -- conflict-free under the XOR swizzle.  Ascending s2 order.
struct SumArgs {
  uint32_t R;  // this CTA's R (shared window)
  int ks, rows_per, row_base, col_base, prank, CG;
};
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
template <int S, bool L2>
__device__ __forceinline__ void splitk_sum(const SumArgs& a, const AgTcParams& p) {
  const int tasks = a.rows_per * 32;
  uint32_t src[S];
#pragma unroll
  for (int s2 = 0; s2 < S; ++s2) src[s2] = L2 ? 0u : mapa_u32(a.R, uint32_t(a.prank + a.CG * s2));
  for (int e = threadIdx.x; e < tasks; e += NUM_THREADS) {
    const int rl = a.ks * a.rows_per + e / 32, g = e % 32;
    const int grow = a.row_base + rl, gcol = a.col_base + g * 4;
    const uint32_t off0 = uint32_t(rl * 1024 + ((g ^ (rl & 7)) * 16));
    const uint32_t off1 = uint32_t(rl * 1024 + (((g + 32) ^ (rl & 7)) * 16));
    float4 x[S], y[S];
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) {
      if (L2) {  // sibling s2's copy sits in slice position s2 of R
        const uint32_t b = a.R + uint32_t((s2 - a.ks) * a.rows_per * 1024);
        x[s2] = lds128f(b + off0);
        y[s2] = lds128f(b + off1);
      } else if (s2 == a.ks) {
        x[s2] = lds128f(a.R + off0);
        y[s2] = lds128f(a.R + off1);
      } else {  // sibling s2's R: same offset in its window
        const uint32_t rb = src[s2];
        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(x[s2].x), "=f"(x[s2].y), "=f"(x[s2].z), "=f"(x[s2].w) : "r"(rb + off0));
        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(y[s2].x), "=f"(y[s2].y), "=f"(y[s2].z), "=f"(y[s2].w) : "r"(rb + off1));
      }
    }
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) {
      acc[0] += x[s2].x; acc[1] += x[s2].y; acc[2] += x[s2].z; acc[3] += x[s2].w;
      acc[4] += y[s2].x; acc[5] += y[s2].y; acc[6] += y[s2].z; acc[7] += y[s2].w;
    }
    if (grow < p.M && !(p.dbg & 1)) {
      __nv_bfloat16* crow = p.C + size_t(grow) * p.ldc;
      if (gcol < p.N)
        *reinterpret_cast<uint2*>(crow + gcol) = make_uint2(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]));
      if (gcol + 128 < p.N)
        *reinterpret_cast<uint2*>(crow + gcol + 128) =
            make_uint2(pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
    }
  }
}

template <int CG, int NH_, int BK_ = 64>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    ag_gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA_own,
                         const __grid_constant__ CUtensorMap tmA_inbox,
                         const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmC,
                         const __grid_constant__ CUtensorMap tmB4, const AgTcParams p) {
  pdl_launch();
  if (p.dbg & 65536) pdl_wait();  // A/B knob: wait at entry (round-2 placement)
  using K_ = Cfg<CG, NH_, BK_>;
  constexpr int STAGES = K_::STAGES, NH = K_::NH, CPH = K_::CPH;
  constexpr int BK = K_::BK, A_BYTES = K_::A_BYTES;  // shadow the 64-deep globals
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * A_BYTES;
  uint8_t* smStage = smem + STAGES * K_::STAGE_BYTES;  // epilogue: 4 warps x 2 x 4 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(smStage + K_::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;  // split-K (L2 exchange): siblings' slices landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Cluster = CG * ksplit CTAs: pairs (cta_group::2) at ranks (2j, 2j+1),
  // split-K siblings of one tile at ranks prank + CG * ks.
  const uint32_t crank = (CG == 2 || p.ksplit > 1) ? cluster_ctarank() : 0;
  const uint32_t prank = CG == 2 ? (crank & 1u) : 0u;   // rank inside the CTA pair
  const uint32_t lead = crank - prank;                  // the pair leader's cluster rank
  const uint16_t pair_mask = uint16_t(3u << lead);
  const bool leader = prank == 0;
  const bool two_prod = NH == 1 && !p.gather && !p.one_producer;  // B boxes from warp 6 (see the producer)
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;
  const int num_mt = (p.num_m + CG - 1) / CG;  // tile rows (BM * CG each)
  // Work items: (tile, k-split).  Split ks covers k-block slots
  // [ks*kb/S, (ks+1)*kb/S) of the rank's rotated k order (never empty:
  // the host keeps kb_total >= 4 * ksplit).
  const int num_tiles = p.total_items;
  auto tcoords = [&](int t, int& mt, int& nb) {
    tile_coords(num_mt, p.num_n, t, mt, nb);
    if (p.mt_rot) mt = (mt + p.mt_rot) % num_mt;
  };
  auto item_coords = [&](int t, int& mt, int& nb, int& i0, int& i1) {
    const int ks = t % p.ksplit;
    tcoords(t / p.ksplit, mt, nb);
    i0 = ks * p.kb_total / p.ksplit;
    i1 = (ks + 1) * p.kb_total / p.ksplit;
  };
  // Item geometry: rows (tile row mt), columns [col0, col0 + w), k-blocks
  // [i0, i1).  The tiles of a partial last wave are cut into q_tail column
  // slices (w = BN_TILE / q_tail: 256 or 128) so every pair has work at the
  // end instead of a quarter of them running whole tiles.
  auto item_geom = [&](int t, int& mt, int& col0, int& w, int& i0, int& i1) {
    int nb;
    if (t < p.full_items) {
      item_coords(t, mt, nb, i0, i1);
      col0 = nb * K_::BN_TILE;
      w = K_::BN_TILE;
    } else {
      const int j = t - p.full_items;
      tcoords(p.full_items + j / p.q_tail, mt, nb);
      w = K_::BN_TILE / p.q_tail;
      col0 = nb * K_::BN_TILE + (j % p.q_tail) * w;
      i0 = 0;
      i1 = p.kb_total;
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA_own);
    tma_prefetch(&tmA_inbox);
    tma_prefetch(&tmB);
    tma_prefetch(&tmC);
    if (p.b4) tma_prefetch(&tmB4);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], CG * (two_prod ? 2 : 1));  // one arrive per producer thread per CTA (leader's copy used)
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * CG);
    }
    mbar_init(rbar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_cg<CG>(tmem_slot);
  tc_fence_before();
  if (CG == 2 || p.ksplit > 1) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the predecessor's writes (A, B, flags, C, counters) are visible from here on
  // Profiling (TFB_DEBUG & 4096): %globaltimer phase stamps of CTA 0, printed at exit.
  __shared__ unsigned long long s_ts[12];
  __shared__ unsigned long long s_kp[24], s_km[24];  // TFB_DEBUG 8192: producer / MMA per-k-block stamps
  const bool tsd = (p.dbg & 4096) && blockIdx.x == 0;
  if (tsd && threadIdx.x == 0)
    for (int i = 0; i < 12; ++i) s_ts[i] = i == 0 ? globaltimer_ns() : 0;

  if (warp == 0 || (two_prod && warp == 6)) {
    // ===== TMA producer (both CTAs of a pair) =====
    // With NH = 1 and no gather work, warp 6 (otherwise idle) issues the B
    // boxes and warp 0 the A boxes: the producer's per-k-block chain is the
    // skinny-M bound (TFB_DEBUG 8192 cadence), and the TMA issue is most of it.
    const bool do_a = warp == 0, do_b = warp == 6 || !two_prod;
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // L2 policies (p.l2hint): A rows are re-read by every tile column of
      // their raster group, B panels only by the tiles running at the same
      // time -- keep A, stream B.
      uint64_t pol_a = 0, pol_b = 0;
      if (p.l2hint & 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_a));
      if (p.l2hint & 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_b));
      // Launch constants hoisted into registers: the k-block loop below is
      // one thread's dependent instruction chain that no other warp hides,
      // so it carries no divisions and no parameter reloads (TFB_DEBUG 8192
      // cadence with loads and MMAs off: ~790 cycles per k-block with the
      // per-iteration `%` / `/` and constant-bank reloads).
      const int own = p.own, kbw = p.kbw, kbt = p.kb_total, nm = p.num_m;
      const bool msh = p.msharded != 0, b4 = p.b4 != 0;
      const bool skip_a = (p.dbg & 256) != 0 || !do_a, skip_b = (p.dbg & 512) != 0 || !do_b;
      const bool kstamp = (p.dbg & 8192) != 0 && do_a;
      const uint64_t* const ready = p.ready;
      const uint32_t full_bar0 = CG == 2 ? mapa(&full[0], lead) : smem_u32(&full[0]);
      const int a_col_own = msh ? 0 : own * p.kw;       // own-shard map: column offset (K-sharded)
      const int a_row_own = msh ? own * p.mpr * BM : 0;  // own-shard map: row offset (M-sharded)
      for (int t = cid; t < num_tiles; t += ncl) {
        int mt, n0, wcol, i0, i1;
        item_geom(t, mt, n0, wcol, i0, i1);
        const int mb = mt * CG + int(prank);  // this CTA's 128-row block
        const int m0 = mb * BM;
        // B chunks (64 columns) this CTA stages per k-block: its share of
        // every 256-column MMA (CG = 2: 128 columns), or of one 128-wide one.
        const int nhalf = wcol >= 256 ? wcol / 256 : 1;
        const int cpc = wcol >= 256 ? CPH : 2 / CG;  // chunks per MMA per CTA
        const uint32_t tx = uint32_t(CG) * uint32_t((skip_a ? 0 : A_BYTES) + (skip_b ? 0 : nhalf * cpc * BK * 128));
        const bool whole = wcol == K_::BN_TILE;
        uint64_t ready_mask = 0;
        // k-block of slot i0 in the rank's rotated order, its owner (column
        // band; M-sharded: row band, rows past M reading the zero-filled
        // edge) and its position inside the owner's band -- then stepped.
        int kb = msh ? i0 : own >= 0 ? (i0 + own * kbw) % kbt : i0;
        int src = !msh ? kb / kbw : mb < nm ? mb / p.mpr : -1;
        int kin = msh ? 0 : kb - src * kbw;
        const bool gated = do_a && ready != nullptr && mb < nm;
        for (int i = i0; i < i1; ++i) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (kstamp && blockIdx.x == 0 && t == cid && i - i0 < 24) s_kp[i - i0] = clock64();
          const bool from_own = src == own;
          if (gated && !from_own && !((ready_mask >> src) & 1ull)) {
            wait_geq(ready + size_t(mb) * p.W + src, p.epoch, p.watchdog_ns, p.err, kWaitSignal, own, p.board,
                     src, mb, 0);
            fence_proxy_async_global();
            ready_mask |= 1ull << src;
            if (p.events)  // first consumer load of this (m-block, source) chunk
              atomicMin(p.events + (size_t(mb) * p.W + src) * 2 + 1, (unsigned long long)globaltimer_ns());
          }
          const uint32_t bar = full_bar0 + uint32_t(stage) * 8u;
          if (leader) mbar_arrive_expect_tx(&full[stage], tx);
          else mbar_arrive_cluster(bar);
          if (!skip_a) {
            uint8_t* a_dst = smA + stage * A_BYTES;
#pragma unroll
            for (int ab = 0; ab < BK / 64; ++ab) {  // 64-column boxes (SW128's 128-byte rows)
              if (from_own)
                tma_load<CG>(a_dst + ab * (BM * 128), &tmA_own, bar, kb * BK + ab * 64 - a_col_own, m0 - a_row_own,
                             pol_a);
              else tma_load<CG>(a_dst + ab * (BM * 128), &tmA_inbox, bar, kb * BK + ab * 64, m0, pol_a);
            }
          }
          uint8_t* b_dst = smB + stage * K_::B_BYTES;
          if (skip_b) {
          } else if (whole && b4) {
            tma_load_4d<CG>(b_dst, &tmB4, bar, kb * BK, int(prank) * CPH, n0 / 256, pol_b);
          } else if (whole) {
#pragma unroll
            for (int h = 0; h < NH; ++h)
#pragma unroll
              for (int c = 0; c < CPH; ++c)
                tma_load<CG>(b_dst + (h * CPH + c) * (BK * 128), &tmB, bar,
                             n0 + h * 256 + int(prank) * (CPH * 64) + c * 64, kb * BK);
          } else {
            for (int h = 0; h < nhalf; ++h)
              for (int c = 0; c < cpc; ++c)
                tma_load<CG>(b_dst + (h * CPH + c) * (BK * 128), &tmB, bar,
                             n0 + h * 256 + int(prank) * (cpc * 64) + c * 64, kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (msh) {
            ++kb;
          } else {
            if (++kb == kbt) kb = 0;
            if (++kin == kbw) {  // next owner's band (rare: W times per tile)
              kin = 0;
              src = kb / kbw;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA, one thread) =====
    // 256 x 512 tiles (NH = 2) keep ONE accumulator (the whole TMEM), so the
    // epilogue of tile t drains it while tile t+1 waits.  The drain is split
    // per 256-column half (tempty[0] / tempty[1]): tile t+1 issues its
    // half-0 MMAs for the first STAGES k-blocks as soon as half 0 is free,
    // and catches up half 1 once the epilogue has drained it.
    if (lane == 0 && leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      // Shared-memory descriptors as base + offset: the start-address field
      // is the low 14 bits of (address >> 4) and never carries (smem < 256
      // KB), so stage / k / half steps are plain adds -- the MMA thread's
      // per-k-block chain stays short (it paced the skinny main loops).
      const uint64_t adesc0 = smem_desc_sw128(smem_u32(smA), 16, 1024);
      const uint64_t bdesc0 = smem_desc_sw128(smem_u32(smB), BK * 128, 1024);
      const bool no_mma = (p.dbg & 2) != 0;
      const bool mstamp = (p.dbg & 8192) != 0 && blockIdx.x == 0;
      const bool kfence = (p.dbg & 32768) == 0;  // TFB_DEBUG 32768: no tcgen05 fence after each full wait (A/B)
      auto mma_kblock = [&](int stg, int h0, int h1, bool first_kb, bool whole, int nhalf, uint32_t idesc) {
        if (no_mma) return;
        const uint64_t a_st = adesc0 + uint64_t(uint32_t(stg * A_BYTES) >> 4);
        const uint64_t b_st = bdesc0 + uint64_t(uint32_t(stg * K_::B_BYTES) >> 4);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          // A: K-major SW128, 8-row groups 1024 B apart; +32 B per K=16
          // inside a 64-column box, boxes BM * 128 B apart.
          const uint64_t ad = a_st + uint64_t(((k >> 2) * (BM * 128) + (k & 3) * 32) >> 4);
          // B: MN-major SW128, 64-column chunks 8 KB apart (LBO), 8-row K
          // groups 1 KB apart (SBO); +16 rows (2 KB) per K=16.  Whole tiles
          // take the unrolled constant-descriptor path: the single issuing
          // thread must stay well ahead of the tensor pipe (a runtime-bounded
          // loop here cost 16 % of the config-2 cycles).
          if (whole) {
#pragma unroll
            for (int h = 0; h < NH; ++h) {
              if (h < h0 || h >= h1) continue;
              const uint64_t bd = b_st + uint64_t((h * CPH * (BK * 128) + k * 2048) >> 4);
              mma_issue<CG>(tmem_base + uint32_t((acc * NH + h) * 256), ad, bd, K_::IDESC, !first_kb || k != 0);
            }
          } else {
            for (int h = 0; h < nhalf; ++h) {
              const uint64_t bd = b_st + uint64_t(uint32_t(h * CPH * (BK * 128) + k * 2048) >> 4);
              mma_issue<CG>(tmem_base + uint32_t((acc * NH + h) * 256), ad, bd, idesc, !first_kb || k != 0);
            }
          }
        }
      };
      auto advance = [&](int& stg, uint32_t& ph) {
        if (++stg == STAGES) {
          stg = 0;
          ph ^= 1;
        }
      };
      for (int t = cid; t < num_tiles; t += ncl) {
        int mt_, c0_, wcol, i0, i1;
        item_geom(t, mt_, c0_, wcol, i0, i1);
        const bool whole = wcol == K_::BN_TILE;
        const int nhalf = wcol >= 256 ? wcol / 256 : 1;
        const uint32_t idesc = wcol >= 256 ? K_::IDESC : idesc_bf16(BM * CG, wcol, 0, 1);
        int i = i0;
        if (NH == 2 && whole) {
          mbar_wait(&tempty[0], aphase ^ 1);
          tc_fence_after();
          const int pre = min(STAGES, i1 - i0);
          int s2 = stage;
          uint32_t p2 = phase;
          for (int j = 0; j < pre; ++j) {
            mbar_wait(&full[s2], p2);
            if (kfence) tc_fence_after();
            mma_kblock(s2, 0, 1, j == 0, true, 2, idesc);
            advance(s2, p2);
          }
          mbar_wait(&tempty[1], aphase ^ 1);
          tc_fence_after();
          for (int j = 0; j < pre; ++j) {
            mma_kblock(stage, 1, 2, j == 0, true, 2, idesc);
            mma_commit_all<CG>(&empty[stage], pair_mask);
            advance(stage, phase);
          }
          i = i0 + pre;
        } else if (NH == 2) {
          mbar_wait(&tempty[0], aphase ^ 1);
          mbar_wait(&tempty[1], aphase ^ 1);
          tc_fence_after();
        } else {
          mbar_wait(&tempty[acc], aphase ^ 1);
          tc_fence_after();
        }
        for (; i < i1; ++i) {
          mbar_wait(&full[stage], phase);
          if (mstamp && t == cid && i - i0 < 24) s_km[i - i0] = clock64();
          if (tsd && !s_ts[1]) s_ts[1] = globaltimer_ns();
          if (kfence) tc_fence_after();
          mma_kblock(stage, 0, NH, i == i0, whole, nhalf, idesc);
          mma_commit_all<CG>(&empty[stage], pair_mask);
          advance(stage, phase);
        }
        if (tsd) s_ts[2] = globaltimer_ns();
        mma_commit_all<CG>(&tfull[acc], pair_mask);
        if (++acc == K_::ACC_BUFS) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
  } else if (warp < 6 || (NH == 2 && !p.gather && warp < 10)) {
    // ===== epilogue (both CTAs): TMEM -> registers -> bf16 -> global =====
    // Warps 2-5; with NH = 2 and no gather work (W = 1, push, baseline) also
    // warps 6-9, the two sets draining the two 256-column halves at once.
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const bool epi8 = NH == 2 && !p.gather;
    const int e = warp - 2, set = epi8 && warp >= 6 ? 1 : 0;
    int acc = 0;
    uint32_t aphase = 0;
    const uint32_t tempty_leader0 = CG == 2 ? mapa(&tempty[0], lead) : smem_u32(&tempty[0]);
    auto arrive = [&](int idx) {
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(tempty_leader0 + uint32_t(idx) * 8);
        else mbar_arrive(&tempty[idx]);
      }
    };
    int nst = 0;  // TMA stores issued by this warp (staging-buffer reuse)
    // Split-K: one item per CTA, reduced after the role loops (below).
    for (int t = p.ksplit > 1 ? num_tiles : cid; t < num_tiles; t += ncl) {
      int mt, col0, wcol;
      int i0_, i1_;
      item_geom(t, mt, col0, wcol, i0_, i1_);
      if (!(p.dbg & 32)) mbar_wait_sleep(&tfull[acc], aphase);
      else mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      // 64-column slabs: two tcgen05.ld (32 columns each) -> bf16 -> a
      // SWIZZLE_128B smem box [32 rows][64 cols] (conflict-free: 16-byte
      // chunk j of row r sits at j ^ (r & 7)) -> one TMA store per warp per
      // slab; the next slab's TMEM reads overlap the store (two staging
      // buffers per warp with four epilogue warps, one with eight).
      const int row0 = (mt * CG + int(prank)) * BM + 32 * q;
      const int slabs = (p.dbg & 64) ? 0 : wcol / 64;
      const int half0 = min(slabs, 4);  // slabs in TMEM columns [0, 256)
      const int c_begin = !epi8 ? 0 : set == 0 ? 0 : half0;
      const int c_end = !epi8 ? slabs : set == 0 ? half0 : slabs;
#pragma unroll 1
      for (int cc = c_begin; cc < c_end; ++cc) {
        uint32_t r0[32], r1[32];
        const uint32_t tcol = uint32_t(acc * NH * 256 + 64 * cc);
        tmem_ld_32x32b_x32(tmem_base + (uint32_t(32 * q) << 16) + tcol, r0);
        tmem_ld_32x32b_x32(tmem_base + (uint32_t(32 * q) << 16) + tcol + 32, r1);
        tmem_ld_wait();
        uint8_t* buf = epi8 ? smStage + e * 4096 : smStage + (e * 2 + (nst & 1)) * 4096;
        if (lane == 0) {
          if (epi8) bulk_wait_read<0>();
          else if (nst >= 2) bulk_wait_read<1>();
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t* src = j < 4 ? &r0[8 * j] : &r1[8 * (j - 4)];
          uint4 pk;
          pk.x = pack_bf16x2(__uint_as_float(src[0]), __uint_as_float(src[1]));
          pk.y = pack_bf16x2(__uint_as_float(src[2]), __uint_as_float(src[3]));
          pk.z = pack_bf16x2(__uint_as_float(src[4]), __uint_as_float(src[5]));
          pk.w = pack_bf16x2(__uint_as_float(src[6]), __uint_as_float(src[7]));
          sts128(smem_u32(buf) + uint32_t(lane * 128 + ((j ^ (lane & 7)) * 16)), pk);
        }
        fence_proxy_async_shared();
        __syncwarp();
        if (lane == 0 && !(p.dbg & 1) && row0 < p.M) {
          tma_store_2d(&tmC, buf, col0 + 64 * cc, row0);
          bulk_commit();
        }
        ++nst;
        if (NH == 2 && !epi8 && cc + 1 == half0) {
          tc_fence_before();
          __syncwarp();
          arrive(0);  // half 0 drained: the next tile's half-0 MMAs may start
        }
      }
      tc_fence_before();
      __syncwarp();
      if (NH == 2) {
        if (epi8) arrive(set);
        else {
          if (half0 == 0) arrive(0);
          arrive(1);
        }
      } else {
        arrive(acc);
      }
      if (++acc == K_::ACC_BUFS) {
        acc = 0;
        aphase ^= 1;
      }
    }
    if (lane == 0) bulk_wait_all();  // C stores complete before the CTA retires
    if (tsd && warp == 2 && lane == 0) s_ts[7] = globaltimer_ns();
  } else if (p.gather) {
    // ===== gather (PULL): peer shard chunks -> local inbox + ready flags =====
    const int gt = threadIdx.x - 6 * 32;  // 0..GATHER_T-1
    __shared__ unsigned int s_chunk;
    // Remote shards only: the TMA producer reads the rank's own k-range
    // straight from its shard, so copying it into the inbox would be a
    // wasted m x kw read + write per call.  A caller-supplied gathered
    // buffer (placement check) gets the own shard too, last.
    const int nsrc = p.W - 1 + p.gather_own;
    // M-sharded: one chunk per m-block this rank does not own (plus its own,
    // last, into a caller's buffer), starting after its own rows -- the
    // order its rotated tile rows consume them.  Rows are contiguous in the
    // owner's shard and in the inbox, so a chunk is one flat copy.
    const unsigned total = p.msharded ? unsigned(p.num_m - (p.gather_own ? 0 : p.mpr))
                                      : unsigned(p.num_m) * unsigned(nsrc);
    const int vec_per_row = (p.msharded ? p.K : p.kw) / 8;  // 16-byte vectors per copied row
    for (;;) {
      if (gt == 0) s_chunk = atomicAdd(&p.ctr[0], 1u);
      named_bar(1, GATHER_T);
      const unsigned c = s_chunk;
      named_bar(1, GATHER_T);
      if (c >= total) break;
      const int mb = p.msharded ? int((unsigned(p.own + 1) * p.mpr + c) % unsigned(p.num_m)) : int(c / nsrc);
      const int src = p.msharded ? mb / p.mpr : (p.own + 1 + int(c % nsrc)) % p.W;
      const int r0 = mb * BM, rows = min(BM, p.M - r0);
      const uint4* s = reinterpret_cast<const uint4*>(
          p.msharded ? p.peer_shard[src] + size_t(r0 - src * p.mpr * BM) * p.K : p.peer_shard[src] + size_t(r0) * p.kw);
      const int nvec = rows * vec_per_row;
      constexpr int U = 8;
      for (int base = 0; base < nvec; base += GATHER_T * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = base + u * GATHER_T + gt;
          if (e < nvec) v[u] = s[e];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = base + u * GATHER_T + gt;
          if (e < nvec) {
            const int rr = e / vec_per_row, cv = e % vec_per_row;
            *reinterpret_cast<uint4*>(p.inbox + size_t(r0 + rr) * p.K + (p.msharded ? 0 : size_t(src) * p.kw) + 8 * cv) =
                v[u];
          }
        }
      }
      fence_proxy_async_global();
      named_bar(1, GATHER_T);
      if (gt == 0) {
        __threadfence();
        if (p.events) p.events[(size_t(mb) * p.W + src) * 2] = globaltimer_ns();  // chunk landed
        red_release_sys(p.ready_w + size_t(mb) * p.W + src, 1);
      }
    }
  }

  if (p.ksplit > 1) {
    // ===== split-K reduction through distributed shared memory =====
    // Every CTA of the cluster holds a 128-row fp32 partial of the same tile
    // (its k-range) in TMEM.  Per 256-column half: the epilogue warps dump it
    // into this CTA's (drained) pipeline smem, the cluster syncs, then CTA ks
    // sums rows [ks*128/S, (ks+1)*128/S) over the S siblings in ascending
    // split order (deterministic) straight from their smem, and stores bf16
    // C.  No workspace, no second launch.  (Measured: a push variant --
    // remote st.shared::cluster into the owner's slots -- costs the same;
    // DSMEM moves ~20 B/clk per SM either way.)
    const int S = p.ksplit;
    const int ks = int(crank) / CG;
    const int rows_per = BM / S;
    int mt, nb, i0_, i1_;
    item_coords(cid, mt, nb, i0_, i1_);
    float* R = reinterpret_cast<float*>(smem);  // [128][256] fp32, 16-byte chunks swizzled by row & 7
    const int row_base = (mt * CG + int(prank)) * BM;
    // The dump runs on warps 2-9 (the gather warps are done by now): two
    // warps per TMEM lane quarter, each 128 of the half's 256 columns.
    if (warp >= 2 && warp < 10) {
      mbar_wait(&tfull[0], 0);
      tc_fence_after();
      if (tsd && warp == 2 && lane == 0) s_ts[3] = globaltimer_ns();
    }
#pragma unroll 1
    for (int h = 0; h < NH; ++h) {
      if (warp >= 2 && warp < 10) {
        const int row = 32 * (warp & 3) + lane;
        const int cc0 = warp < 6 ? 0 : 4;
#pragma unroll 1
        for (int cc = cc0; cc < cc0 + 4; ++cc) {
          uint32_t r0[32];
          tmem_ld_32x32b_x32(tmem_base + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(h * 256 + 32 * cc), r0);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = cc * 8 + j;  // 16-byte chunk of the 256-column row
            sts128(smem_u32(R) + uint32_t(row * 1024 + ((c ^ (row & 7)) * 16)),
                   make_uint4(r0[4 * j], r0[4 * j + 1], r0[4 * j + 2], r0[4 * j + 3]));
          }
        }
      }
      if (p.ws) {
        // L2 exchange: slice j of this partial (rows [j*rp, (j+1)*rp), whole
        // 1 KB rows, contiguous in R) goes to workspace ws[cta][h] by one
        // bulk copy each; after the cluster barrier each CTA bulk-loads its
        // siblings' copies of the slice it owns into the vacated slice
        // positions of its own R, then sums all S from local smem in
        // ascending split order (the same bits as the DSMEM path).  DSMEM
        // moves ~8-9 B/clk per SM when every SM reduces at once
        // (tools/micro_dsmem.cu).
        const uint32_t slice = uint32_t(rows_per) * 1024u;
        uint8_t* wsme = p.ws + (size_t(blockIdx.x) * NH + h) * (size_t(BM) * 1024);
        fence_proxy_async_shared();
        named_bar(2, NUM_THREADS);
        if (tsd && threadIdx.x == 0 && h == 0) s_ts[8] = globaltimer_ns();  // partial dumped
        if (p.xchg_lsu) {
          // Every thread copies 16-byte words of the outgoing slices (raw
          // bytes, layout kept); the cluster barrier's release orders them
          // before the siblings' loads -- no TMA-store drain on the chain.
          for (int j = 0; j < S; ++j) {
            if (j == ks) continue;
            const uint4* from = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(R) + j * slice);
            uint4* to = reinterpret_cast<uint4*>(wsme + j * slice);
            for (int v = threadIdx.x; v < int(slice / 16); v += NUM_THREADS) __stcg(to + v, from[v]);
          }
          if (threadIdx.x == 0) mbar_arrive_expect_tx(rbar, slice * uint32_t(S - 1));
        } else if (threadIdx.x == 0) {
          for (int j = 0; j < S; ++j) {
            if (j == ks) continue;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(wsme + j * slice),
                         "r"(smem_u32(R) + j * slice), "r"(slice)
                         : "memory");
          }
          bulk_commit();
          bulk_wait_all();
          if (tsd && h == 0) s_ts[9] = globaltimer_ns();  // slices in L2
          asm volatile("fence.proxy.async.global;" ::: "memory");
          mbar_arrive_expect_tx(rbar, slice * uint32_t(S - 1));
        }
        cluster_sync();
        if (tsd && threadIdx.x == 0 && h == 0) s_ts[10] = globaltimer_ns();  // cluster synced
        if (threadIdx.x == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          const int cta0 = int(blockIdx.x) - int(crank);  // cluster's first CTA
          for (int j = 0; j < S; ++j) {
            if (j == ks) continue;
            const uint8_t* from = p.ws + (size_t(cta0 + int(prank) + CG * j) * NH + h) * (size_t(BM) * 1024) +
                                  size_t(ks) * slice;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(R) + j * slice),
                "l"(from), "r"(slice), "r"(smem_u32(rbar))
                : "memory");
          }
        }
        mbar_wait(rbar, uint32_t(h & 1));
      } else {
        cluster_sync();
      }
      if (tsd && threadIdx.x == 0 && h == 0) s_ts[4] = globaltimer_ns();  // partials exchanged
      // The owned rows' ascending S-way sum and bf16 C stores, specialised
      // on S and the exchange route: the generic loop's per-sibling branches
      // made it instruction-bound at 10 warps (~650 cycles per 320 tasks,
      // 2.6 us of the M = 256 tail; clock64 per warp, TFB_DEBUG 4096).
      if (!(p.dbg & 16)) {
        const SumArgs sa{smem_u32(R), ks, rows_per, row_base, nb * K_::BN_TILE + h * 256, int(prank), CG};
        const bool l2 = p.ws != nullptr;
        if (S == 2) l2 ? splitk_sum<2, true>(sa, p) : splitk_sum<2, false>(sa, p);
        else if (S == 4) l2 ? splitk_sum<4, true>(sa, p) : splitk_sum<4, false>(sa, p);
        else l2 ? splitk_sum<8, true>(sa, p) : splitk_sum<8, false>(sa, p);
      }
      if (tsd && threadIdx.x == 0) s_ts[5 + h] = globaltimer_ns();  // half h summed + stored
      // R fully read (siblings included) before the next half's dump; after
      // the last half the kernel's closing cluster barrier does it.
      if (h + 1 < NH) {
        if (p.ws) named_bar(2, NUM_THREADS);
        else cluster_sync();
      }
    }
  }

  tc_fence_before();
  if (CG == 2 || p.ksplit > 1) cluster_sync();
  else __syncthreads();
  if ((p.dbg & 8192) && blockIdx.x == 0 && threadIdx.x == 0) {
    printf("[ag cta0 k-block cadence, cycles] producer-empty:");
    for (int i = 1; i < 24; ++i) printf(" %lld", (long long)(s_kp[i] - s_kp[i - 1]));
    printf("\n[ag cta0 k-block cadence, cycles] mma-full:      ");
    for (int i = 1; i < 24; ++i) printf(" %lld", (long long)(s_km[i] - s_km[i - 1]));
    printf("\n[ag cta0] mma-full[i] - producer-empty[i]:");
    for (int i = 0; i < 24; ++i) printf(" %lld", (long long)(s_km[i] - s_kp[i]));
    printf("\n");
  }
  if (tsd && threadIdx.x == 0) {
    auto rel = [&](int i) { return s_ts[i] ? (long long)(s_ts[i] - s_ts[0]) : -1ll; };
    printf("[ag cta0 CG=%d NH=%d S=%d] first-stage %lld last-commit %lld tfull %lld dumped %lld inl2 %lld "
           "synced %lld exchanged %lld sum0 %lld sum1 %lld epilogue %lld exit %lld ns\n", CG, NH, p.ksplit, rel(1),
           rel(2), rel(3), rel(8), rel(9), rel(10), rel(4), rel(5), rel(6), rel(7),
           (long long)(globaltimer_ns() - s_ts[0]));
  }
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc_cg<CG>(tmem_base);
  }
  if (threadIdx.x == 0 && p.ctr) {
    __threadfence();
    if (atomicAdd(&p.ctr[1], 1u) == gridDim.x - 1) {
      p.ctr[0] = 0;
      p.ctr[1] = 0;
      __threadfence();
    }
  }
}

// PUSH producer (ag_gemm.hpp:241-260): claim (dst, m_blk) chunks, store this
// rank's rows [m_blk*128, +128) x kw into dst's inbox at column self*kw, then
// raise dst's ready[m_blk][self] with release semantics.  Never waits.
struct PushParams {
  const __nv_bfloat16* shard;
  __nv_bfloat16* inbox[64];
  uint64_t* ready[64];
  unsigned long long* events[64];  // every rank's event log (or null)
  int M, K, kw, W, self, num_m;
  int msharded, mpr;  // M-sharded A: push this rank's own row band
  unsigned int* ctr;  // [0] chunk counter, [1] done
};

__global__ void __launch_bounds__(512) ag_push_kernel(const PushParams p) {
  __shared__ unsigned int s_chunk;
  const unsigned total = p.msharded ? unsigned(p.mpr) * p.W : unsigned(p.num_m) * p.W;
  const int vec_per_row = (p.msharded ? p.K : p.kw) / 8;
  for (;;) {
    if (threadIdx.x == 0) s_chunk = atomicAdd(&p.ctr[0], 1u);
    __syncthreads();
    const unsigned c = s_chunk;
    __syncthreads();
    if (c >= total) break;
    // m-block major so every consumer's first tiles are fed first; peers
    // before self (the consumer reads its own shard directly).
    const int mb = p.msharded ? p.self * p.mpr + int(c / p.W) : int(c / p.W);
    const int dst = (p.self + 1 + int(c % p.W)) % p.W;
    const int r0 = mb * BM, rows = min(BM, p.M - r0);
    const uint4* s = reinterpret_cast<const uint4*>(p.msharded ? p.shard + size_t(r0 - p.self * p.mpr * BM) * p.K
                                                               : p.shard + size_t(r0) * p.kw);
    __nv_bfloat16* ib = p.inbox[dst];
    const int nvec = rows * vec_per_row;
    constexpr int U = 8;  // 64 KB of loads in flight per CTA feeding peer stores
    for (int base = 0; base < nvec; base += 512 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * 512 + threadIdx.x;
        if (e < nvec) v[u] = s[e];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * 512 + threadIdx.x;
        if (e < nvec) {
          const int rr = e / vec_per_row, cv = e % vec_per_row;
          *reinterpret_cast<uint4*>(ib + size_t(r0 + rr) * p.K + (p.msharded ? 0 : size_t(p.self) * p.kw) + 8 * cv) =
              v[u];
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_sys();
      if (p.events[dst]) p.events[dst][(size_t(mb) * p.W + p.self) * 2] = globaltimer_ns();  // chunk stored
      red_release_sys(p.ready[dst] + size_t(mb) * p.W + p.self, 1);
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&p.ctr[1], 1u) == gridDim.x - 1) {
      p.ctr[0] = 0;
      p.ctr[1] = 0;
      __threadfence();
    }
  }
}

// PUSH producer on the TMA engine: one warp per CTA, one elected thread.
// Each claimed m-block of this rank's shard is staged box by box (64 x 256
// bf16 = 32 KB, SWIZZLE_NONE) into a kPushStages-deep smem ring by TMA
// loads, and every staged box is written to all W inboxes by TMA stores
// (read once, stored W times -- the multicast-shaped part of push).  After
// an m-block's stores complete (bulk wait_group 0), its W flags are raised
// with system-scope release.  The SM does no per-element work, so a few
// CTAs move what 16 register-copy CTAs did (tools/probe_push.py).
constexpr int kPushStages = 4;
constexpr int kPushMaxW = 8;
struct PushMaps {
  CUtensorMap src;                // this rank's shard: K-sharded [M][kw], M-sharded [mr][K]
  CUtensorMap dst[kPushMaxW];     // every rank's inbox [M][K]
};
struct PushTmaParams {
  uint64_t* ready[kPushMaxW];
  unsigned long long* events[kPushMaxW];
  int W, self, nmb;          // m-blocks this rank pushes
  int msharded, mpr;
  int box_c, box_r;          // box columns / rows
  int cols;                  // shard columns (kw or K)
  int M;
  int local;                 // every destination inbox is on this CTA's device
  int skip_self;             // own block read in place: only its flag is raised
  unsigned int* ctr;         // [0] m-block counter, [1] done
};

__global__ void __launch_bounds__(32) ag_push_tma_kernel(const __grid_constant__ PushMaps maps,
                                                         const __grid_constant__ PushTmaParams p) {
  extern __shared__ __align__(1024) uint8_t push_smem[];
  __shared__ __align__(8) uint64_t full[kPushStages];
  if (threadIdx.x != 0) return;
  const uint32_t box_bytes = uint32_t(p.box_c) * uint32_t(p.box_r) * 2u;
  for (int s = 0; s < kPushStages; ++s) mbar_init(&full[s], 1);
  fence_mbar_init();
  tma_prefetch(&maps.src);
  for (int d = 0; d < p.W; ++d) tma_prefetch(&maps.dst[d]);
  const int ncb = p.cols / p.box_c, nrb = BM / p.box_r, nbox = ncb * nrb;
  uint32_t issued = 0, consumed = 0;  // ring positions (box sequence numbers) of this CTA
  for (;;) {
    const int i = int(atomicAdd(&p.ctr[0], 1u));
    if (i >= p.nmb) break;
    const int mb = p.msharded ? p.self * p.mpr + i : i;   // global m-block (inbox rows)
    const int r_src = p.msharded ? i * BM : mb * BM;      // rows in the shard map
    const int c_dst = p.msharded ? 0 : p.self * p.cols;   // inbox column of the shard's column 0
    auto box_at = [&](int j, int& c, int& r) {
      c = (j % ncb) * p.box_c;
      r = (j / ncb) * p.box_r;
    };
    // Prime S - 1 stages, then: wait box j, store it to every inbox, and
    // load box j + S - 1 into the stage of box j - 1 (whose stores have read
    // it: every group but the newest).
    int next = 0;
    auto load_next = [&]() {
      const uint32_t st = issued % kPushStages;
      int c, r;
      box_at(next, c, r);
      mbar_arrive_expect_tx(&full[st], box_bytes);
      tma_load_2d(push_smem + st * box_bytes, &maps.src, &full[st], c, r_src + r);
      ++issued;
      ++next;
    };
    while (next < nbox && issued - consumed < uint32_t(kPushStages - 1)) load_next();
    for (int j = 0; j < nbox; ++j) {
      const uint32_t st = consumed % kPushStages;
      mbar_wait(&full[st], (consumed / kPushStages) & 1u);
      int c, r;
      box_at(j, c, r);
      for (int k = 1; k <= p.W - p.skip_self; ++k) {  // peers first, own inbox last
        const int d = (p.self + k) % p.W;
        tma_store_2d(&maps.dst[d], push_smem + st * box_bytes, c_dst + c, mb * BM + r);
      }
      bulk_commit();
      ++consumed;
      if (next < nbox) {
        bulk_wait_read<1>();  // box j - 1's stores have read their stage
        load_next();
      }
    }
    bulk_wait_all();             // this m-block's stores are complete
    fence_proxy_async_global();  // async-proxy writes before the generic release
    if (p.local) __threadfence();  // every inbox on this device: gpu scope suffices
    else __threadfence_system();
    for (int k = 1; k <= p.W; ++k) {
      const int d = (p.self + k) % p.W;
      if (p.events[d]) p.events[d][(size_t(mb) * p.W + p.self) * 2] = globaltimer_ns();
      if (p.local) red_release_gpu(p.ready[d] + size_t(mb) * p.W + p.self, 1);
      else red_release_sys(p.ready[d] + size_t(mb) * p.W + p.self, 1);
    }
  }
  __threadfence();
  if (atomicAdd(&p.ctr[1], 1u) == gridDim.x - 1) {
    p.ctr[0] = 0;
    p.ctr[1] = 0;
    __threadfence();
  }
}

// ---- host ------------------------------------------------------------------------

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

CUtensorMapL2promotion l2_promotion() {
  if (const char* e = std::getenv("TFB_L2PROMO")) {
    switch (std::atoi(e)) {
      case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
      case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
      case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
      default: break;
    }
  }
  return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// 2-D bf16 map: `inner` contiguous elements per row, `outer` rows, row pitch
// `pitch_elems`; box {box_inner, box_outer}; 128-byte swizzle.
tf_status make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                   uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer, bool f32 = false,
                   bool swizzle = true) {
  EncodeFn enc = encode_fn();
  if (!enc) return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch_elems * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return TF_OK;
}

}  // namespace

// Launches the tensor-core GEMM for local rank r.  own: shard owner index
// for the shard map (-1 => every k-block from `inbox`).
static tf_status launch_gemm(World* w, int r, const tf_ag_shape& sh, const void* shard,
                             const void* inbox, const void* b, void* c, const uint64_t* ready,
                             uint64_t epoch, int own, int gather, const AgTcParams& proto,
                             cudaStream_t st, int board, unsigned grid_cap, const AgLayout& lay) {
  const int W = w->W;
  const size_t kw = sh.k / W;
  const size_t ldb = lay.ldb ? lay.ldb : sh.n, ldc = lay.ldc ? lay.ldc : sh.n;
  CUtensorMap mOwn{}, mInbox{}, mB{}, mC{};
  // C: 64-column x 32-row boxes, one per epilogue warp per store.
  TFB_CHECK(make_map(&mC, c, sh.n, sh.m, ldc, 64, 32));
  if (shard && proto.msharded) TFB_CHECK(make_map(&mOwn, shard, sh.k, sh.m / W, sh.k, BK, BM));
  else if (shard) TFB_CHECK(make_map(&mOwn, shard, kw, sh.m, kw, BK, BM));
  if (inbox) TFB_CHECK(make_map(&mInbox, inbox, sh.k, sh.m, sh.k, BK, BM));
  if (!shard) mOwn = mInbox;
  if (!inbox) mInbox = mOwn;
  TFB_CHECK(make_map(&mB, b, sh.n, sh.k, ldb, 64, BK));
  AgTcParams p = proto;
  p.M = int(sh.m);
  p.N = int(sh.n);
  p.K = int(sh.k);
  p.kw = int(kw);
  p.W = W;
  p.own = own;
  p.num_m = int((sh.m + BM - 1) / BM);
  p.kb_total = int(sh.k / BK);
  p.kbw = int(kw / BK);
  p.C = static_cast<__nv_bfloat16*>(c);
  p.ready = ready;
  p.epoch = epoch;
  p.gather = gather;
  p.watchdog_ns = w->watchdog_ns;
  p.err = w->err_of(r);
  p.board = board;
  if (const char* e = std::getenv("TFB_DEBUG")) p.dbg = std::atoi(e);
  if (const char* e = std::getenv("TFB_L2HINT")) p.l2hint = std::atoi(e);
  p.one_producer = std::getenv("TFB_ONE_PRODUCER") ? 1 : 0;
  p.xchg_lsu = std::getenv("TFB_SPLITK_LSU") ? 1 : 0;
  const int dev = w->ranks[r].device;
  cudaSetDevice(dev);
  // Kernel shapes: CTA pairs (cta_group::2) with 256 x 512 tiles whenever
  // there are two 128-row blocks to pair; 256 x 256 pair tiles when that
  // fills the SMs better (skinny M); single CTAs (128 x 256) for M <= 128.
  struct Shape {
    int CG, NH;
    void (*kern)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, AgTcParams);
    size_t smem;
    int id;
  };
  const Shape shapes[4] = {
      {1, 1, ag_gemm_sm100_kernel<1, 1>, Cfg<1, 1>::SMEM, 0},
      {2, 2, ag_gemm_sm100_kernel<2, 2>, Cfg<2, 2>::SMEM, 1},
      {2, 1, ag_gemm_sm100_kernel<2, 1>, Cfg<2, 1>::SMEM, 2},
      {2, 1, ag_gemm_sm100_kernel<2, 1, 128>, Cfg<2, 1, 128>::SMEM, 3},  // narrow, 128-deep k-blocks
  };
  // Skinny M: too few tiles to occupy the SMs -> split K across a cluster
  // of S CTAs (pairs) per tile, reduced in-kernel through DSMEM in
  // ascending split order.  S is a power of two (it divides the 128 rows a
  // CTA reduces), CG * S <= 8 (portable cluster), >= 4 k-blocks per split,
  // and every cluster resident in one wave (a cluster is co-scheduled
  // inside one GPC).  BASELINE config 5's low end.
  auto plan = [&](const Shape& shp, int& tiles, int& num_n, int& ks) -> tf_status {
    num_n = int((sh.n + 256 * shp.NH - 1) / (256 * shp.NH));
    tiles = ((p.num_m + shp.CG - 1) / shp.CG) * num_n;
    const unsigned busy = unsigned(tiles) * shp.CG;
    ks = 1;
    if (busy * 2 <= grid_cap)
      while (ks * 2 * busy <= grid_cap && ks * 2 * shp.CG <= 8 && ks * 2 * 4 <= p.kb_total) ks *= 2;
    if (const char* e = std::getenv("TFB_KSPLIT")) {
      const int want = std::max(1, std::atoi(e));
      ks = 1;
      while (ks * 2 <= want && ks * 2 * shp.CG <= 8 && ks * 2 * 4 <= p.kb_total) ks *= 2;
    }
    if (!lay.split_k) ks = 1;
    while (ks > 1) {
      // Per (shape, split, device) occupancy cache; atomics so concurrent
      // worlds on other host threads never race on it (a stale read only
      // recomputes the same value).
      static std::atomic<int> max_active[4][9][16];
      std::atomic<int>& slot = max_active[shp.id][ks][dev & 15];
      int ma = slot.load(std::memory_order_relaxed);
      if (ma == 0) {
        TFB_CUDA(cudaFuncSetAttribute(shp.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shp.smem)));
        cudaLaunchConfig_t qc{};
        qc.gridDim = dim3(unsigned(shp.CG * ks));
        qc.blockDim = dim3(NUM_THREADS);
        qc.dynamicSmemBytes = shp.smem;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = unsigned(shp.CG * ks);
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.attrs = qa;
        qc.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&ma, shp.kern, &qc) != cudaSuccess || ma < 1) {
          cudaGetLastError();
          ma = -1;
        }
        slot.store(ma, std::memory_order_relaxed);
      }
      if (ma > 0 && unsigned(tiles) <= unsigned(ma)) break;
      if (std::getenv("TFB_KSPLIT_FORCE")) break;
      ks /= 2;
    }
    return TF_OK;
  };
  const Shape* shp = &shapes[(p.num_m >= 2 && !(p.dbg & 8)) ? 1 : 0];
  int tiles = 0, num_n = 0, ks = 1;
  TFB_CHECK(plan(*shp, tiles, num_n, ks));
  if (shp->CG == 2 && std::getenv("TFB_FORCE_NARROW")) {
    shp = &shapes[2];
    TFB_CHECK(plan(*shp, tiles, num_n, ks));
  } else if (shp->CG == 2 && !std::getenv("TFB_NO_NARROW")) {
    int t2, n2, k2;
    TFB_CHECK(plan(shapes[2], t2, n2, k2));
    // Narrow pair tiles only when the wide ones leave a quarter of the SMs
    // idle and the narrow ones fit one wave (M = 768: 96 narrow tiles on 74
    // pairs ran 148 us vs 89 us for 48 wide tiles, tools/skinny_ab.py).
    if (unsigned(tiles * ks * 2) * 4 < grid_cap * 3 && t2 * k2 > tiles * ks &&
        unsigned(t2 * k2 * 2) <= grid_cap) {
      shp = &shapes[2];
      tiles = t2;
      num_n = n2;
      ks = k2;
    }
  }
  // Whole-K plans with a partial last round: compare rounds x tile time
  // across the three tile shapes (tile times relative to a 256 x 512 pair
  // tile, measured at K = N = 8192: 256 x 256 pairs 0.72, 128 x 256 CTAs
  // 0.77).  M = 1152: 80 wide tiles on 74 pairs run two rounds (162 us),
  // 288 single-CTA tiles two nearly full ones (125 us; cuBLAS 122).
  if (shp->CG == 2 && ks == 1 && !(p.dbg & 8) && !std::getenv("TFB_NO_NARROW") && !std::getenv("TFB_FORCE_NARROW")) {
    auto rounds = [](long items, long slots) { return double((items + slots - 1) / slots); };
    const long pairs = long(grid_cap / 2);
    double best = rounds(long(tiles), pairs) * (shp->NH == 2 ? 1.0 : 0.72);
    const Shape* pick = shp;
    int t0, n0, k0;
    TFB_CHECK(plan(shapes[0], t0, n0, k0));
    if (k0 == 1 && rounds(t0, long(grid_cap)) * 0.77 < best * 0.95) {
      best = rounds(t0, long(grid_cap)) * 0.77;
      pick = &shapes[0];
    }
    if (shp->NH == 2) {
      int t2, n2, k2;
      TFB_CHECK(plan(shapes[2], t2, n2, k2));
      if (k2 == 1 && rounds(t2, pairs) * 0.72 < best * 0.95) {
        best = rounds(t2, pairs) * 0.72;
        pick = &shapes[2];
      }
    }
    if (pick != shp) {
      shp = pick;
      TFB_CHECK(plan(*shp, tiles, num_n, ks));
    }
  }
  // Narrow pair tiles take 128-deep k-blocks when every owner band is a
  // whole number of them: their k-block is paced by a ~560-cycle producer /
  // MMA ring round, not by its 4 MMAs (TFB_DEBUG 8192 cadence), so half the
  // rounds per FLOP (profiles/r2_skinny_analysis.md).  TFB_BK64 keeps 64.
  int bk = 64;
  if (shp->id == 2 && (p.msharded ? sh.k % 128 == 0 : kw % 128 == 0) && !std::getenv("TFB_BK64")) {
    const int kb64 = p.kb_total, kbw64 = p.kbw;
    p.kb_total = int(sh.k / 128);
    p.kbw = int(kw / 128);
    int t3, n3, k3;
    TFB_CHECK(plan(shapes[3], t3, n3, k3));
    if (t3 == tiles && k3 == ks) {
      shp = &shapes[3];
      bk = 128;
      TFB_CHECK(make_map(&mB, b, sh.n, sh.k, ldb, 64, 128));
    } else {  // the deeper k-block would change the split: keep 64
      p.kb_total = kb64;
      p.kbw = kbw64;
    }
  }
  const int CG = shp->CG;
  p.num_n = num_n;
  p.mt_rot = (p.msharded && own >= 0) ? (own * p.mpr / CG) % ((p.num_m + CG - 1) / CG) : 0;
  p.num_tiles = tiles;
  p.ksplit = ks;
  p.full_items = tiles * ks;
  p.q_tail = 1;
  p.total_items = tiles * ks;
  if (std::getenv("TFB_KSPLIT_VERBOSE"))
    std::fprintf(stderr, "[ag] m=%zu n=%zu k=%zu CG=%d NH=%d BK=%d tiles=%d ksplit=%d\n", sh.m, sh.n, sh.k, CG,
                 shp->NH, bk, tiles, ks);
  p.ldc = int(ldc);
  auto kern = shp->kern;
  const size_t smem = shp->smem;
  static std::atomic<bool> attr_set[4][64];  // idempotent attribute, set once per (shape, device)
  if (!attr_set[shp->id][dev & 63].load(std::memory_order_acquire)) {
    TFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_set[shp->id][dev & 63].store(true, std::memory_order_release);
  }
  const unsigned pair_tiles = unsigned((p.num_m + CG - 1) / CG) * unsigned(p.num_n) * unsigned(p.ksplit);
  if (const char* e = std::getenv("TFB_GRID")) grid_cap = std::min(grid_cap, unsigned(std::atoi(e)));
  unsigned grid = std::min(pair_tiles * CG, grid_cap / CG * CG);
  grid = std::max(grid, unsigned(CG));
  if (p.ksplit > 1) grid = pair_tiles * CG;  // exactly one item per CTA (the reduction aliases its smem)
  p.ws = nullptr;
  // Split-K partials are summed straight from the siblings' smem (DSMEM)
  // since the sum loop was specialised on S (M = 128 / 256: 30.0 / 37.2 us
  // vs 32.5 / 38.1 through L2 bulk copies, tools/skinny_ab.py; before it the
  // branchy generic loop made the L2 route the faster one).  The L2
  // exchange (TFB_SPLITK_L2) stays as an A/B path -- bitwise equal.
  if (p.ksplit > 1 && std::getenv("TFB_SPLITK_L2") && !std::getenv("TFB_SPLITK_DSMEM")) {
    void* ws = nullptr;
    TFB_CHECK(ensure_scratch(w, r, 2, size_t(grid) * shp->NH * BM * 1024, &ws));
    p.ws = static_cast<uint8_t*>(ws);
  }
  // Last-wave balance (CTA pairs, whole-K tiles): when the tiles leave a
  // partial last round, cut its tiles into 2 or 4 column slices so that
  // round runs on (nearly) every pair for a half or quarter of a tile time.
  if (CG == 2 && p.ksplit == 1 && !std::getenv("TFB_NO_TAIL_SPLIT")) {
    const int ncl = int(grid) / CG, T = p.num_tiles;
    const int fr = T / ncl, rem = T % ncl;
    if (fr >= 1 && rem > 0) {
      // Off by default: a column slice ran as long as a whole tile at every
      // shape measured (M = 1152 / 4096, K = N = 8192: 172 / 410 us with 4
      // slices, 162 / 395 whole; config 2 within noise) -- the slice's
      // k-block chain, not its MMA width, sets its time.  TFB_TAIL_Q = 2 / 4
      // turns it on.
      int q = 1;
      if (const char* e = std::getenv("TFB_TAIL_Q")) q = std::max(1, std::atoi(e));
      while (q > 1 && rem * q > ncl) q /= 2;
      if (q > 1) {
        p.full_items = fr * ncl;
        p.q_tail = q;
        p.total_items = p.full_items + rem * q;
      }
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG * p.ksplit;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1 + unsigned(pdl_attrs(&attr[1]));
  {
    // TFB_GROUP_M (profiling knob) lives in a __constant__ per device.
    static std::atomic<int> last_gm[64];
    int gm = 0;
    if (const char* e = std::getenv("TFB_GROUP_M")) gm = std::atoi(e);
    if (last_gm[dev & 63].exchange(gm) != gm) TFB_CUDA(cudaMemcpyToSymbol(g_group_m, &gm, sizeof(int)));
  }
  // B as 4-D (64 columns, K rows, 4 chunks of a 256-column group, N/256
  // groups): one box (64, BK, CPH, NH) is a CTA's whole B stage.
  CUtensorMap mB4{};
  p.b4 = 0;
  if (sh.n % 256 == 0 && !std::getenv("TFB_NO_B4")) {
    EncodeFn enc = encode_fn();
    cuuint64_t dims[4] = {64, sh.k, 4, sh.n / 256};
    cuuint64_t strides[3] = {ldb * 2, 128, 512};
    cuuint32_t box[4] = {64, uint32_t(bk), uint32_t(4 / CG), uint32_t(shp->NH)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (enc && enc(&mB4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(b), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      p.b4 = 1;
  }
  TFB_CUDA(cudaLaunchKernelEx(&cfg, kern, mOwn, mInbox, mB, mC, mB4, p));
  ++w->launches;
  return TF_OK;
}

// GEMM grid cap per rank for the push schedule: n ranks on one device share
// its SMs with their n producers (an even number of CTAs: pairs).
static unsigned push_cap(unsigned sms, unsigned push_ctas, unsigned n) {
  if (n == 0) n = 1;
  const unsigned left = sms > push_ctas * n ? sms - push_ctas * n : 2;
  return std::max(2u, left / n / 2 * 2);
}

tf_status ag_bf16_run(World* w, tf_ag_variant variant, const tf_ag_shape& sh, void* const* a_shard,
                      const void* const* b, void* const* c, void* const* gathered,
                      const std::vector<cudaStream_t>& streams, const AgLayout& lay) {
  const int W = w->W;
  const size_t m = sh.m, n = sh.n, k = sh.k, kw = k / W;
  const bool msh = sh.shard == TF_SHARD_M && W > 1;  // W = 1: both layouts are the whole A
  const size_t mr = m / size_t(W);                    // M-sharded: rows per rank
  if (msh ? k % BK != 0 : kw % BK != 0)
    return set_error(TF_ERR_SHAPE, msh ? "ag_gemm(bf16, M-sharded): k = " + std::to_string(k) +
                                             " must be a multiple of 64"
                                       : "ag_gemm(bf16): k / world_size = " + std::to_string(kw) +
                                             " must be a multiple of 64");
  if (n % 8 != 0) return set_error(TF_ERR_SHAPE, "ag_gemm(bf16): n must be a multiple of 8");
  if (m > (size_t(1) << 31) || n > (size_t(1) << 31) || k > (size_t(1) << 31))
    return set_error(TF_ERR_SHAPE, "ag_gemm(bf16): dimensions must fit in int32");
  const int num_m = int((m + BM - 1) / BM);
  const unsigned sms = unsigned(w->sm_count);

  if (!lay.inbox_complete) w->record_ag(m, kw, 2, msh);
  if (W == 1) {
    // No exchange: the fused kernel degenerates to the GEMM over the shard.
    if (!w->ranks[0].local) return TF_OK;
    if (!lay.inbox_complete) w->ag_src[0][0] = {a_shard[0], kw};
    AgTcParams proto{};
    TFB_CHECK(launch_skew(w, 0, streams[0]));
    TFB_CHECK(launch_gemm(w, 0, sh, a_shard[0], nullptr, b[0], c[0], nullptr, 0, 0, 0, proto,
                          streams[0], -1, sms, lay));
    if (gathered && gathered[0])
      TFB_CUDA(cudaMemcpyAsync(gathered[0], a_shard[0], m * k * 2, cudaMemcpyDefault, streams[0]));
    return TF_OK;
  }

  // Gathered operand per rank: caller's buffer, else the heap inbox
  // (double-buffered by epoch parity for PUSH, where peers write into it).
  size_t inbox_off = 0, ctr_off = 0;
  TFB_CHECK(heap_get(w, "ag.inbox.bf16[" + std::to_string(m * k) + "]", 2 * m * k * 2, &inbox_off));
  TFB_CHECK(heap_get(w, "ag.ctr", 256, &ctr_off));
  BoardEntry rb;
  // Only the signalling schedules (pull, push) advance the ready board's
  // epoch; BASELINE never touches it (every rank/process must agree on e).
  if (variant == TF_AG_BASELINE || lay.inbox_complete) {
    const std::string bname = "ag.ready[" + std::to_string(num_m) + "x" + std::to_string(W) + "]";
    TFB_CHECK(board_get(w, bname, num_m, W, &rb));
    rb.epoch = w->boards[bname].epoch;
  } else {
    TFB_CHECK(board_next_epoch(w, "ag.ready", num_m, W, &rb));
    w->ag_flags = FlagSnapshot{w->board_names[rb.id], size_t(num_m) * W, rb.epoch};
  }
  const int parity = int(rb.epoch & 1);
  auto inbox_of = [&](int r) -> __nv_bfloat16* {
    if (gathered && gathered[r]) return static_cast<__nv_bfloat16*>(gathered[r]);
    return reinterpret_cast<__nv_bfloat16*>(w->ptr(r, inbox_off)) + size_t(parity) * m * k;
  };
  // PUSH on the TMA producer (W <= 8): peers' inboxes only -- like pull, a
  // rank's own block is read in place from its shard (unless the caller
  // asked for the gathered operand in its own buffer).
  const bool tma_push = variant == TF_AG_PUSH && W <= kPushMaxW && !std::getenv("TFB_PUSH_LSU");
  if (!lay.inbox_complete)
    for (int r = 0; r < W; ++r)
      for (int s = 0; s < W; ++s)
        w->ag_src[r][s] = ((variant == TF_AG_PULL || tma_push) && s == r && !(gathered && gathered[r]))
                              ? World::AgBlock{a_shard[r], msh ? k : kw}  // read in place by the TMA producer
                              : World::AgBlock{inbox_of(r) + (msh ? size_t(s) * mr * k : size_t(s) * kw), k};
  auto ready_of = [&](int r) { return reinterpret_cast<uint64_t*>(w->ptr(r, rb.offset)); };
  auto ctr_of = [&](int r, int slot) { return reinterpret_cast<unsigned int*>(w->ptr(r, ctr_off)) + slot * 4; };
  // Event log (tf_world_set_events; debug, untimed): per (m-block, source)
  // the %globaltimer of the chunk's store and of its first consumer load.
  // Filled with ~0 synchronously before anything launches: a peer's
  // producer may record into this rank's log as soon as it runs.
  size_t ev_off = 0;
  const bool events = w->events && variant != TF_AG_BASELINE && !lay.inbox_complete;
  if (events) {
    const size_t bytes = size_t(num_m) * W * 2 * sizeof(unsigned long long);
    TFB_CHECK(heap_get(w, "ag.events[" + std::to_string(num_m) + "x" + std::to_string(W) + "]", bytes, &ev_off));
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      cudaSetDevice(w->ranks[r].device);
      TFB_CUDA(cudaDeviceSynchronize());
      TFB_CUDA(cudaMemset(w->ptr(r, ev_off), 0xFF, bytes));
      TFB_CUDA(cudaDeviceSynchronize());
    }
    w->ag_events_off = ev_off;
    w->ag_events_n = size_t(num_m) * W * 2;
  }
  auto events_of = [&](int r) -> unsigned long long* {
    return events ? reinterpret_cast<unsigned long long*>(w->ptr(r, ev_off)) : nullptr;
  };
  // Every schedule lands the gathered operand in HBM once per rank (PULL via
  // the gather warps; the reference's pull re-fetches tiles instead).
  if (lay.inbox_complete) {
    // The inbox already holds the gathered A (an earlier run on these
    // streams): the GEMM alone, ungated, own k-range from the shard.
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      AgTcParams proto{};
      // Same k order as the schedule that gathered (BASELINE: ascending,
      // pull/push: own shard first), so every slab matches a one-shot run.
      const int own = variant == TF_AG_BASELINE ? -1 : r;
      TFB_CHECK(launch_gemm(w, r, sh, own < 0 ? nullptr : a_shard[r], inbox_of(r), b[r], c[r], nullptr, 0,
                            own, 0, proto, streams[r], -1, sms, lay));
    }
    return TF_OK;
  }
  for (int r = 0; r < W; ++r)
    if (w->ranks[r].local) w->stage(r, m * k * 2);

  if (variant == TF_AG_BASELINE) {
    TFB_CHECK(world_barrier(w, streams));
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      cudaSetDevice(w->ranks[r].device);
      for (int s = 0; s < W; ++s) {
        if (msh)  // row band s: one contiguous copy
          TFB_CUDA(cudaMemcpyAsync(inbox_of(r) + size_t(s) * mr * k, a_shard[s], mr * k * 2, cudaMemcpyDefault,
                                   streams[r]));
        else
          TFB_CUDA(cudaMemcpy2DAsync(inbox_of(r) + size_t(s) * kw, k * 2, a_shard[s], kw * 2, kw * 2, m,
                                     cudaMemcpyDefault, streams[r]));
      }
    }
    TFB_CHECK(world_barrier(w, streams));
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      AgTcParams proto{};
      TFB_CHECK(launch_skew(w, r, streams[r]));
      TFB_CHECK(launch_gemm(w, r, sh, nullptr, inbox_of(r), b[r], c[r], nullptr, 0, -1, 0, proto,
                            streams[r], -1, sms, lay));
    }
    return TF_OK;
  }

  if (variant == TF_AG_PULL) {
    for (int r = 0; r < W; ++r) {
      if (!w->ranks[r].local) continue;
      AgTcParams proto{};
      for (int s = 0; s < W; ++s) proto.peer_shard[s] = static_cast<const __nv_bfloat16*>(a_shard[s]);
      proto.inbox = inbox_of(r);
      proto.gather_own = (gathered && gathered[r]) ? 1 : 0;
      proto.msharded = msh;
      proto.mpr = int(mr / BM);
      proto.ready_w = ready_of(r);
      proto.ctr = ctr_of(r, 0);
      proto.events = events_of(r);
      TFB_CHECK(launch_skew(w, r, streams[r]));
      TFB_CHECK(launch_gemm(w, r, sh, a_shard[r], inbox_of(r), b[r], c[r], ready_of(r), rb.epoch, r,
                            1, proto, streams[r], rb.id, sms, lay));
    }
    return TF_OK;
  }

  // PUSH into caller-supplied gathered buffers (single, not parity-buffered
  // like the internal inbox): a world barrier first, so no peer stores into
  // a buffer whose owner may still be reading it from its previous run.
  bool caller = false;
  for (int r = 0; r < W && gathered; ++r) caller |= gathered[r] != nullptr;
  if (caller) TFB_CHECK(world_barrier(w, streams));
  // PUSH: producers first on the side streams (they never wait), then the
  // gated GEMMs with a few SMs left for the producers.  Ranks sharing a
  // device (loopback) split its SMs: every rank's GEMM and producer CTAs
  // must fit at once, or GEMM CTAs spinning on flags could hold every SM
  // while a peer's producer waits for one.
  std::map<int, unsigned> per_dev;
  for (int r = 0; r < W; ++r)
    if (w->ranks[r].local) ++per_dev[w->ranks[r].device];
  // 16 producer CTAs per device, split among the ranks sharing it.
  // TMA producer (W <= 8): a few one-warp CTAs per device; the register-copy
  // producer (TFB_PUSH_LSU, or W > 8): 16.
  // Producer CTAs: TMA, 4 per rank (a TMA store engine moves ~62 GB/s per SM,
  // tools/micro_tma_store.cu; a rank's GEMM consumes its A at well under
  // 200 GB/s, so 4 keep ahead of it -- loopback W = 8 config 2: 8 / 16 / 24
  // / 32 CTAs per device 5378 / 4062 / 3697 / 3580 us); register copy, 16 per
  // device.  TFB_PUSH_CTAS: CTAs per device.
  unsigned push_total = 0;
  if (const char* e = std::getenv("TFB_PUSH_CTAS")) push_total = unsigned(std::max(1, std::atoi(e)));
  auto push_ctas_of = [&](int r) {
    const unsigned n = per_dev[w->ranks[r].device];
    if (tma_push) return push_total ? std::max(1u, push_total / n) : 4u;
    return std::max(2u, (push_total ? push_total : 16u) / n);
  };
  for (int r = 0; r < W; ++r) {
    if (!w->ranks[r].local) continue;
    cudaSetDevice(w->ranks[r].device);
    cudaEvent_t ev;
    TFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TFB_CUDA(cudaEventRecord(ev, streams[r]));
    TFB_CUDA(cudaStreamWaitEvent(w->ranks[r].side, ev, 0));
    cudaEventDestroy(ev);
    PushParams pp{};
    pp.shard = static_cast<const __nv_bfloat16*>(a_shard[r]);
    for (int d = 0; d < W; ++d) {
      pp.inbox[d] = inbox_of(d);
      pp.ready[d] = ready_of(d);
    }
    pp.M = int(m);
    pp.K = int(k);
    pp.kw = int(kw);
    pp.W = W;
    pp.self = r;
    pp.num_m = num_m;
    pp.msharded = msh;
    pp.mpr = int(mr / BM);
    pp.ctr = ctr_of(r, 1);
    for (int d = 0; d < W; ++d) pp.events[d] = events_of(d);
    if (tma_push) {
      PushMaps maps{};
      PushTmaParams tp{};
      const size_t cols = msh ? k : kw;
      tp.box_c = cols % 256 == 0 ? 256 : cols % 128 == 0 ? 128 : 64;
      tp.box_r = std::min(BM, 16384 / tp.box_c);
      tp.cols = int(cols);
      TFB_CHECK(make_map(&maps.src, a_shard[r], cols, msh ? mr : m, cols, uint32_t(tp.box_c), uint32_t(tp.box_r),
                         false, false));
      for (int d = 0; d < W; ++d) {
        TFB_CHECK(make_map(&maps.dst[d], inbox_of(d), k, m, k, uint32_t(tp.box_c), uint32_t(tp.box_r), false, false));
        tp.ready[d] = ready_of(d);
        tp.events[d] = events_of(d);
      }
      tp.W = W;
      tp.self = r;
      tp.nmb = msh ? int(mr / BM) : num_m;
      tp.msharded = msh;
      tp.mpr = int(mr / BM);
      tp.M = int(m);
      tp.local = 1;
      for (int d = 0; d < W; ++d)
        if (!w->ranks[d].local || w->ranks[d].device != w->ranks[r].device) tp.local = 0;
      if (std::getenv("TFB_PUSH_SYS")) tp.local = 0;
      tp.skip_self = !(gathered && gathered[r]);
      tp.ctr = ctr_of(r, 1);
      const int smem = kPushStages * tp.box_c * tp.box_r * 2;
      static std::atomic<bool> push_attr[64];
      if (!push_attr[w->ranks[r].device & 63].exchange(true))
        TFB_CUDA(cudaFuncSetAttribute(ag_push_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kPushStages * 32768));
      ag_push_tma_kernel<<<push_ctas_of(r), 32, smem, w->ranks[r].side>>>(maps, tp);
    } else {
      ag_push_kernel<<<push_ctas_of(r), 512, 0, w->ranks[r].side>>>(pp);
    }
    TFB_CUDA(cudaGetLastError());
    ++w->launches;
  }
  for (int r = 0; r < W; ++r) {
    if (!w->ranks[r].local) continue;
    AgTcParams proto{};
    proto.events = events_of(r);
    proto.msharded = msh;
    proto.mpr = int(mr / BM);
    TFB_CHECK(launch_skew(w, r, streams[r]));
    TFB_CHECK(launch_gemm(w, r, sh, a_shard[r], inbox_of(r), b[r], c[r], ready_of(r), rb.epoch, r, 0,
                          proto, streams[r], rb.id, push_cap(sms, push_ctas_of(r), per_dev[w->ranks[r].device]), lay));
    cudaEvent_t ev;
    TFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TFB_CUDA(cudaEventRecord(ev, w->ranks[r].side));
    TFB_CUDA(cudaStreamWaitEvent(streams[r], ev, 0));
    cudaEventDestroy(ev);
  }
  return TF_OK;
}

void ag_sm100_preload() {  // see ag_exact_preload
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, ag_gemm_sm100_kernel<1, 1>);
  cudaFuncGetAttributes(&a, ag_gemm_sm100_kernel<2, 2>);
  cudaFuncGetAttributes(&a, ag_gemm_sm100_kernel<2, 1>);
  cudaFuncGetAttributes(&a, ag_gemm_sm100_kernel<2, 1, 128>);
  cudaFuncGetAttributes(&a, ag_push_kernel);
}

}  // namespace tfb
