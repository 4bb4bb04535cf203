// world.hpp -- host-side world: ranks, per-rank streams, the symmetric heap
// registry, signal boards, epochs and the error record.  This is the B200
// form of the reference's World/RankCtx (fabric.hpp:253-692): a "rank" is a
// GPU (or, in a loopback world, a slice of one GPU's memory), a symmetric
// tensor is one bump allocation at the same offset in every rank's heap, and
// a signal board is a heap region of u64 counters.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "tilefabric_b200/tf_abi.h"

namespace tfb {

struct RankRes {
  int device = 0;
  char* heap = nullptr;       // base of this rank's heap, valid in this process
  bool local = false;         // launched by this process
  bool owns_heap = false;     // allocated (vs IPC-opened) here
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // producer stream (push variants)
  // Host-buffer runs (ag_host.cu): copy-engine streams and device operand
  // buffers, created on first use, grow-only.
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t legacy_ev = nullptr;  // order_after_legacy
  // [0] B / [1] C device operands of host-buffer runs, [2] split-K
  // workspace, [3] B / [4] C of the second host-run buffer set (W = 1)
  void* scratch[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t scratch_bytes[5] = {0, 0, 0, 0, 0};
  // Host-buffer runs of a one-rank world alternate two buffer sets so that
  // back-to-back calls on different streams overlap (ag_host.cu): per set,
  // the event after its last GEMM (B / shard free) and after its last C
  // read-back (C free).
  int host_par = 0;
  cudaEvent_t host_reads_done[2] = {nullptr, nullptr}, host_d2h_done[2] = {nullptr, nullptr};
};

struct HeapEntry {
  size_t offset = 0;
  size_t bytes = 0;
};

struct BoardEntry {
  int id = 0;
  int rows = 0;
  int slots = 0;
  size_t offset = 0;  // heap offset of the rows x slots u64 grid
  uint64_t epoch = 0; // completed-run count: a run waits for cells >= epoch
};

// Records the last push-style run's flag geometry for *_flag_counts.
struct FlagSnapshot {
  std::string board;
  size_t cells = 0;     // per rank
  uint64_t epoch = 0;   // value a completed run leaves in every cell
  // Device-epoch schedules: the epoch is read from the launch's cell
  // (heap offset dev_off, index dev_idx of the rank's device lead) -- it
  // advances in graph replays the host never sees.
  bool dev = false;
  size_t dev_off = 0;
  int dev_idx = 0;
};

struct World {
  int W = 0;
  bool ipc = false;
  int first_local = 0;
  int n_local = 0;
  double watchdog_secs = 10.0;
  uint64_t watchdog_ns = 10000000000ull;
  size_t heap_bytes = 0;
  size_t heap_used = 0;
  std::vector<RankRes> ranks;
  std::map<std::string, HeapEntry> heap;
  std::map<std::string, BoardEntry> boards;
  std::vector<std::string> board_names;  // id -> name
  // Error records in device memory, one per local device: cheap to poll
  // from spinning kernels; the host reads them after a sync.
  std::map<int, DevErr*> errs;
  uint64_t launches = 0;
  uint64_t tax_launch_base = 0;        // tf_tax_reset point
  std::vector<uint64_t> staged_bytes;  // per rank: bytes landed in staging/inbox tensors
  // Straggler model (WorldConfig::skew, fabric.hpp:59-62, 100-110): extra
  // delay at the start of the rank's first compute stage of every run.
  std::vector<uint64_t> skew_ns;
  uint64_t skew_of(int r) const { return skew_ns.empty() ? 0 : skew_ns[r]; }
  void stage(int r, uint64_t bytes) {
    if (staged_bytes.size() != size_t(W)) staged_bytes.assign(W, 0);
    staged_bytes[r] += bytes;
  }
  uint64_t barrier_epoch = 0;
  bool barrier_ready = false;     // tf.barrier board + its device pointer table written
  size_t barrier_table_off = 0;
  uint64_t ag_epoch = 0;
  uint64_t fd_epoch = 0;
  FlagSnapshot ag_flags, fd_flags;
  // Where the last AG run's gathered operand lives, per rank r and source
  // block s: (pointer to the block's first element, row pitch in elements)
  // -- the inbox/stage the GEMM consumed, or the owner's shard where the
  // schedule reads it in place (tf_ag_gathered).
  struct AgBlock {
    const void* p = nullptr;
    size_t pitch = 0;
  };
  std::vector<std::vector<AgBlock>> ag_src;
  size_t ag_m = 0, ag_kw = 0, ag_esz = 0;
  bool ag_msharded = false;  // blocks are row bands (TF_SHARD_M), else column bands
  void record_ag(size_t m, size_t kw, size_t esz, bool msharded = false) {
    ag_m = m;
    ag_kw = kw;
    ag_esz = esz;
    ag_msharded = msharded;
    ag_src.assign(W, std::vector<AgBlock>(W));
  }
  // Event log (tf_world_set_events): the last pull/push run's per-chunk
  // store / first-load timestamps, [num_m][W][2] u64 in every rank's heap.
  bool events = false;
  size_t ag_events_off = 0, ag_events_n = 0;
  size_t fd_events_off = 0, fd_events_n = 0;  // fused FD: [W src][G][2]
  // Named monotonic epochs for counters that live in the heap (tickets,
  // soak boards); cleared with the heap.
  std::map<std::string, uint64_t> epochs;
  int sm_count = 148;
  // Loopback: several ranks share one device.
  bool loopback = false;

  char* ptr(int rank, size_t offset) const { return ranks[rank].heap + offset; }
  DevErr* err_of(int r) const { return errs.at(ranks[r].device); }
  bool is_local(int r) const { return r >= first_local && r < first_local + n_local; }
};

// ---- status plumbing -----------------------------------------------------
tf_status set_error(tf_status s, const std::string& msg);
tf_status cuda_status(cudaError_t e, const char* what);
#define TFB_CUDA(call)                                              \
  do {                                                              \
    cudaError_t _e = (call);                                        \
    if (_e != cudaSuccess) return ::tfb::cuda_status(_e, #call);    \
  } while (0)
#define TFB_CHECK(call)                      \
  do {                                       \
    tf_status _s = (call);                   \
    if (_s != TF_OK) return _s;              \
  } while (0)

// Straggler delay (world.skew_ns[r] > 0): a one-thread %globaltimer sleep
// kernel ahead of rank r's compute on stream s.  Not counted as a launch:
// it stands in for the reference's precise_sleep inside ComputeScope
// (fabric.hpp:695-706).
tf_status launch_skew(World* w, int r, cudaStream_t s);

// Allocate the world barrier's board and per-rank cell table once, with
// synchronous copies, before a schedule launches anything: a first-call
// allocation (device sync / pageable copy) inside a schedule would
// serialize the ranks' streams and hide the barrier waits being measured.
tf_status ensure_barrier(World* w);

// Per-file kernel preloads, run for every local device at world creation.
void ag_exact_preload();
void ag_sm100_preload();
void fd_preload();

// Heap/board helpers used by the pattern implementations.
tf_status heap_get(World* w, const std::string& name, size_t bytes, size_t* offset);
tf_status board_get(World* w, const std::string& name, int rows, int slots, BoardEntry* out);
// Geometry-keyed board for a pattern run; returns it with its epoch bumped
// (monotonic counters: run e waits for >= e, fabric.hpp:515-517).
tf_status board_next_epoch(World* w, const std::string& base, int rows, int slots,
                           BoardEntry* out);
// Device-side world barrier over every rank (fabric.hpp:574-584): one tiny
// kernel per local rank, red.release.sys onto every rank's barrier cell,
// then an acquire spin on its own.
tf_status world_barrier(World* w, const std::vector<cudaStream_t>& streams, int only_rank = -1);
// Resolve caller streams (NULL -> world streams).
std::vector<cudaStream_t> resolve_streams(World* w, void* const* streams);
// For ranks driven on the world's own (non-blocking) streams: order them
// after everything already issued on the legacy default stream, where a
// caller typically produced the inputs (torch, cudaMemcpy, ...).
tf_status order_after_legacy(World* w, void* const* streams);
// Multi-rank schedules bake host state (flag epochs, board epochs) into
// their launches, so a captured graph would replay stale waits: refuse
// (TF_ERR_CONFIG) when W > 1 and any rank's stream is capturing.
tf_status refuse_multi_rank_capture(World* w, const std::vector<cudaStream_t>& s, const char* what);
// Launch attributes for the hot kernels: programmatic dependent launch
// unless TFB_NO_PDL is set (A/B).  Returns the number of attributes filled.
inline int pdl_attrs(cudaLaunchAttribute* a) {
  if (std::getenv("TFB_NO_PDL")) return 0;
  a->id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a->val.programmaticStreamSerializationAllowed = 1;
  return 1;
}

// Grow-only device scratch of rank r (slot < 5); first use allocates.
tf_status ensure_scratch(World* w, int r, int slot, size_t bytes, void** out);
// Wait for local streams and turn the device error record into a status.
tf_status sync_and_check(World* w, const std::vector<cudaStream_t>& streams);
tf_status check_record(World* w);

// Checks that [p, p+bytes) lies inside rank r's heap.
bool in_heap(const World* w, int r, const void* p, size_t bytes);

}  // namespace tfb

struct tf_world {
  tfb::World impl;
};
