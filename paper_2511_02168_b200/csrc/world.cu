// world.cu -- tf_world lifecycle, symmetric heap, signal boards, the device
// world barrier and the error-record -> tf_status mapping.
//
// Reference mapping (proj/include/tilefabric/):
//   tf_world_create      WorldConfig::validate + launch_world   fabric.hpp:71-96, 831-889
//   tf_heap_alloc        World::alloc_tensor                   fabric.hpp:276-317
//   tf_board_alloc       World::alloc_board                    fabric.hpp:319-350
//   tf_signal            RankCtx::atomic_signal                fabric.hpp:503-507
//   tf_wait_signal       RankCtx::wait_signal                  fabric.hpp:519-569
//   world_barrier        RankCtx::barrier / CentralBarrier     fabric.hpp:204-246, 574-584
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

#include "world.hpp"

namespace tfb {

static thread_local std::string g_last_error;

tf_status set_error(tf_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

tf_status cuda_status(cudaError_t e, const char* what) {
  return set_error(TF_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                                    cudaGetErrorString(e) + ") in " + what);
}

static double default_watchdog_secs() {
  // common.hpp:97-107
  if (const char* env = std::getenv("TILEFABRIC_WATCHDOG_SECS")) {
    char* end = nullptr;
    double s = std::strtod(env, &end);
    if (end != env && s > 0.0) return s;
  }
  return 10.0;
}

bool in_heap(const World* w, int r, const void* p, size_t bytes) {
  const char* c = static_cast<const char*>(p);
  const char* base = w->ranks[r].heap;
  return c >= base && c + bytes <= base + w->heap_bytes;
}

tf_status heap_get(World* w, const std::string& name, size_t bytes, size_t* offset) {
  if (name.empty()) return set_error(TF_ERR_CONFIG, "alloc_symmetric: empty tensor name");
  if (bytes == 0)
    return set_error(TF_ERR_CONFIG, "alloc_symmetric(\"" + name + "\"): zero-size dimension");
  auto it = w->heap.find(name);
  if (it != w->heap.end()) {
    if (it->second.bytes != bytes)
      return set_error(TF_ERR_CONFIG,
                       "alloc_symmetric(\"" + name + "\"): shape/staging mismatch across ranks");
    *offset = it->second.offset;
    return TF_OK;
  }
  const size_t align = 4096;
  size_t off = (w->heap_used + align - 1) / align * align;
  if (off + bytes > w->heap_bytes)
    return set_error(TF_ERR_CONFIG, "alloc_symmetric(\"" + name + "\"): symmetric heap exhausted (" +
                                        std::to_string(off + bytes) + " > " +
                                        std::to_string(w->heap_bytes) + " bytes per rank)");
  // Zero-filled by construction (fabric.hpp:142-144): the heap is zeroed
  // (and synchronized) when the world is created or reset, and bump
  // allocations never reuse memory.  No memset here: in a multi-process
  // world a peer that allocated its copy first may already be storing into
  // this rank's new region (pushes, flags), and a late zero-fill would wipe
  // those stores (a lost flag = a deadlock; found with two processes).
  w->heap_used = off + bytes;
  w->heap[name] = HeapEntry{off, bytes};
  *offset = off;
  return TF_OK;
}

tf_status board_get(World* w, const std::string& name, int rows, int slots, BoardEntry* out) {
  if (name.empty()) return set_error(TF_ERR_CONFIG, "alloc_board: empty board name");
  if (rows < 1 || slots < 1)
    return set_error(TF_ERR_CONFIG, "alloc_board(\"" + name + "\"): rows and slots must be >= 1");
  auto it = w->boards.find(name);
  if (it != w->boards.end()) {
    if (it->second.rows != rows || it->second.slots != slots)
      return set_error(TF_ERR_CONFIG, "alloc_board(\"" + name + "\"): grid mismatch across ranks");
    *out = it->second;
    return TF_OK;
  }
  BoardEntry b;
  b.id = static_cast<int>(w->board_names.size());
  b.rows = rows;
  b.slots = slots;
  TFB_CHECK(heap_get(w, "board:" + name, sizeof(uint64_t) * size_t(rows) * size_t(slots), &b.offset));
  w->boards[name] = b;
  w->board_names.push_back(name);
  *out = b;
  return TF_OK;
}

tf_status board_next_epoch(World* w, const std::string& base, int rows, int slots,
                           BoardEntry* out) {
  const std::string name = base + "[" + std::to_string(rows) + "x" + std::to_string(slots) + "]";
  TFB_CHECK(board_get(w, name, rows, slots, out));
  out->epoch = ++w->boards[name].epoch;
  return TF_OK;
}

std::vector<cudaStream_t> resolve_streams(World* w, void* const* streams) {
  std::vector<cudaStream_t> s(w->W, nullptr);
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local) continue;
    s[r] = (streams && streams[r]) ? static_cast<cudaStream_t>(streams[r]) : w->ranks[r].stream;
  }
  return s;
}

tf_status ensure_scratch(World* w, int r, int slot, size_t bytes, void** out) {
  RankRes& rr = w->ranks[r];
  if (rr.scratch_bytes[slot] < bytes) {
    cudaSetDevice(rr.device);
    if (rr.scratch[slot]) {
      TFB_CUDA(cudaDeviceSynchronize());
      TFB_CUDA(cudaFree(rr.scratch[slot]));
      rr.scratch[slot] = nullptr;
      rr.scratch_bytes[slot] = 0;
    }
    TFB_CUDA(cudaMalloc(&rr.scratch[slot], bytes));
    rr.scratch_bytes[slot] = bytes;
  }
  *out = rr.scratch[slot];
  return TF_OK;
}

tf_status refuse_multi_rank_capture(World* w, const std::vector<cudaStream_t>& s, const char* what) {
  if (w->W == 1) return TF_OK;
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local) continue;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s[r], &cs) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (cs != cudaStreamCaptureStatusNone)
      return set_error(TF_ERR_CONFIG, std::string(what) +
                                          ": graph capture of a multi-rank schedule is unsupported (its flag "
                                          "epochs are host state; a replay would wait on stale values)");
  }
  return TF_OK;
}

tf_status order_after_legacy(World* w, void* const* streams) {
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local || (streams && streams[r])) continue;
    RankRes& rr = w->ranks[r];
    cudaSetDevice(rr.device);
    if (!rr.legacy_ev) TFB_CUDA(cudaEventCreateWithFlags(&rr.legacy_ev, cudaEventDisableTiming));
    TFB_CUDA(cudaEventRecord(rr.legacy_ev, 0));
    TFB_CUDA(cudaStreamWaitEvent(rr.stream, rr.legacy_ev, 0));
  }
  return TF_OK;
}

tf_status check_record(World* w) {
  DevErr rec{};
  DevErr* dev_rec = nullptr;
  for (auto& kv : w->errs) {
    cudaSetDevice(kv.first);
    TFB_CUDA(cudaMemcpy(&rec, kv.second, sizeof(DevErr), cudaMemcpyDeviceToHost));
    if (rec.code != 0) {
      dev_rec = kv.second;
      break;
    }
  }
  if (!dev_rec) return TF_OK;
  DevErr* e = &rec;
  const int code = rec.code;
  std::string msg;
  const std::string rank = "rank " + std::to_string(e->rank) + ": ";
  const std::string board = (e->board >= 0 && e->board < (int)w->board_names.size())
                                ? w->board_names[e->board]
                                : std::string("?");
  switch (e->kind) {
    case kWaitSignal:
      msg = rank + "wait_signal(board \"" + board + "\", row " + std::to_string(e->row) +
            ", slot " + std::to_string(e->slot) + ") on rank " + std::to_string(e->rank) +
            ": expected >= " + std::to_string(e->expected) + ", observed " +
            std::to_string(e->observed) + " within the watchdog";
      break;
    case kWaitBarrier: {
      // observed counts arrivals of this generation (fabric.hpp:227-230).
      msg = rank + "barrier generation " + std::to_string(e->aux) + ": only " +
            std::to_string(e->observed) + " of " + std::to_string(e->expected) +
            " ranks arrived within the watchdog";
      break;
    }
    case kNumeric:
      msg = rank + "attention_partial: non-finite score at head " +
            std::to_string(e->aux >> 32) + ", position " + std::to_string(e->aux & 0xffffffffu);
      break;
    case kPage:
      msg = rank + "flash_decode (paged KV): block table entry " + std::to_string(e->observed) +
            " at batch " + std::to_string(e->row) + ", page slot " + std::to_string(e->slot) +
            " is outside the pool of " + std::to_string(e->expected) + " pages";
      break;
    case kEmpty:
      msg = rank + "finalize: head " + std::to_string(e->aux) +
            " has an empty normalizer (no keys folded)";
      break;
    default:
      msg = rank + "device error";
  }
  for (auto& kv : w->errs) {
    cudaSetDevice(kv.first);
    cudaMemset(kv.second, 0, offsetof(DevErr, waits));  // keep the tax counters
  }
  return set_error(static_cast<tf_status>(code == -1 ? TF_ERR_WORLD : code), msg);
}

tf_status sync_and_check(World* w, const std::vector<cudaStream_t>& streams) {
  cudaError_t first = cudaSuccess;
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local) continue;
    cudaSetDevice(w->ranks[r].device);
    cudaError_t e = cudaStreamSynchronize(streams[r]);
    if (e != cudaSuccess && first == cudaSuccess) first = e;
    e = cudaStreamSynchronize(w->ranks[r].side);
    if (e != cudaSuccess && first == cudaSuccess) first = e;
  }
  if (first != cudaSuccess) return cuda_status(first, "stream synchronize");
  return check_record(w);
}

// ---- kernels ---------------------------------------------------------------

__global__ void barrier_kernel(uint64_t* const* cells, int self, int W, uint64_t epoch,
                               uint64_t watchdog_ns, DevErr* err, int board) {
  if (threadIdx.x != 0) return;
  fence_sys();
  for (int r = 0; r < W; ++r) red_release_sys(cells[r], 1);
  const uint64_t target = epoch * uint64_t(W);
  if (!wait_geq(cells[self], target, watchdog_ns, err, kWaitBarrier, self, board, 0, 0,
                epoch - 1)) {
    // Rewrite observed/expected as "arrived of W" for the message.  The raw
    // cell counts every generation's arrivals; a cell still short of the
    // previous generations (a rank that never arrived at an earlier barrier
    // either) reads as 0 arrivals, never as a wrapped subtraction.
    if (err->kind == kWaitBarrier && err->rank == self) {
      const uint64_t base = (epoch - 1) * uint64_t(W);
      const uint64_t seen = err->observed;
      err->observed = seen >= base ? (seen - base < uint64_t(W) ? seen - base : uint64_t(W)) : 0;
      err->expected = uint64_t(W);
    }
  }
}

__global__ void signal_kernel(uint64_t* cell) {
  fence_sys();
  red_release_sys(cell, 1);
}

__global__ void wait_kernel(const uint64_t* cell, uint64_t expected, uint64_t watchdog_ns,
                            DevErr* err, int rank, int board, int row, int slot) {
  wait_geq(cell, expected, watchdog_ns, err, kWaitSignal, rank, board, row, slot, 0);
}

__device__ __forceinline__ uint32_t mix32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return static_cast<uint32_t>(x);
}

// harness.hpp:146-195 on the device: for every peer p, warp 0 produces
// `rounds` payloads into p's mailbox (waiting for p's ack before reusing it)
// and warp 1 consumes p's payloads, checking each against the expected
// pattern right after the acquire.  Seeded __nanosleep jitter on both sides
// randomises the interleaving.  mail: [W src][4] u32 per rank;
// flags/acks: [W] u64 per rank.
__global__ void soak_kernel(uint32_t* const* mail, uint64_t* const* flags,
                            uint64_t* const* acks, int self, int W, uint64_t seed, int rounds,
                            uint64_t base, unsigned long long* violations,
                            uint64_t watchdog_ns, DevErr* err, int board) {
  const int peer = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (lane != 0) return;
  if (warp == 0) {  // producer toward `peer`
    for (int r = 0; r < rounds; ++r) {
      if (r > 0 && !wait_geq(&acks[self][peer], base + r, watchdog_ns, err, kWaitSignal, self,
                             board, peer, 1, 0))
        return;
      __nanosleep(mix32(seed * 1315423911ull + r * 7 + self * 131 + peer) % 2000);
      uint32_t* box = mail[peer] + size_t(self) * 4;
      for (int i = 0; i < 4; ++i)
        box[i] = mix32((seed << 20) ^ (uint64_t(self) << 40) ^ (uint64_t(peer) << 48) ^
                       (uint64_t(r) << 4) ^ i);
      red_release_sys(&flags[peer][self], 1);
    }
  } else {  // consumer of `peer`'s payloads
    for (int r = 0; r < rounds; ++r) {
      __nanosleep(mix32(seed * 2654435761ull + r * 13 + peer * 17 + self) % 2000);
      if (!wait_geq(&flags[self][peer], base + r + 1, watchdog_ns, err, kWaitSignal, self, board,
                    peer, 0, 0))
        return;
      const volatile uint32_t* box = mail[self] + size_t(peer) * 4;
      for (int i = 0; i < 4; ++i) {
        uint32_t want = mix32((seed << 20) ^ (uint64_t(peer) << 40) ^ (uint64_t(self) << 48) ^
                              (uint64_t(r) << 4) ^ i);
        if (box[i] != want) atomicAdd(violations, 1ull);
      }
      red_release_sys(&acks[peer][self], 1);
    }
  }
}

tf_status ensure_barrier(World* w) {
  if (w->barrier_ready) return TF_OK;
  BoardEntry b;
  TFB_CHECK(board_get(w, "tf.barrier", 1, 1, &b));
  std::vector<uint64_t*> cells(w->W);
  for (int r = 0; r < w->W; ++r) cells[r] = reinterpret_cast<uint64_t*>(w->ptr(r, b.offset));
  TFB_CHECK(heap_get(w, "tf.barrier.table", sizeof(uint64_t*) * 64, &w->barrier_table_off));
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local) continue;
    TFB_CUDA(cudaSetDevice(w->ranks[r].device));
    TFB_CUDA(cudaMemcpy(w->ptr(r, w->barrier_table_off), cells.data(), sizeof(uint64_t*) * w->W,
                        cudaMemcpyHostToDevice));
  }
  w->barrier_ready = true;
  return TF_OK;
}

tf_status world_barrier(World* w, const std::vector<cudaStream_t>& streams, int only_rank) {
  TFB_CHECK(ensure_barrier(w));
  const int board = w->boards["tf.barrier"].id;
  const uint64_t epoch = ++w->barrier_epoch;
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local || (only_rank >= 0 && r != only_rank)) continue;
    cudaSetDevice(w->ranks[r].device);
    uint64_t** table = reinterpret_cast<uint64_t**>(w->ptr(r, w->barrier_table_off));
    barrier_kernel<<<1, 32, 0, streams[r]>>>(table, r, w->W, epoch, w->watchdog_ns, w->err_of(r), board);
    TFB_CUDA(cudaGetLastError());
    ++w->launches;
  }
  return TF_OK;
}

__global__ void skew_kernel(uint64_t ns);

static tf_status world_init_common(World* w) {
  for (const RankRes& rr : w->ranks) {
    if (!rr.local || w->errs.count(rr.device)) continue;
    DevErr* e = nullptr;
    TFB_CUDA(cudaSetDevice(rr.device));
    TFB_CUDA(cudaMalloc(reinterpret_cast<void**>(&e), sizeof(DevErr)));
    TFB_CUDA(cudaMemset(e, 0, sizeof(DevErr)));
    w->errs[rr.device] = e;
    // Load every kernel now, not lazily inside a schedule's first call.
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, barrier_kernel);
    cudaFuncGetAttributes(&a, signal_kernel);
    cudaFuncGetAttributes(&a, wait_kernel);
    cudaFuncGetAttributes(&a, soak_kernel);
    cudaFuncGetAttributes(&a, skew_kernel);
    ag_exact_preload();
    ag_sm100_preload();
    fd_preload();
    TFB_CUDA(cudaGetLastError());
  }
  // Heap/record memsets ran on the legacy stream; the world's non-blocking
  // streams must not overtake them.
  for (auto& kv : w->errs) {
    TFB_CUDA(cudaSetDevice(kv.first));
    TFB_CUDA(cudaDeviceSynchronize());
  }
  return TF_OK;
}

static tf_status check_device(int dev) {
  int n = 0;
  TFB_CUDA(cudaGetDeviceCount(&n));
  if (dev < 0 || dev >= n)
    return set_error(TF_ERR_CONFIG, "device " + std::to_string(dev) + " out of range (" +
                                        std::to_string(n) + " visible)");
  cudaDeviceProp p;
  TFB_CUDA(cudaGetDeviceProperties(&p, dev));
  if (p.major != 10)
    return set_error(TF_ERR_CUDA, std::string("device ") + p.name +
                                      " is not sm_100 (Blackwell); this build targets sm_100a only");
  return TF_OK;
}

__global__ void skew_kernel(uint64_t ns) {
  const uint64_t t0 = globaltimer_ns();
  while (globaltimer_ns() - t0 < ns) __nanosleep(1000);
}

tf_status launch_skew(World* w, int r, cudaStream_t s) {
  const uint64_t ns = w->skew_of(r);
  if (!ns) return TF_OK;
  cudaSetDevice(w->ranks[r].device);
  skew_kernel<<<1, 1, 0, s>>>(ns);
  TFB_CUDA(cudaGetLastError());
  return TF_OK;
}

}  // namespace tfb

using namespace tfb;

extern "C" {

const char* tf_last_error(void) { return g_last_error.c_str(); }
int tf_abi_version(void) { return TF_ABI_VERSION; }

tf_status tf_world_create(int world_size, const int* devices, size_t heap_bytes_per_rank,
                          double watchdog_secs, tf_world** out) {
  if (!out) return set_error(TF_ERR_CONFIG, "tf_world_create: out is NULL");
  *out = nullptr;
  if (world_size < 1 || world_size > 64)
    return set_error(TF_ERR_CONFIG,
                     "world_size must be in [1, 64], got " + std::to_string(world_size));
  if (heap_bytes_per_rank == 0) return set_error(TF_ERR_CONFIG, "heap_bytes_per_rank must be > 0");
  auto* tw = new tf_world();
  World* w = &tw->impl;
  w->W = world_size;
  w->watchdog_secs = watchdog_secs > 0 ? watchdog_secs : default_watchdog_secs();
  w->watchdog_ns = static_cast<uint64_t>(w->watchdog_secs * 1e9);
  w->heap_bytes = (heap_bytes_per_rank + 4095) / 4096 * 4096;
  w->first_local = 0;
  w->n_local = world_size;
  w->ranks.resize(world_size);
  auto fail = [&](tf_status s) {
    tf_world_destroy(tw);
    return s;
  };
  for (int r = 0; r < world_size; ++r) {
    const int dev = devices ? devices[r] : 0;
    tf_status s = check_device(dev);
    if (s != TF_OK) return fail(s);
    w->ranks[r].device = dev;
    w->ranks[r].local = true;
  }
  for (int r = 0; r < world_size; ++r)
    for (int q = 0; q < r; ++q)
      if (w->ranks[r].device == w->ranks[q].device) w->loopback = true;
  // Peer mappings between distinct devices (NVLink through NVSwitch).
  for (int r = 0; r < world_size; ++r) {
    for (int q = 0; q < world_size; ++q) {
      const int a = w->ranks[r].device, b = w->ranks[q].device;
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (!can)
        return fail(set_error(TF_ERR_CUDA, "device " + std::to_string(a) +
                                               " cannot access peer device " + std::to_string(b)));
      cudaSetDevice(a);
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return fail(cuda_status(e, "cudaDeviceEnablePeerAccess"));
    }
  }
  for (int r = 0; r < world_size; ++r) {
    RankRes& rr = w->ranks[r];
    cudaError_t e = cudaSetDevice(rr.device);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&rr.heap), w->heap_bytes);
    if (e == cudaSuccess) e = cudaMemset(rr.heap, 0, w->heap_bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeros land before any peer can map the heap
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&rr.stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&rr.side, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(cuda_status(e, "rank heap/stream setup"));
    rr.owns_heap = true;
  }
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, w->ranks[0].device);
  w->sm_count = p.multiProcessorCount;
  tf_status s = world_init_common(w);
  if (s != TF_OK) return fail(s);
  *out = tw;
  return TF_OK;
}

tf_status tf_world_create_ipc(int rank, int world_size, int device, size_t heap_bytes_per_rank,
                              double watchdog_secs, tf_world** out) {
  if (!out) return set_error(TF_ERR_CONFIG, "tf_world_create_ipc: out is NULL");
  *out = nullptr;
  if (world_size < 1 || world_size > 64)
    return set_error(TF_ERR_CONFIG,
                     "world_size must be in [1, 64], got " + std::to_string(world_size));
  if (rank < 0 || rank >= world_size)
    return set_error(TF_ERR_CONFIG, "rank " + std::to_string(rank) + " out of range");
  TFB_CHECK(check_device(device));
  auto* tw = new tf_world();
  World* w = &tw->impl;
  w->W = world_size;
  w->ipc = true;
  w->first_local = rank;
  w->n_local = 1;
  w->watchdog_secs = watchdog_secs > 0 ? watchdog_secs : default_watchdog_secs();
  w->watchdog_ns = static_cast<uint64_t>(w->watchdog_secs * 1e9);
  w->heap_bytes = (heap_bytes_per_rank + 4095) / 4096 * 4096;
  w->ranks.resize(world_size);
  RankRes& rr = w->ranks[rank];
  rr.device = device;
  rr.local = true;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&rr.heap), w->heap_bytes);
  if (e == cudaSuccess) e = cudaMemset(rr.heap, 0, w->heap_bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeros land before the handle is exported
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&rr.stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&rr.side, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    tf_world_destroy(tw);
    return cuda_status(e, "ipc rank setup");
  }
  rr.owns_heap = true;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, device);
  w->sm_count = p.multiProcessorCount;
  tf_status s = world_init_common(w);
  if (s != TF_OK) {
    tf_world_destroy(tw);
    return s;
  }
  *out = tw;
  return TF_OK;
}

tf_status tf_world_ipc_export(tf_world* tw, void* handle_out) {
  if (!tw || !handle_out) return set_error(TF_ERR_CONFIG, "tf_world_ipc_export: NULL argument");
  World* w = &tw->impl;
  if (!w->ipc) return set_error(TF_ERR_CONFIG, "tf_world_ipc_export: not an IPC world");
  cudaIpcMemHandle_t h;
  cudaSetDevice(w->ranks[w->first_local].device);
  TFB_CUDA(cudaIpcGetMemHandle(&h, w->ranks[w->first_local].heap));
  static_assert(sizeof(h) == TF_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  return TF_OK;
}

tf_status tf_world_ipc_import(tf_world* tw, const void* all_handles) {
  if (!tw || !all_handles) return set_error(TF_ERR_CONFIG, "tf_world_ipc_import: NULL argument");
  World* w = &tw->impl;
  if (!w->ipc) return set_error(TF_ERR_CONFIG, "tf_world_ipc_import: not an IPC world");
  const int self = w->first_local;
  cudaSetDevice(w->ranks[self].device);
  for (int r = 0; r < w->W; ++r) {
    if (r == self) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(all_handles) + size_t(r) * TF_IPC_HANDLE_BYTES,
                sizeof(h));
    void* p = nullptr;
    TFB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    w->ranks[r].heap = static_cast<char*>(p);
    w->ranks[r].device = -1;
  }
  w->barrier_ready = false;  // the cell table needs the peers' heaps
  return TF_OK;
}

tf_status tf_world_destroy(tf_world* tw) {
  if (!tw) return TF_OK;
  World* w = &tw->impl;
  for (int r = 0; r < (int)w->ranks.size(); ++r) {
    RankRes& rr = w->ranks[r];
    if (rr.local) cudaSetDevice(rr.device);
    if (rr.stream) cudaStreamSynchronize(rr.stream), cudaStreamDestroy(rr.stream);
    if (rr.side) cudaStreamSynchronize(rr.side), cudaStreamDestroy(rr.side);
    if (rr.h2d) cudaStreamSynchronize(rr.h2d), cudaStreamDestroy(rr.h2d);
    if (rr.legacy_ev) cudaEventDestroy(rr.legacy_ev);
    if (rr.d2h) cudaStreamSynchronize(rr.d2h), cudaStreamDestroy(rr.d2h);
    for (void* p : rr.scratch)
      if (p) cudaFree(p);
    for (int i = 0; i < 2; ++i) {
      if (rr.host_reads_done[i]) cudaEventDestroy(rr.host_reads_done[i]);
      if (rr.host_d2h_done[i]) cudaEventDestroy(rr.host_d2h_done[i]);
    }
  }
  for (int r = 0; r < (int)w->ranks.size(); ++r) {
    RankRes& rr = w->ranks[r];
    if (!rr.heap) continue;
    if (rr.owns_heap) {
      cudaSetDevice(rr.device);
      cudaFree(rr.heap);
    } else if (w->ipc) {
      cudaIpcCloseMemHandle(rr.heap);
    }
  }
  for (auto& kv : w->errs) {
    cudaSetDevice(kv.first);
    cudaFree(kv.second);
  }
  delete tw;
  return TF_OK;
}

int tf_world_size(const tf_world* tw) { return tw ? tw->impl.W : 0; }

int tf_world_local_ranks(const tf_world* tw, int* first_rank) {
  if (!tw) return 0;
  if (first_rank) *first_rank = tw->impl.first_local;
  return tw->impl.n_local;
}

void* tf_world_stream(tf_world* tw, int rank) {
  if (!tw || rank < 0 || rank >= tw->impl.W || !tw->impl.ranks[rank].local) return nullptr;
  return tw->impl.ranks[rank].stream;
}

tf_status tf_world_reset_heap(tf_world* tw) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  auto streams = resolve_streams(w, nullptr);
  TFB_CHECK(sync_and_check(w, streams));
  w->heap.clear();
  w->epochs.clear();
  w->boards.clear();
  w->board_names.clear();
  w->heap_used = 0;
  w->barrier_epoch = w->ag_epoch = w->fd_epoch = 0;
  w->barrier_ready = false;
  w->ag_flags = FlagSnapshot{};
  w->fd_flags = FlagSnapshot{};
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local) continue;
    TFB_CUDA(cudaSetDevice(w->ranks[r].device));
    TFB_CUDA(cudaMemset(w->ranks[r].heap, 0, w->heap_bytes));
    TFB_CUDA(cudaDeviceSynchronize());
  }
  return TF_OK;
}

tf_status tf_heap_alloc(tf_world* tw, const char* name, size_t bytes_per_rank,
                        void** per_rank_ptrs) {
  if (!tw || !name) return set_error(TF_ERR_CONFIG, "tf_heap_alloc: NULL argument");
  World* w = &tw->impl;
  size_t off;
  TFB_CHECK(heap_get(w, name, bytes_per_rank, &off));
  if (per_rank_ptrs)
    for (int r = 0; r < w->W; ++r) per_rank_ptrs[r] = w->ranks[r].heap ? w->ptr(r, off) : nullptr;
  return TF_OK;
}

tf_status tf_board_alloc(tf_world* tw, const char* name, int rows, int slots,
                         uint64_t** per_rank_cells) {
  if (!tw || !name) return set_error(TF_ERR_CONFIG, "tf_board_alloc: NULL argument");
  World* w = &tw->impl;
  BoardEntry b;
  TFB_CHECK(board_get(w, name, rows, slots, &b));
  if (per_rank_cells)
    for (int r = 0; r < w->W; ++r)
      per_rank_cells[r] = w->ranks[r].heap ? reinterpret_cast<uint64_t*>(w->ptr(r, b.offset)) : nullptr;
  return TF_OK;
}

static tf_status find_cell(World* w, const char* board, int rank, int row, int slot,
                           const char* what, BoardEntry* b, uint64_t** cell) {
  if (!board) return set_error(TF_ERR_CONFIG, std::string(what) + ": NULL board");
  auto it = w->boards.find(board);
  if (it == w->boards.end())
    return set_error(TF_ERR_CONFIG, std::string(what) + ": unknown board \"" + board + "\"");
  *b = it->second;
  if (rank < 0 || rank >= w->W)
    return set_error(TF_ERR_BOUNDS, std::string(what) + ": rank " + std::to_string(rank) +
                                        " out of range for world_size " + std::to_string(w->W));
  if (row < 0 || row >= b->rows || slot < 0 || slot >= b->slots)
    return set_error(TF_ERR_BOUNDS, std::string(what) + "(board \"" + board + "\"): cell (" +
                                        std::to_string(row) + ", " + std::to_string(slot) +
                                        ") out of range");
  *cell = reinterpret_cast<uint64_t*>(w->ptr(rank, b->offset)) + size_t(row) * b->slots + slot;
  return TF_OK;
}

tf_status tf_signal(tf_world* tw, const char* board, int src_rank, int dst_rank, int row,
                    int slot) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  BoardEntry b;
  uint64_t* cell;
  TFB_CHECK(find_cell(w, board, dst_rank, row, slot, "atomic_signal", &b, &cell));
  if (src_rank < 0 || src_rank >= w->W || !w->ranks[src_rank].local)
    return set_error(TF_ERR_BOUNDS, "atomic_signal: source rank " + std::to_string(src_rank) +
                                        " is not local to this process");
  cudaSetDevice(w->ranks[src_rank].device);
  signal_kernel<<<1, 1, 0, w->ranks[src_rank].stream>>>(cell);
  TFB_CUDA(cudaGetLastError());
  ++w->launches;
  TFB_CUDA(cudaStreamSynchronize(w->ranks[src_rank].stream));
  return check_record(w);
}

tf_status tf_wait_signal(tf_world* tw, const char* board, int rank, int row, int slot,
                         uint64_t expected) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  BoardEntry b;
  uint64_t* cell;
  TFB_CHECK(find_cell(w, board, rank, row, slot, "wait_signal", &b, &cell));
  if (!w->ranks[rank].local)
    return set_error(TF_ERR_BOUNDS, "wait_signal: rank " + std::to_string(rank) + " is not local");
  cudaSetDevice(w->ranks[rank].device);
  wait_kernel<<<1, 1, 0, w->ranks[rank].stream>>>(cell, expected, w->watchdog_ns, w->err_of(rank), rank,
                                                  b.id, row, slot);
  TFB_CUDA(cudaGetLastError());
  ++w->launches;
  TFB_CUDA(cudaStreamSynchronize(w->ranks[rank].stream));
  return check_record(w);
}

tf_status tf_read_signal(tf_world* tw, const char* board, int rank, int row, int slot,
                         uint64_t* value) {
  if (!tw || !value) return set_error(TF_ERR_CONFIG, "NULL argument");
  World* w = &tw->impl;
  BoardEntry b;
  uint64_t* cell;
  TFB_CHECK(find_cell(w, board, rank, row, slot, "read_signal", &b, &cell));
  TFB_CUDA(cudaMemcpy(value, cell, sizeof(uint64_t), cudaMemcpyDefault));
  return TF_OK;
}

tf_status tf_signal_soak(tf_world* tw, uint64_t seed, int rounds, uint64_t* violations) {
  if (!tw || !violations || rounds < 1) return set_error(TF_ERR_CONFIG, "tf_signal_soak: bad args");
  World* w = &tw->impl;
  BoardEntry fb, ab;
  TFB_CHECK(board_get(w, "soak.flags", 1, w->W, &fb));
  TFB_CHECK(board_get(w, "soak.acks", 1, w->W, &ab));
  size_t mail_off, tab_off, cnt_off;
  TFB_CHECK(heap_get(w, "soak.mail", sizeof(uint32_t) * 4 * w->W, &mail_off));
  TFB_CHECK(heap_get(w, "soak.tables", sizeof(void*) * 3 * 64, &tab_off));
  TFB_CHECK(heap_get(w, "soak.violations", sizeof(unsigned long long), &cnt_off));
  // Monotonic boards: this soak's counters start where the last one ended.
  uint64_t& soak_epoch = w->epochs["soak"];
  const uint64_t base = soak_epoch;
  soak_epoch += uint64_t(rounds);
  std::vector<void*> tables(3 * 64, nullptr);
  for (int r = 0; r < w->W; ++r) {
    tables[r] = w->ptr(r, mail_off);
    tables[64 + r] = w->ptr(r, fb.offset);
    tables[128 + r] = w->ptr(r, ab.offset);
  }
  auto streams = resolve_streams(w, nullptr);
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local) continue;
    cudaSetDevice(w->ranks[r].device);
    void** t = reinterpret_cast<void**>(w->ptr(r, tab_off));
    TFB_CUDA(cudaMemcpyAsync(t, tables.data(), sizeof(void*) * tables.size(),
                             cudaMemcpyHostToDevice, streams[r]));
    TFB_CUDA(cudaMemsetAsync(w->ptr(r, cnt_off), 0, sizeof(unsigned long long), streams[r]));
  }
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local) continue;
    cudaSetDevice(w->ranks[r].device);
    void** t = reinterpret_cast<void**>(w->ptr(r, tab_off));
    soak_kernel<<<w->W, 64, 0, streams[r]>>>(
        reinterpret_cast<uint32_t* const*>(t), reinterpret_cast<uint64_t* const*>(t + 64),
        reinterpret_cast<uint64_t* const*>(t + 128), r, w->W, seed, rounds, base,
        reinterpret_cast<unsigned long long*>(w->ptr(r, cnt_off)), w->watchdog_ns, w->err_of(r),
        fb.id);
    TFB_CUDA(cudaGetLastError());
    ++w->launches;
  }
  TFB_CHECK(sync_and_check(w, streams));
  uint64_t total = 0;
  for (int r = 0; r < w->W; ++r) {
    if (!w->ranks[r].local) continue;
    unsigned long long v = 0;
    TFB_CUDA(cudaMemcpy(&v, w->ptr(r, cnt_off), sizeof(v), cudaMemcpyDefault));
    total += v;
  }
  *violations = total;
  return TF_OK;
}

tf_status tf_world_barrier(tf_world* tw, int only_rank) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  if (only_rank >= w->W) return set_error(TF_ERR_BOUNDS, "tf_world_barrier: rank out of range");
  auto streams = resolve_streams(w, nullptr);
  TFB_CHECK(world_barrier(w, streams, only_rank));
  tf_status s = sync_and_check(w, streams);
  if (s != TF_OK && only_rank >= 0) {
    const std::string msg = tf_last_error();
    // The lone waiter gave up; re-align the barrier counters so the world
    // stays usable: the missing ranks' arrivals are added on their behalf.
    BoardEntry b;
    board_get(w, "tf.barrier", 1, 1, &b);
    for (int r = 0; r < w->W; ++r) {
      if (r == only_rank || !w->ranks[r].local) continue;
      for (int q = 0; q < w->W; ++q) {
        uint64_t* cell = reinterpret_cast<uint64_t*>(w->ptr(q, b.offset));
        cudaSetDevice(w->ranks[r].device);
        signal_kernel<<<1, 1, 0, streams[r]>>>(cell);
      }
    }
    sync_and_check(w, streams);
    set_error(s, msg);
  }
  return s;
}

int tf_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

tf_status tf_world_set_skew(tf_world* tw, int rank, uint64_t delay_ns) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  if (rank < 0 || rank >= w->W)  // fabric.hpp:100-105
    return set_error(TF_ERR_CONFIG, "inject_skew: rank " + std::to_string(rank) +
                                        " out of range for world_size " + std::to_string(w->W));
  if (w->skew_ns.size() != size_t(w->W)) w->skew_ns.assign(w->W, 0);
  w->skew_ns[rank] = delay_ns;
  return TF_OK;
}

tf_status tf_tax_report(tf_world* tw, int rank, tf_taxes* out) {
  if (!tw || !out) return set_error(TF_ERR_CONFIG, "tf_tax_report: NULL argument");
  World* w = &tw->impl;
  if (rank < 0 || rank >= w->W || !w->ranks[rank].local)
    return set_error(TF_ERR_BOUNDS, "tf_tax_report: rank " + std::to_string(rank) + " is not local");
  DevErr rec{};
  cudaSetDevice(w->ranks[rank].device);
  TFB_CUDA(cudaMemcpy(&rec, w->err_of(rank), sizeof(DevErr), cudaMemcpyDeviceToHost));
  out->launches = w->launches - w->tax_launch_base;
  // This rank's own waits (a loopback device's record also keeps per-rank
  // rows, so ranks sharing a device are still told apart).
  out->signal_waits = rec.rank_waits[rank & 63];
  out->wait_idle_ns = rec.rank_wait_ns[rank & 63];
  out->barrier_waits = rec.rank_barriers[rank & 63];
  out->bulk_sync_ns = rec.rank_barrier_ns[rank & 63];
  out->staged_bytes = w->staged_bytes.empty() ? 0 : w->staged_bytes[rank];
  return TF_OK;
}

tf_status tf_tax_reset(tf_world* tw) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  TFB_CHECK(sync_and_check(w, resolve_streams(w, nullptr)));
  for (auto& kv : w->errs) {
    TFB_CUDA(cudaSetDevice(kv.first));
    TFB_CUDA(cudaMemset(reinterpret_cast<char*>(kv.second) + offsetof(DevErr, waits), 0,
                        sizeof(DevErr) - offsetof(DevErr, waits)));
  }
  w->tax_launch_base = w->launches;
  std::fill(w->staged_bytes.begin(), w->staged_bytes.end(), 0);
  return TF_OK;
}

tf_status tf_world_sync(tf_world* tw) {
  if (!tw) return set_error(TF_ERR_CONFIG, "NULL world");
  World* w = &tw->impl;
  return sync_and_check(w, resolve_streams(w, nullptr));
}

uint64_t tf_launch_count(const tf_world* tw) { return tw ? tw->impl.launches : 0; }

tf_status tf_uniform_reals(uint64_t seed, size_t n, float* out) {
  if (!out && n) return set_error(TF_ERR_CONFIG, "tf_uniform_reals: NULL out");
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
  for (size_t i = 0; i < n; ++i) out[i] = dist(rng);
  return TF_OK;
}

tf_status tf_memcpy(tf_world* tw, void* dst, const void* src, size_t bytes) {
  if (!tw || (!dst && bytes) || (!src && bytes)) return set_error(TF_ERR_CONFIG, "tf_memcpy: NULL argument");
  if (bytes == 0) return TF_OK;
  TFB_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
  return TF_OK;
}

tf_status tf_memcpy_async(tf_world* tw, void* dst, const void* src, size_t bytes, void* stream) {
  if (!tw || (!dst && bytes) || (!src && bytes)) return set_error(TF_ERR_CONFIG, "tf_memcpy_async: NULL argument");
  if (bytes == 0) return TF_OK;
  TFB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return TF_OK;
}

tf_status tf_device_alloc(tf_world* tw, int rank, size_t bytes, void** out) {
  if (!tw || !out) return set_error(TF_ERR_CONFIG, "tf_device_alloc: NULL argument");
  World* w = &tw->impl;
  if (rank < 0 || rank >= w->W || !w->ranks[rank].local)
    return set_error(TF_ERR_BOUNDS, "tf_device_alloc: rank " + std::to_string(rank) + " is not local");
  TFB_CUDA(cudaSetDevice(w->ranks[rank].device));
  TFB_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  TFB_CUDA(cudaMemset(*out, 0, bytes ? bytes : 1));
  TFB_CUDA(cudaDeviceSynchronize());
  return TF_OK;
}

tf_status tf_device_free(tf_world* tw, int rank, void* p) {
  if (!tw) return set_error(TF_ERR_CONFIG, "tf_device_free: NULL world");
  World* w = &tw->impl;
  if (rank < 0 || rank >= w->W || !w->ranks[rank].local)
    return set_error(TF_ERR_BOUNDS, "tf_device_free: rank " + std::to_string(rank) + " is not local");
  TFB_CUDA(cudaSetDevice(w->ranks[rank].device));
  TFB_CUDA(cudaFree(p));
  return TF_OK;
}

}  // extern "C"
