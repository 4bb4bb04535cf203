// common.cuh -- device-side fabric primitives shared by every kernel:
// system-scope release/acquire flags (the B200 form of SignalBoard,
// fabric.hpp:159-194, 503-569), the %globaltimer watchdog, and the error
// record the host turns back into the reference's exception taxonomy.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "tilefabric_b200/tf_abi.h"

namespace tfb {

// One record per device of a world, in device memory (cheap for spinning
// kernels to poll; the host reads it after a sync).  The first failing
// thread wins the CAS on `code`; everyone else spinning sees code != 0 and
// bails out (the device analogue of World::abort, fabric.hpp:352-363).
struct DevErr {
  int code;       // tf_status
  int rank;       // rank that observed the failure
  int board;      // board id (host maps it to the name)
  int row;
  int slot;
  int kind;       // 0 = signal wait, 1 = barrier, 2 = numeric, 3 = empty
  uint64_t expected;
  uint64_t observed;
  uint64_t aux;   // numeric: flat (head, position); barrier: generation
  // Three-Tax meter (taxmeter.hpp:45-63 on the device): every acquire wait
  // adds its spin time; barrier waits are kept apart (bulk-sync tax).
  unsigned long long waits, wait_ns, barriers, barrier_ns;
  // The same, per waiting rank (a loopback device hosts several ranks).
  unsigned long long rank_waits[64], rank_wait_ns[64], rank_barriers[64], rank_barrier_ns[64];
};

enum : int { kWaitSignal = 0, kWaitBarrier = 1, kNumeric = 2, kEmpty = 3, kPage = 4 };

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// atomic_signal (fabric.hpp:503-507): release-ordered increment on a
// (possibly peer) counter.  Everything this thread wrote before it --
// including peer stores -- is visible to whoever acquires the new value.
__device__ __forceinline__ void red_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Same-device destination: a gpu-scope release is enough and avoids the
// MEMBAR.SYS a sys-scope release costs (~us under load).
__device__ __forceinline__ void red_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Ticket counter: release publishes the CTA's prior writes (cumulative over
// a preceding bar.sync), acquire lets the winner read everyone else's.
__device__ __forceinline__ unsigned long long atom_add_acq_rel_gpu(unsigned long long* p,
                                                                   unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

__device__ __forceinline__ uint64_t atom_add_acq_rel_sys(uint64_t* p, uint64_t v) {
  uint64_t old;
  asm volatile("atom.acq_rel.sys.global.add.u64 %0, [%1], %2;"
               : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// Generic-proxy writes <-> async-proxy (TMA) reads of the same global bytes.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ bool err_raised(const DevErr* e) {
  return *reinterpret_cast<const volatile int*>(&e->code) != 0;
}

__device__ __forceinline__ void raise_err(DevErr* e, int code, int kind, int rank, int board,
                                          int row, int slot, uint64_t expected,
                                          uint64_t observed, uint64_t aux) {
  if (atomicCAS(&e->code, 0, -1) == 0) {
    e->rank = rank;
    e->board = board;
    e->row = row;
    e->slot = slot;
    e->kind = kind;
    e->expected = expected;
    e->observed = observed;
    e->aux = aux;
    __threadfence_system();
    atomicExch(&e->code, code);
    __threadfence_system();
  }
}

// wait_signal (fabric.hpp:519-569): acquire-spin until *cell >= expected.
// Backs off with __nanosleep, checks the watchdog every 256 polls, and
// aborts when another thread already raised an error.  Returns false when
// the wait failed (the caller must unwind without touching the payload).
static __device__ __noinline__ bool wait_geq(const uint64_t* cell, uint64_t expected,
                                      uint64_t watchdog_ns, DevErr* err, int kind,
                                      int rank, int board, int row, int slot,
                                      uint64_t aux) {
  const bool barrier = kind == kWaitBarrier;
  uint64_t seen = ld_acquire_sys(cell);
  const int rk = rank & 63;
  if (seen >= expected) {
    atomicAdd(barrier ? &err->barriers : &err->waits, 1ull);
    atomicAdd(barrier ? &err->rank_barriers[rk] : &err->rank_waits[rk], 1ull);
    return true;
  }
  const uint64_t t0 = globaltimer_ns();
  unsigned ns = 32;
  bool ok = true;
  for (uint32_t polls = 1;; ++polls) {
    seen = ld_acquire_sys(cell);
    if (seen >= expected) break;
    if ((polls & 255u) == 0) {
      if (err_raised(err)) {
        ok = false;
        break;
      }
      if (globaltimer_ns() - t0 > watchdog_ns) {
        raise_err(err, TF_ERR_DEADLOCK, kind, rank, board, row, slot, expected, seen, aux);
        ok = false;
        break;
      }
    }
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;  // short cap: wake-up latency is on the critical path
  }
  const unsigned long long dt = globaltimer_ns() - t0;
  atomicAdd(barrier ? &err->barriers : &err->waits, 1ull);
  atomicAdd(barrier ? &err->barrier_ns : &err->wait_ns, dt);
  atomicAdd(barrier ? &err->rank_barriers[rk] : &err->rank_waits[rk], 1ull);
  atomicAdd(barrier ? &err->rank_barrier_ns[rk] : &err->rank_wait_ns[rk], dt);
  return ok;
}

// Programmatic dependent launch (the hot kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel lets the
// next launch on its stream start being scheduled at once (the ~3 us
// launch gap overlaps its tail) and waits for its own predecessor's memory
// before touching any global data -- stream order is unchanged.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// Split form: launch_dependents at entry, wait once the kernel's on-chip
// setup (mbarriers, TMEM, cluster sync) is done -- that setup touches no
// global memory, so it overlaps the predecessor's tail.
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace tfb
