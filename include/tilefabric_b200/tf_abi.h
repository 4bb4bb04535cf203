/*
 * tf_abi.h -- the C-ABI drop-in boundary of the B200-native tilefabric hot
 * paths (All-Gather+GEMM and multi-GPU Flash Decode).
 *
 * Plain pointers and sizes only; no torch or C++ types.  Every entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj/include/tilefabric/).  The C++ shim in
 * include/tilefabric_b200/tilefabric.hpp rebuilds the reference's own
 * signatures (tilefabric::ag::run_pull(problem, cfg) ...) on top of this;
 * INTEGRATION.md shows the binding a maintainer adds.
 *
 * Threading: one host thread drives a world.  Calls enqueue work on the
 * per-rank streams and, unless documented otherwise, return after every
 * local rank's stream has finished (the reference's launch_world is
 * blocking, fabric.hpp:831-889).  The *_async variants only enqueue.
 *
 * Errors: every call returns a tf_status that maps 1:1 onto the reference's
 * exception classes (common.hpp:39-94); tf_last_error() returns the
 * thread-local message, worded like the reference's (e.g. the watchdog text
 * of fabric.hpp:543-548).  There is no CPU fallback: without a usable
 * sm_100 device every compute entry point fails with TF_ERR_CUDA.
 */
#ifndef TILEFABRIC_B200_TF_ABI_H_
#define TILEFABRIC_B200_TF_ABI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TF_ABI_VERSION 1

typedef struct tf_world tf_world;

/* common.hpp:39-94 -- one status per reference exception class. */
typedef enum {
  TF_OK = 0,
  TF_ERR_CONFIG = 1,          /* ConfigError          common.hpp:46 */
  TF_ERR_BOUNDS = 2,          /* BoundsError          common.hpp:52 */
  TF_ERR_SHAPE = 3,           /* ShapeError           common.hpp:58 */
  TF_ERR_DEADLOCK = 4,        /* DeadlockError        common.hpp:65 */
  TF_ERR_WORLD = 5,           /* WorldError           common.hpp:71 */
  TF_ERR_EMPTY_ATTENTION = 6, /* EmptyAttentionError  common.hpp:77 */
  TF_ERR_NUMERIC = 7,         /* NumericError         common.hpp:84 */
  TF_ERR_CUDA = 8             /* no reference analogue: device failure */
} tf_status;

/* ag_gemm.hpp:134 / :185 / :228 */
typedef enum { TF_AG_BASELINE = 0, TF_AG_PULL = 1, TF_AG_PUSH = 2 } tf_ag_variant;

/* flash_decode.hpp:50 (Variant) */
typedef enum {
  TF_FD_BSP = 0,
  TF_FD_INDEPENDENT_AG = 1,
  TF_FD_FINE_WAITS = 2,
  TF_FD_FUSED = 3,
  /* run_fused with FdOptions::fold_by_arrival (flash_decode.hpp:108-114,
   * 377-408): fold whichever source landed first; not bitwise reproducible. */
  TF_FD_FUSED_BY_ARRIVAL = 4,
  /* Extension (not in the reference): fused, owner-combine.
   * Group g = (b, kv_head) is folded by rank g % W only: every rank pushes
   * its partial rows of g to that owner, the owner folds them in ascending
   * source order (bitwise the other schedules' result), finalizes, and
   * pushes the finished rows to every other rank -- (W-1)/W x (rows of
   * partials + rows of outputs) on the fabric instead of (W-1) x partial
   * rows.  One launch, no barriers; W = 1 is TF_FD_FUSED. */
  TF_FD_FUSED_OWNER = 5
} tf_fd_variant;

typedef enum { TF_F32 = 0, TF_BF16 = 1 } tf_dtype;

const char* tf_last_error(void);
int tf_abi_version(void);

/* ---- world: WorldConfig + launch_world (fabric.hpp:46-96, 831-889) ----
 * Single process, one rank per entry of `devices` (entries may repeat: a
 * "loopback" world runs several ranks on one GPU, the B200 analogue of the
 * reference's oversubscribed thread worlds).  heap_bytes_per_rank sizes
 * each rank's symmetric heap (fabric.hpp:119-153).  watchdog_secs <= 0
 * takes TILEFABRIC_WATCHDOG_SECS or 10 s (common.hpp:35, 97-107).
 * world_size must be in [1, 64] (fabric.hpp:72-75). */
tf_status tf_world_create(int world_size, const int* devices,
                          size_t heap_bytes_per_rank, double watchdog_secs,
                          tf_world** out);

/* Multi-process world (one process per GPU, e.g. torchrun): create the local
 * rank, export its heap handle (TF_IPC_HANDLE_BYTES), all-gather the handles
 * out of band (torch.distributed), then import all of them. */
#define TF_IPC_HANDLE_BYTES 64
tf_status tf_world_create_ipc(int rank, int world_size, int device,
                              size_t heap_bytes_per_rank, double watchdog_secs,
                              tf_world** out);
tf_status tf_world_ipc_export(tf_world* w, void* handle_out);
tf_status tf_world_ipc_import(tf_world* w, const void* all_handles);

tf_status tf_world_destroy(tf_world* w);
int tf_world_size(const tf_world* w);
/* Number of ranks driven by this process and the first one's index. */
int tf_world_local_ranks(const tf_world* w, int* first_rank);
/* Per-rank CUDA stream the world uses when callers pass streams == NULL. */
void* tf_world_stream(tf_world* w, int rank);
/* Drop every heap allocation and board (the next run starts from a zeroed
 * heap, as every launch_world does). */
tf_status tf_world_reset_heap(tf_world* w);

/* ---- symmetric heap: alloc_symmetric (fabric.hpp:276-317, 406-410) ----
 * Collective by construction: allocates `bytes_per_rank` at the same offset
 * in every rank's heap, zero-filled; per_rank_ptrs[r] receives rank r's
 * region as a pointer valid in THIS process (peer regions are mapped over
 * NVLink / P2P).  Re-allocating an existing name returns the same regions
 * when the size matches and TF_ERR_CONFIG otherwise; an empty name or a zero
 * size is TF_ERR_CONFIG (fabric.hpp:279-292, 302-308). */
tf_status tf_heap_alloc(tf_world* w, const char* name, size_t bytes_per_rank,
                        void** per_rank_ptrs);

/* ---- signal boards: alloc_board / atomic_signal / read_signal /
 *      wait_signal (fabric.hpp:159-194, 319-350, 503-569) ----
 * A board is a rows x slots grid of monotonic u64 counters per rank, living
 * in the symmetric heap.  Signals are device-side red.release.sys adds,
 * waits are ld.acquire.sys spins with a %globaltimer watchdog. */
tf_status tf_board_alloc(tf_world* w, const char* name, int rows, int slots,
                         uint64_t** per_rank_cells);
/* One device-side signal from src_rank onto dst_rank's (row, slot). */
tf_status tf_signal(tf_world* w, const char* board, int src_rank, int dst_rank,
                    int row, int slot);
/* Device-side acquire wait on rank's own (row, slot) until >= expected;
 * TF_ERR_DEADLOCK with the reference's message past the watchdog. */
tf_status tf_wait_signal(tf_world* w, const char* board, int rank, int row,
                         int slot, uint64_t expected);
tf_status tf_read_signal(tf_world* w, const char* board, int rank, int row,
                         int slot, uint64_t* value);
/* World barrier on the device (RankCtx::barrier, fabric.hpp:574-584): every
 * local rank's stream runs one barrier kernel.  only_rank >= 0 enters the
 * barrier with that rank alone (the reference's mismatched-barrier
 * diagnostic, acceptance_test.cpp:342-353): TF_ERR_DEADLOCK "barrier
 * generation G: only X of W ranks arrived within the watchdog". */
tf_status tf_world_barrier(tf_world* w, int only_rank);
/* Signal-carries-data soak on the device (harness.hpp:146-195 analogue):
 * `rounds` producer/consumer handshakes between every ordered rank pair,
 * payload written before each release, checked after each acquire.
 * *violations receives the number of stale reads. */
tf_status tf_signal_soak(tf_world* w, uint64_t seed, int rounds,
                         uint64_t* violations);

/* ---- All-Gather + GEMM (ag_gemm.hpp:47-66, 134-305) ----
 * C[m x n] = A[m x k] * B[k x n], all row-major.  A is sharded along k: rank
 * r holds columns [r*kw, (r+1)*kw), kw = k / W, as an m x kw row-major
 * region (ag_gemm.hpp:101-112).  Every rank computes the full C.
 *   dtype TF_F32  -> exact-order CUDA-core path: each C element is one
 *                    ascending-k chain of separately rounded fp32 multiplies
 *                    and adds, bitwise equal to reference::gemm
 *                    (reference.hpp:36-49); any shape, tiles bm/bn/bk follow
 *                    the reference's TileSpec (tilemath.hpp:78-88).
 *   dtype TF_BF16 -> tcgen05/TMEM tensor-core path, fp32 accumulate, bf16 C;
 *                    requires kw % 64 == 0, n % 8 == 0 (TMA strides).
 * a_shard[r] must be a symmetric-heap region (peers read or push it), and
 * every rank's shard must be complete before any rank's call starts: the
 * reference fences the placement (RankCtx::setup_fence after fill_shard,
 * ag_gemm.hpp:189-191, 232-233; fabric.hpp:586-592) outside the timed
 * schedule, and so does this API -- fill the shards, then tf_world_barrier
 * (or, across processes, the launcher's own barrier after a device sync),
 * then call.  PULL reads peer shards with no further fence.
 * gathered_opt[r] (m x k, dtype of A) receives the gathered operand, bit for
 * bit the logical A (the reference's inbox/stage, ag_gemm.hpp:139,234); pass
 * NULL to let the world use an internal heap buffer (double-buffered where
 * peers write it).  A caller buffer is a single buffer, so PUSH then enters a
 * world barrier before its producers run (no peer may store into a buffer
 * its owner is still reading); use tf_ag_gathered instead to inspect the
 * internal operand without it.  streams: per-rank
 * cudaStream_t or NULL (world streams, ordered after the work already
 * issued on the legacy default stream -- where callers usually produce the
 * inputs; with explicit streams the caller owns the ordering).  CUDA-graph
 * capture: a single-rank world's *_async calls may be captured on an
 * explicit stream and replayed (per-launch counters reset on the device;
 * after one eager call, so lazily allocated workspace exists); capturing a
 * multi-rank schedule returns TF_ERR_CONFIG.  The tensor-core GEMM and the
 * Flash Decode kernels are launched with programmatic dependent launch
 * (cudaLaunchAttributeProgrammaticStreamSerialization): each waits for its
 * stream predecessor's memory (griddepcontrol.wait) before touching any
 * global data, so stream order is unchanged -- only the launch latency
 * overlaps the predecessor's tail (TFB_NO_PDL=1 turns it off).  Arrays are
 * indexed by global rank; entries for ranks not local to this process are
 * ignored except a_shard, whose peer entries must be the heap mappings
 * tf_heap_alloc returned. */
/* How A is sharded before the all-gather.  TF_SHARD_K (0, the reference,
 * ag_gemm.hpp:100-107): rank r holds columns [r*k/W, (r+1)*k/W), an m x k/W
 * shard.  TF_SHARD_M (1, an extension: the alternative sharding the paper
 * lists and the reference leaves out): rank r holds rows
 * [r*m/W, (r+1)*m/W), an (m/W) x k shard; bf16 only, m/W a multiple of
 * 128; the gathered operand and C are the same m x k / m x n. */
typedef enum { TF_SHARD_K = 0, TF_SHARD_M = 1 } tf_ag_shard;

typedef struct {
  size_t m, n, k;
  size_t bm, bn, bk; /* TileSpec; 0 -> 16 (tilemath.hpp:79-81) */
  tf_dtype dtype;
  tf_ag_shard shard; /* zero-initialised = TF_SHARD_K, the reference's layout */
} tf_ag_shape;

tf_status tf_ag_gemm(tf_world* w, tf_ag_variant variant, const tf_ag_shape* shape,
                     void* const* a_shard, const void* const* b, void* const* c,
                     void* const* gathered_opt, void* const* streams);
tf_status tf_ag_gemm_async(tf_world* w, tf_ag_variant variant,
                           const tf_ag_shape* shape, void* const* a_shard,
                           const void* const* b, void* const* c,
                           void* const* gathered_opt, void* const* streams);
/* The gathered operand of the last All-Gather+GEMM run on `rank`, m x k
 * row-major (dtype of A) into dst (host or device, >= m*k*esz bytes): the
 * inbox/stage that run's GEMM consumed, with the blocks a schedule reads in
 * place (PULL's own shard; every block of an fp32 PULL, which stages
 * nothing, ag_gemm.hpp:185-222) taken from the shards.  The placement check
 * of ag_gemm_test.cpp:113-169.  Waits for the world's streams first. */
tf_status tf_ag_gathered(tf_world* w, int rank, void* dst, size_t bytes);
/* Host-buffer All-Gather+GEMM: the reference's calling convention, where
 * AgGemmProblem holds host vectors and AgGemmRun returns host C
 * (ag_gemm.hpp:47-99, 134-305).  a_host[r]: rank r's m x kw shard, b_host[r]:
 * k x n, c_host[r]: m x n output, all row-major host memory of `dtype`.  The
 * shard is placed in the symmetric heap, B streams to the device in column
 * slabs and each slab's GEMM starts as soon as it has landed (slab 0 runs
 * the variant's exchange, later slabs reuse the gathered operand); C slabs
 * stream back as their GEMMs retire -- H2D, compute and D2H overlap on three
 * streams per rank.  Pinned host memory (cudaHostAlloc/cudaHostRegister)
 * gives the full overlap; pageable memory is correct but the driver
 * serialises it.  Results are bitwise those of tf_ag_gemm on the same
 * operands (the GEMM of a column slab is the same per-tile computation).
 * The _async form returns once the work is enqueued on the per-rank
 * streams (the host buffers must stay valid until they are idle). */
tf_status tf_ag_gemm_host(tf_world* w, tf_ag_variant variant, const tf_ag_shape* shape,
                          const void* const* a_host, const void* const* b_host,
                          void* const* c_host, void* const* streams);
tf_status tf_ag_gemm_host_async(tf_world* w, tf_ag_variant variant,
                                const tf_ag_shape* shape, const void* const* a_host,
                                const void* const* b_host, void* const* c_host,
                                void* const* streams);

/* Event log (the reference's protocol-safety and overlap checks,
 * ag_gemm_test.cpp:175-244, made on the device): while enabled, every
 * pull/push run records per (m-block, source) chunk the %globaltimer of the
 * chunk's store into the consumer's inbox (gather warp or push producer,
 * just before the release) and of the consumer's first acquire of it (the
 * TMA producer, just before the first load).  tf_ag_events copies rank's
 * record of the last such run: num_m x W pairs {store_ns, first_load_ns}
 * (~0 where nothing was recorded: the rank's own shard).  Debug aid --
 * enabling it adds a device sync per run. */
tf_status tf_world_set_events(tf_world* w, int enable);
tf_status tf_ag_events(tf_world* w, int rank, uint64_t* out, size_t cap, size_t* count);
/* Flash Decode, fused (W > 1): per (source, group) the %globaltimer of the
 * source's release of its rows into this rank's inbox and of this rank's
 * fold reading them (flash_decode_test.cpp:200-247): W x G pairs. */
tf_status tf_fd_events(tf_world* w, int rank, uint64_t* out, size_t cap, size_t* count);

/* Flag snapshot after the last push run (ag_gemm.hpp:296-302): per rank,
 * `count` counters normalised so that one completed run reads 1.
 * *count receives the number of cells per rank. */
tf_status tf_ag_flag_counts(tf_world* w, int rank, uint64_t* out, size_t cap,
                            size_t* count);

/* ---- Flash Decode (flash_decode.hpp:66-106, 212-438) ----
 * Extends DecodeProblem with batch and GQA: q [batch][q_heads][d],
 * k/v shards [batch][kv_heads][kv_len/W][d] (rank r holds positions
 * [r*L/W, (r+1)*L/W), flash_decode.hpp:140-160), out [batch][q_heads][d].
 * q_heads % kv_heads == 0; batch=1, kv_heads=q_heads is the reference.
 * kv_dtype applies to q, k, v.  inbox_opt[r] (symmetric heap,
 * W x batch x q_heads x (d+2) fp32) receives every source's wire rows
 * [m | l | o] (tilemath.hpp:244-258, flash_decode.hpp:353-368).  Every rank
 * folds the W partials in ascending source order, so all ranks' outputs are
 * bitwise identical. */
typedef struct {
  int batch, q_heads, kv_heads, head_dim;
  size_t kv_len;
  float scale;
  tf_dtype kv_dtype, out_dtype;
} tf_fd_shape;

tf_status tf_flash_decode(tf_world* w, tf_fd_variant variant,
                          const tf_fd_shape* shape, const void* const* q,
                          const void* const* k_shard, const void* const* v_shard,
                          void* const* out, void* const* inbox_opt,
                          void* const* streams);
tf_status tf_flash_decode_async(tf_world* w, tf_fd_variant variant,
                                const tf_fd_shape* shape, const void* const* q,
                                const void* const* k_shard,
                                const void* const* v_shard, void* const* out,
                                void* const* inbox_opt, void* const* streams);
/* Paged KV cache (an extension: the reference lists paged KV as a non-goal,
 * SPEC.md:327).  Rank r's K and V are page pools k_pool[r], v_pool[r]
 * (kv_dtype), TF_PAGED_NHD [num_pages][page_size][kv_heads][head_dim] or
 * TF_PAGED_HND [num_pages][kv_heads][page_size][head_dim] (one head's keys
 * of a page contiguous: the faster layout for decode streaming),
 * and block_tables[r]: int32 [batch][pages_per_seq] (device memory) maps
 * the rank's local position x of sequence b (x < kv_len / W, the same
 * position split as tf_flash_decode) to row x % page_size of page
 * block_tables[r][b][x / page_size].  page_size is a power of two;
 * pages_per_seq * page_size >= kv_len / W.  Every schedule, the wire rows
 * and the output are bitwise those of tf_flash_decode over the same logical
 * KV.  A table entry outside [0, num_pages) fails the call with
 * TF_ERR_SHAPE (the device reads page 0 instead of faulting). */
typedef enum { TF_PAGED_NHD = 0, TF_PAGED_HND = 1 } tf_paged_layout;
typedef struct {
  int page_size, pages_per_seq, num_pages;
  tf_paged_layout layout;
} tf_fd_paged;

tf_status tf_flash_decode_paged(tf_world* w, tf_fd_variant variant, const tf_fd_shape* shape,
                                const tf_fd_paged* paged, const void* const* q,
                                const void* const* k_pool, const void* const* v_pool,
                                const void* const* block_tables, void* const* out,
                                void* const* inbox_opt, void* const* streams);
tf_status tf_flash_decode_paged_async(tf_world* w, tf_fd_variant variant,
                                      const tf_fd_shape* shape, const tf_fd_paged* paged,
                                      const void* const* q, const void* const* k_pool,
                                      const void* const* v_pool,
                                      const void* const* block_tables, void* const* out,
                                      void* const* inbox_opt, void* const* streams);
/* The BSP schedule's two compute stages, for callers that bring their own
 * collective (e.g. NCCL all_gather_into_tensor of the rows in between, the
 * north_star's BSP baseline):
 *   tf_fd_partial_async  attention_partial + serialize_partial for every
 *                        (batch, q-head) of each local rank's shard
 *                        (tilemath.hpp:145-181, 244-258;
 *                        flash_decode.hpp:162-167): rows[r] receives the
 *                        rank's wire rows [B][Hq][d+2] fp32 -- bitwise the
 *                        rows every other schedule exchanges.
 *   tf_fd_combine_async  fold_rows + finalize (flash_decode.hpp:171-180,
 *                        tilemath.hpp:186-239): rows[r] holds W sources'
 *                        rows [W][B][Hq][d+2]; folded in ascending source
 *                        order into out[r] (out_dtype) -- bitwise every
 *                        schedule's output.  TF_ERR_EMPTY_ATTENTION on an
 *                        empty normalizer.
 * Both only enqueue (streams as for tf_flash_decode). */
tf_status tf_fd_partial_async(tf_world* w, const tf_fd_shape* shape, const void* const* q,
                              const void* const* k_shard, const void* const* v_shard,
                              void* const* rows, void* const* streams);
tf_status tf_fd_combine_async(tf_world* w, const tf_fd_shape* shape, const void* const* rows,
                              void* const* out, void* const* streams);
/* fd flag row after the last push-style run (flash_decode.hpp:198-206):
 * per source, normalised so one completed run reads 1. */
tf_status tf_fd_flag_counts(tf_world* w, int rank, uint64_t* out, size_t cap,
                            size_t* count);

/* Plumbing for FFI hosts without their own CUDA bindings (the C++ shim, a
 * cgo/ctypes binding): blocking copy between any host/device/heap pointers
 * (cudaMemcpyDefault), used for the untimed input placement the reference
 * does in fill_shard / slice_shard (ag_gemm.hpp:103-112,
 * flash_decode.hpp:140-160); and caller-owned device buffers. */
tf_status tf_memcpy(tf_world* w, void* dst, const void* src, size_t bytes);
/* Stream-ordered variant (stream: cudaStream_t, NULL = legacy default). */
tf_status tf_memcpy_async(tf_world* w, void* dst, const void* src, size_t bytes, void* stream);
tf_status tf_device_alloc(tf_world* w, int rank, size_t bytes, void** out);
tf_status tf_device_free(tf_world* w, int rank, void* p);

/* uniform_reals (common.hpp:132-140): the reference's seeded inputs,
 * std::mt19937_64 + uniform_real_distribution<float>(-1, 1), bit for bit
 * (host code; make_problem's generator, ag_gemm.hpp:79, flash_decode.hpp:98). */
tf_status tf_uniform_reals(uint64_t seed, size_t n, float* out);

/* Blocks until every local rank's stream is idle and reports any device
 * error record (watchdog, NumericError, EmptyAttentionError). */
tf_status tf_world_sync(tf_world* w);

/* GPUs visible to this process (0 without a driver/GPU; never fails). */
int tf_device_count(void);

/* Number of kernels this library launched since world creation (bench.py's
 * gpu_launches evidence). */
uint64_t tf_launch_count(const tf_world* w);

/* The Three Taxes measured on the device (taxmeter.hpp:45-63):
 * kernel launches (launch tax), acquire waits on signal boards and their
 * spin time (wait_idle), device-barrier waits and their time (bulk-sync
 * tax), bytes stored into staging/inbox tensors (staged_bytes, the
 * inter-kernel locality proxy).  Wait counters are accumulated on the
 * device by every spinning thread (%globaltimer) and reported for the
 * waiting rank (loopback ranks sharing a device are kept apart); launches
 * and staged bytes are host-side counts.  tf_tax_reset zeroes them. */
typedef struct {
  uint64_t launches;
  uint64_t signal_waits, wait_idle_ns;
  uint64_t barrier_waits, bulk_sync_ns;
  uint64_t staged_bytes;
} tf_taxes;
tf_status tf_tax_report(tf_world* w, int rank, tf_taxes* out);

/* Straggler injection (WorldConfig::skew / inject_skew, fabric.hpp:59-62,
 * 100-110): every later run delays `rank`'s first compute stage by
 * delay_ns (0 clears it).  TF_ERR_CONFIG for a rank outside [0, W). */
tf_status tf_world_set_skew(tf_world* w, int rank, uint64_t delay_ns);
tf_status tf_tax_reset(tf_world* w);

#ifdef __cplusplus
}
#endif
#endif /* TILEFABRIC_B200_TF_ABI_H_ */
