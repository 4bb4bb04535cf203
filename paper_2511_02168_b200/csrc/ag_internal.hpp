// ag_internal.hpp -- internal entry points of the All-Gather+GEMM path.
#pragma once
#include <algorithm>
#include <vector>

#include "world.hpp"

namespace tfb {

// fp32 exact-order path (ag_exact.cu).
tf_status ag_exact_run(World* w, tf_ag_variant variant, const tf_ag_shape& sh,
                       void* const* a_shard, const void* const* b, void* const* c,
                       void* const* gathered, const std::vector<cudaStream_t>& streams);

// Operand layout of one bf16 run.  ldb/ldc: row pitch (elements) of B and C
// (0 -> n): a run may cover a column slab of wider B/C buffers (the
// host-streaming entry, ag_host.cu).  inbox_complete: a previous run of the
// same variant and shape already gathered A into the inbox (stream-ordered
// before this one) -- skip the exchange and run the GEMM ungated from it.
// split_k: allow the skinny-M split-K (off for slabs, so a slab's bits
// never depend on how the columns were cut).
struct AgLayout {
  size_t ldb = 0, ldc = 0;
  bool inbox_complete = false;
  bool split_k = true;
};

// bf16 tcgen05 path (ag_sm100.cu).
tf_status ag_bf16_run(World* w, tf_ag_variant variant, const tf_ag_shape& sh,
                      void* const* a_shard, const void* const* b, void* const* c,
                      void* const* gathered, const std::vector<cudaStream_t>& streams,
                      const AgLayout& lay = AgLayout());

}  // namespace tfb
