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

// bf16 tcgen05 path (ag_sm100.cu).
tf_status ag_bf16_run(World* w, tf_ag_variant variant, const tf_ag_shape& sh,
                      void* const* a_shard, const void* const* b, void* const* c,
                      void* const* gathered, const std::vector<cudaStream_t>& streams);

}  // namespace tfb
