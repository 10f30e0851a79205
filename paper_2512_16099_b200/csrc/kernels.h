// Host-visible launch wrappers of engine_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include "dev_types.h"

namespace msgk {


// Launch the per-trace event-loop kernel; spl in {1, 2, 4, 8}.
cudaError_t launch_sim(int spl, const SimArgs& a, cudaStream_t stream);

// Launch the block engine over a.large_idx (traces with more than 32 GPUs).
cudaError_t launch_cluster(const SimArgs& a, cudaStream_t stream);

// Load the event-loop and block-engine kernels (msg_engine_create).
cudaError_t preload_engine_kernels();

}  // namespace msgk
