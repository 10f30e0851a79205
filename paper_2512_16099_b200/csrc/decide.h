// Host-visible launch wrappers of the decision-level kernels.
#pragma once
#include <cuda_runtime.h>

#include "dev_types.h"

namespace msgk {

struct ScoreArgs {
    const DevTables* tables;
    const uint16_t* stab;     // build_score_table (host_tables.h): [profile][popc busy_c][busy_m]
    const uint64_t* words;    // n * G packed GPU words (msg_pack_gpu_word)
    const uint8_t* profile;   // n job profiles
    uint64_t* out;            // 2 per snapshot: argmin key, (lazy << 32 | busy) candidate counts
    uint64_t G;
    uint32_t n;
    uint32_t lb, dyn, lazymask;
    uint32_t* scratch;        // unused (kept for the ABI's scratch sizing)
    uint64_t* items;  // TMA path: 2 words per item (score_items_bytes)
};

cudaError_t launch_snapshot(const SnapArgs& a, cudaStream_t stream);
cudaError_t launch_score(const ScoreArgs& a, cudaStream_t stream);
size_t score_items_bytes(uint32_t n, uint64_t G);
cudaError_t launch_frag_cost(const DevTables* tb, const uint64_t* words, uint32_t n, int32_t* num, double* cost,
                             cudaStream_t stream);

}  // namespace msgk
