// decide.cu — decision-level kernels: the reference's per-callback policy
// functions on cluster snapshots (scheduler.hpp:59-83, migration.hpp:46-63).
//
//   snapshot_kernel<SPL>  one warp per snapshot of G <= 32 GPUs, running the
//                         same device code as the event loop (engine_core.cuh):
//                         schedule / first_fit_schedule / dispatch_schedule,
//                         try_dequeue, on_departure / plan_intra / plan_inter.
#include <cuda_runtime.h>

#include "decide.h"
#include "engine_core.cuh"

namespace msgk {

constexpr int kSnapWarps = 4;

template <int SPL>
__global__ void __launch_bounds__(32 * kSnapWarps) snapshot_kernel(SnapArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    DevTables* tb = reinterpret_cast<DevTables*>(smem);
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.tables);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (unsigned i = threadIdx.x; i < sizeof(DevTables) / 16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const unsigned w = threadIdx.x >> 5;
    const uint32_t i = blockIdx.x * kSnapWarps + w;
    if (i >= a.n) return;
    WarpSmem<SPL>* ws = reinterpret_cast<WarpSmem<SPL>*>(smem + sizeof(DevTables) + w * sizeof(WarpSmem<SPL>));
    snapshot_op<SPL>(a, tb, ws, i);
}

template <int SPL>
static cudaError_t launch_snap_t(const SnapArgs& a, cudaStream_t stream) {
    const size_t smem = sizeof(DevTables) + kSnapWarps * sizeof(WarpSmem<SPL>);
    if (smem > 48 * 1024) {
        cudaError_t e =
            cudaFuncSetAttribute(snapshot_kernel<SPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const unsigned blocks = (a.n + kSnapWarps - 1) / kSnapWarps;
    if (!blocks) return cudaSuccess;
    snapshot_kernel<SPL><<<blocks, 32 * kSnapWarps, smem, stream>>>(a);
    return cudaGetLastError();
}

// frag_cost (frag.cpp:60-65) of n GPUs from their packed words: the 4-mask
// cost (busy masks drive the ideal counts, blocked memory the feasible
// ones) through the exact tables — numerator over 25200 and the double.
__global__ void frag_cost_kernel(const DevTables* tb, const uint64_t* words, uint32_t n, int32_t* num,
                                 double* cost) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned w = (unsigned)words[i];
    const unsigned row = (unsigned)__popc(w & 0x7Fu) * 9u + (unsigned)__popc((w >> 8) & 0xFFu);
    const unsigned id = tb->cost4pair[tb->idealid[row] * 32u + tb->feasid[(w >> 16) & 0xFFu]];
    if (num) num[i] = (int32_t)tb->cost4k[id];
    if (cost) cost[i] = tb->cost4val[id];
}

cudaError_t launch_frag_cost(const DevTables* tb, const uint64_t* words, uint32_t n, int32_t* num, double* cost,
                             cudaStream_t stream) {
    if (!n) return cudaSuccess;
    frag_cost_kernel<<<(n + 255) / 256, 256, 0, stream>>>(tb, words, n, num, cost);
    return cudaGetLastError();
}

cudaError_t launch_snapshot(const SnapArgs& a, cudaStream_t stream) {
    const int G = a.G;
    if (G <= 4) return launch_snap_t<1>(a, stream);
    if (G <= 8) return launch_snap_t<2>(a, stream);
    if (G <= 16) return launch_snap_t<4>(a, stream);
    if (G <= 32) return launch_snap_t<8>(a, stream);
    return cudaErrorInvalidValue;
}

}  // namespace msgk
