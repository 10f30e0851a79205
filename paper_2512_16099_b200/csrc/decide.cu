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
    TraceSim<SPL> sim;
    sim.setup_snapshot(a, tb, ws, i);
    int32_t out[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int arg = a.arg ? a.arg[i] : 0;
    if (a.op <= SOP_DISPATCH) {
        if (a.op == SOP_SCHEDULE) sim.cflags |= CF_LB;
        if (a.op == SOP_FIRST_FIT) sim.cflags &= ~CF_LB;
        const Decision d = sim.dispatch(arg);
        out[0] = d.placed;
        out[1] = d.placed ? d.g : -1;
        out[2] = d.placed ? d.s : 0;
        out[3] = d.placed ? (int)ms_of(arg) : 0;
        out[4] = d.placed && d.reused;
        out[5] = (int)d.evals;
    } else if (a.op == SOP_TRY_DEQUEUE) {
        sim.dequeue_pass();
        out[0] = (int)sim.q_head;  // placed heads
        out[1] = (int)sim.n_ev;
        sim.store_snapshot(a, i);
    } else {
        // on_departure (migration.cpp:212-220) / plan_intra / plan_inter
        int kind = -1, status = 0;
        const unsigned w0 = ws->gw[arg];
        const bool lazy = (sim.lazymask >> __popc(w0 & 0x7Fu)) & 1u;
        if (a.op == SOP_ON_DEPARTURE) {
            if (a.enabled) {
                kind = lazy ? 1 : 0;
                if (lazy) sim.plan_inter(arg);
                else sim.plan_intra(arg);
            }
        } else if (a.op == SOP_PLAN_INTRA) {
            kind = 0;
            sim.plan_intra(arg);
        } else {
            if (!lazy) {
                status = 5;  // NotLazy (migration.cpp:127-129)
            } else {
                kind = 1;
                sim.plan_inter(arg);
            }
        }
        out[0] = status;
        out[1] = kind;
        out[2] = (int)sim.n_mig;
        out[3] = (int)sim.n_plan_iter;
        out[4] = kind == 0 ? sim.max_intra : sim.max_inter;
        out[5] = (int)sim.n_ev;
        sim.store_snapshot(a, i);
    }
    if (sim.L == 0)
        for (int k = 0; k < 8; ++k) a.out[(size_t)i * 8 + k] = out[k];
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

cudaError_t launch_snapshot(const SnapArgs& a, cudaStream_t stream) {
    const int G = a.G;
    if (G <= 4) return launch_snap_t<1>(a, stream);
    if (G <= 8) return launch_snap_t<2>(a, stream);
    if (G <= 16) return launch_snap_t<4>(a, stream);
    if (G <= 32) return launch_snap_t<8>(a, stream);
    return cudaErrorInvalidValue;
}

}  // namespace msgk
