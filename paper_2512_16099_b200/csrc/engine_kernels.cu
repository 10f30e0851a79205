// engine_kernels.cu — sm_100a kernels of the MIG scheduler engine.
//
//   sim_kernel<SPL>   one warp per trace: the reference's whole event loop
//                     (sim.cpp:71-410) with the scheduler (scheduler.cpp)
//                     and migration planners (migration.cpp) in-kernel; no
//                     host round trips.  SPL = slots per lane = ceil(8G/32).
//
// The host side (host_runtime.cpp) calls the launch_* wrappers below.
#include <cuda_runtime.h>

#include "cluster_core.cuh"
#include "engine_core.cuh"
#include "kernels.h"

namespace msgk {

#ifndef MSG_SIM_WPB
#define MSG_SIM_WPB 4
#endif
constexpr int kWarpsPerBlock = MSG_SIM_WPB;

#ifdef MSG_TRACE_TIMES
// Development aid (-DMSG_TRACE_TIMES): per-trace start / end globaltimer and
// SM of the event-loop kernel, read back with msg_debug_trace_times.
constexpr uint32_t kTraceTimesCap = 1u << 16;
__device__ unsigned long long g_ttimes[4 * kTraceTimesCap];
__device__ unsigned g_tt_n;
#endif

template <int SPL, bool DETAIL, bool IO, bool ND>
#ifndef MSG_SIM_MINB
#define MSG_SIM_MINB 7
#endif
__global__ void __launch_bounds__(32 * kWarpsPerBlock, MSG_SIM_MINB) sim_kernel(SimArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    DevTables* tb = reinterpret_cast<DevTables*>(smem);
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.tables);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (unsigned i = threadIdx.x; i < sizeof(DevTables) / 16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const unsigned w = threadIdx.x >> 5;
    WarpSmem<SPL>* ws = reinterpret_cast<WarpSmem<SPL>*>(smem + sizeof(DevTables) + w * sizeof(WarpSmem<SPL>));
    const uint32_t t = blockIdx.x * kWarpsPerBlock + w;
    if (t >= a.n_traces || a.traces[t].large) return;

#ifdef MSG_TRACE_TIMES
    const uint64_t t0 = wp::gtime_ns();
#endif
    simulate_trace<SPL, DETAIL, IO, ND>(a, tb, ws, t);
#ifdef MSG_TRACE_TIMES
    if (wp::lane() == 0) {
        const unsigned k = atomicAdd(&g_tt_n, 1u);
        if (k < kTraceTimesCap) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            g_ttimes[4 * k] = t0;
            g_ttimes[4 * k + 1] = wp::gtime_ns();
            g_ttimes[4 * k + 2] = sm;
            g_ttimes[4 * k + 3] = a.traces[t].job_off;  // identifies the trace across chunked launches
        }
    }
#endif
}

template <int SPL, bool DETAIL, bool IO, bool ND>
static cudaError_t launch_sim_t(const SimArgs& a, cudaStream_t stream) {
    static_assert(sizeof(DevTables) % 16 == 0, "tables must be 16-byte sized");
    static_assert(sizeof(WarpSmem<SPL>) % 16 == 0, "warp state must be 16-byte sized");
    const size_t smem = sizeof(DevTables) + kWarpsPerBlock * sizeof(WarpSmem<SPL>);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(sim_kernel<SPL, DETAIL, IO, ND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const unsigned blocks = (a.n_traces + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blocks == 0) return cudaSuccess;
    sim_kernel<SPL, DETAIL, IO, ND><<<blocks, 32 * kWarpsPerBlock, smem, stream>>>(a);
    return cudaGetLastError();
}

// Block engine for clusters of more than 32 GPUs: one thread-block cluster
// of a.shards CTAs per trace (a.shards = 1: one block), each CTA one shard
// of the trace's GPUs (cluster_core.cuh).  NT threads per CTA: 512 when a
// CTA owns thousands of GPUs (S <= 8), 256 at 16 shards, where the
// per-event chain of block barriers and exchanges dominates the (then
// small) per-shard scans: C4 at S = 16 runs 2.2x faster with 256 threads
// than with 512 (profiles/r01).
#ifndef MSG_CLUSTER_THREADS_WIDE
#define MSG_CLUSTER_THREADS_WIDE 512
#endif
#ifndef MSG_CLUSTER_THREADS_NARROW
#define MSG_CLUSTER_THREADS_NARROW 256
#endif

template <bool DETAIL, int NT>
__global__ void __launch_bounds__(NT, 1) cluster_kernel(SimArgs a) {
    __shared__ __align__(16) DevTables tb;
    __shared__ BlockScratch sc;
    extern __shared__ __align__(16) unsigned char gpu_smem[];  // 9 B per owned GPU when they fit
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.tables);
        uint4* dst = reinterpret_cast<uint4*>(&tb);
        for (unsigned i = threadIdx.x; i < sizeof(DevTables) / 16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const unsigned S = wp::cluster_size();
    const uint32_t t = a.large_idx[wp::cluster_id() / (a.vdev < 1 ? 1u : a.vdev)];
    const uint32_t G = (uint32_t)a.configs[a.traces[t].cfg].G;
    const bool in_smem = (G + S - 1) / S <= a.smem_gpus;
    simulate_large_trace<DETAIL>(a, &tb, &sc, in_smem ? gpu_smem : nullptr, in_smem && a.smem_slots, t);
}

// Bytes of dynamic shared memory for the per-GPU words of G GPUs (and their
// slots: 96 B more per GPU).
static size_t gpu_smem_bytes(uint32_t G, bool slots) { return ((size_t)G * (slots ? 105 : 9) + 15) & ~(size_t)15; }

template <bool DETAIL, int NT>
static cudaError_t launch_cluster_t(SimArgs a, cudaStream_t stream) {
    static int optin = -1;
    static size_t static_smem = 0;
    if (optin < 0) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaFuncAttributes fa;
        if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, cluster_kernel<DETAIL, NT>);
        if (e == cudaSuccess && kMaxShards > 8)
            e = cudaFuncSetAttribute(cluster_kernel<DETAIL, NT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        static_smem = fa.sharedSizeBytes;
    }
    const uint32_t S = a.shards < 1 ? 1u : a.shards;
    if (S > (uint32_t)kMaxShards) return cudaErrorInvalidValue;
    const uint32_t per = (a.max_gpus + S - 1) / S;  // GPUs per shard (largest trace)
    const size_t room = (size_t)optin > static_smem + 1024 ? (size_t)optin - static_smem - 1024 : 0;
    size_t dyn = 0;
    a.smem_gpus = 0;
    a.smem_slots = 0;
    if (gpu_smem_bytes(per, true) <= room) {
        a.smem_gpus = per;
        a.smem_slots = 1;
        dyn = gpu_smem_bytes(per, true);
    } else if (gpu_smem_bytes(per, false) <= room) {
        a.smem_gpus = per;
        dyn = gpu_smem_bytes(per, false);
    }
    if (dyn > 48 * 1024) {
        cudaError_t e =
            cudaFuncSetAttribute(cluster_kernel<DETAIL, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (e != cudaSuccess) return e;
    }
    const uint32_t groups = a.n_large * (a.vdev < 1 ? 1u : a.vdev);  // clusters in this launch
    if (S == 1 && groups == a.n_large) {
        cluster_kernel<DETAIL, NT><<<a.n_large, NT, dyn, stream>>>(a);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(groups * S);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (groups > a.n_large) {
        // device groups on one GPU spin on each other: all must be co-resident
        int max_clusters = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&max_clusters, cluster_kernel<DETAIL, NT>, &cfg);
        if (e != cudaSuccess) return e;
        if ((uint32_t)max_clusters < groups) return cudaErrorCooperativeLaunchTooLarge;
    }
    return cudaLaunchKernelEx(&cfg, cluster_kernel<DETAIL, NT>, a);
}

cudaError_t launch_cluster(const SimArgs& a, cudaStream_t stream) {
    if (!a.n_large) return cudaSuccess;
    const bool detail = (a.out_flags & (OF_EVENTS | OF_TIMELINE)) != 0;
    constexpr int W = MSG_CLUSTER_THREADS_WIDE, N = MSG_CLUSTER_THREADS_NARROW;
    if (a.shards >= 16)
        return detail ? launch_cluster_t<true, N>(a, stream) : launch_cluster_t<false, N>(a, stream);
    return detail ? launch_cluster_t<true, W>(a, stream) : launch_cluster_t<false, W>(a, stream);
}

template <bool ND>
static cudaError_t launch_sim_nd(int spl, const SimArgs& a, cudaStream_t stream) {
    const bool detail = (a.out_flags & (OF_EVENTS | OF_TIMELINE)) != 0;
    if (a.zc_arrival || a.prog_host) {  // the pipelined msg_run_batch's host-I/O kernel (summary / rows only)
        if (detail) return cudaErrorInvalidValue;
        switch (spl) {
            case 1: return launch_sim_t<1, false, true, ND>(a, stream);
            case 2: return launch_sim_t<2, false, true, ND>(a, stream);
            case 4: return launch_sim_t<4, false, true, ND>(a, stream);
            case 8: return launch_sim_t<8, false, true, ND>(a, stream);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (spl) {
        case 1: return detail ? launch_sim_t<1, true, false, ND>(a, stream) : launch_sim_t<1, false, false, ND>(a, stream);
        case 2: return detail ? launch_sim_t<2, true, false, ND>(a, stream) : launch_sim_t<2, false, false, ND>(a, stream);
        case 4: return detail ? launch_sim_t<4, true, false, ND>(a, stream) : launch_sim_t<4, false, false, ND>(a, stream);
        case 8: return detail ? launch_sim_t<8, true, false, ND>(a, stream) : launch_sim_t<8, false, false, ND>(a, stream);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_sim(int spl, const SimArgs& a, cudaStream_t stream) {
    return a.no_delay ? launch_sim_nd<true>(spl, a, stream) : launch_sim_nd<false>(spl, a, stream);
}

// Load every event-loop and block-engine kernel now (the runtime otherwise
// loads a kernel lazily at its first launch, ~10 ms on the first call).
cudaError_t preload_engine_kernels() {
    cudaFuncAttributes fa;
#define MSG_SIM_FNS(ND)                                                                                   \
    (const void*)sim_kernel<1, false, false, ND>, (const void*)sim_kernel<1, true, false, ND>,             \
        (const void*)sim_kernel<2, false, false, ND>, (const void*)sim_kernel<2, true, false, ND>,         \
        (const void*)sim_kernel<4, false, false, ND>, (const void*)sim_kernel<4, true, false, ND>,         \
        (const void*)sim_kernel<8, false, false, ND>, (const void*)sim_kernel<8, true, false, ND>,         \
        (const void*)sim_kernel<1, false, true, ND>, (const void*)sim_kernel<2, false, true, ND>,           \
        (const void*)sim_kernel<4, false, true, ND>, (const void*)sim_kernel<8, false, true, ND>
    const void* fns[] = {
        MSG_SIM_FNS(false), MSG_SIM_FNS(true),
#undef MSG_SIM_FNS
        (const void*)cluster_kernel<false, MSG_CLUSTER_THREADS_WIDE>,
        (const void*)cluster_kernel<true, MSG_CLUSTER_THREADS_WIDE>,
        (const void*)cluster_kernel<false, MSG_CLUSTER_THREADS_NARROW>,
        (const void*)cluster_kernel<true, MSG_CLUSTER_THREADS_NARROW>};
    for (const void* f : fns) {
        const cudaError_t e = cudaFuncGetAttributes(&fa, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace msgk

#ifdef MSG_PHASE_PROF
extern "C" int msg_debug_phase(unsigned long long* out, int n, int reset) {
    if (n > 16) n = 16;
    if (cudaMemcpyFromSymbol(out, msgk::g_phase, n * sizeof(unsigned long long)) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(msgk::g_phase, z, sizeof(z));
    }
    return n;
}
#endif

#ifdef MSG_TRACE_TIMES
extern "C" int msg_debug_trace_times(unsigned long long* out, unsigned n) {
    // (start ns, end ns, SM, job offset) per finished trace in completion
    // order since the last call; resets the record counter
    unsigned k = 0;
    if (cudaMemcpyFromSymbol(&k, msgk::g_tt_n, sizeof(k)) != cudaSuccess) return -1;
    if (k > n) k = n;
    if (k > msgk::kTraceTimesCap) k = msgk::kTraceTimesCap;
    if (cudaMemcpyFromSymbol(out, msgk::g_ttimes, 4ull * k * sizeof(unsigned long long)) != cudaSuccess) return -1;
    const unsigned z = 0;
    cudaMemcpyToSymbol(msgk::g_tt_n, &z, sizeof(z));
    return (int)k;
}
#endif

#ifdef MSG_SIM_PHASES
extern "C" int msg_debug_sim_phases(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, msgk::g_simph, 8 * sizeof(unsigned long long)) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(msgk::g_simph, z, sizeof(z));
    }
    return 8;
}
#endif
