// Warp-level primitives used by the engine (engine_core.cuh).
//
// On the device these are single sm_100a instructions: REDUX.MIN/ADD/OR
// (redux.sync), VOTE.BALLOT, SHFL.IDX, WARPSYNC, and the round-to-nearest
// FP64 intrinsics, which nvcc never contracts into DFMA — bit-exactness
// with the reference's -ffp-contract=off build depends on that (SURVEY §7,
// hard part 1).
//
// When compiled without nvcc (tests/emu only: the CPU-side unit tests of the
// kernel logic), the same names are provided by MSG_EMU_PRIMS, a host-thread
// emulation of one warp.  That build is test infrastructure and is never
// loaded by the product.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)

#define MSG_DI __device__ __forceinline__
#define MSG_GLOBAL __global__

namespace wp {
MSG_DI unsigned lane() {
    unsigned l;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}
MSG_DI unsigned ballot(bool p) { return __ballot_sync(0xffffffffu, p); }
MSG_DI unsigned rmin(unsigned x) { return __reduce_min_sync(0xffffffffu, x); }
MSG_DI unsigned radd(unsigned x) { return __reduce_add_sync(0xffffffffu, x); }
MSG_DI unsigned ror(unsigned x) { return __reduce_or_sync(0xffffffffu, x); }
MSG_DI unsigned rmax(unsigned x) { return __reduce_max_sync(0xffffffffu, x); }
MSG_DI unsigned shfl(unsigned x, int src) { return __shfl_sync(0xffffffffu, x, src); }
MSG_DI int shfl(int x, int src) { return __shfl_sync(0xffffffffu, x, src); }
MSG_DI double shfl(double x, int src) { return __shfl_sync(0xffffffffu, x, src); }
MSG_DI void sync() { __syncwarp(); }
MSG_DI int popc(unsigned x) { return __popc(x); }
MSG_DI int ffs(unsigned x) { return __ffs(x); }  // 1-based, 0 if none
MSG_DI double dadd(double a, double b) { return __dadd_rn(a, b); }
MSG_DI double dsub(double a, double b) { return __dsub_rn(a, b); }
MSG_DI double dmul(double a, double b) { return __dmul_rn(a, b); }
MSG_DI double ddiv(double a, double b) { return __ddiv_rn(a, b); }
MSG_DI uint64_t dbits(double d) { return (uint64_t)__double_as_longlong(d); }
// block level (cluster_core.cuh)
MSG_DI void bsync() { __syncthreads(); }
MSG_DI unsigned tid() { return threadIdx.x; }
MSG_DI unsigned nthreads() { return blockDim.x; }
// thread-block cluster (the sharded block engine, cluster_core.cuh): rank
// and size, a full cluster barrier with release/acquire semantics, and the
// distributed-shared-memory view of a shared variable in another CTA.
MSG_DI unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
MSG_DI unsigned cluster_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
MSG_DI void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <class T>
MSG_DI const T* cluster_map(const T* p, unsigned rank) {
    uint64_t r;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
    return reinterpret_cast<const T*>(r);
}
MSG_DI void gfence() { __threadfence(); }
}  // namespace wp

#else  // host emulation (tests/emu)
#ifndef MSG_EMU_PRIMS
#error "engine_core.cuh outside nvcc requires the test-only warp emulation (tests/emu)"
#endif
#include MSG_EMU_PRIMS
#endif
