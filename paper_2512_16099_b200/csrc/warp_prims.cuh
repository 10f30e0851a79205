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
#define MSG_DNI __device__ __noinline__
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
MSG_DI unsigned cluster_id() {  // index of this cluster in the grid (1-D grids)
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
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
MSG_DI void gfence_sys() { __threadfence_system(); }
// Cross-GPU signalling for device groups (stores land in a peer's memory
// over NVLink): release/acquire at system scope on a 32-bit stamp.
MSG_DI void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
MSG_DI uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
MSG_DI uint64_t gtime_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
[[noreturn]] MSG_DI void fail_stop() { __trap(); }
MSG_DI void spin_pause() {}
// Record push between the CTAs of a cluster (the sharded engine's
// exchange): st.async of 16-byte pieces into the same shared-memory
// location of CTA `rank`, each completing its bytes on that CTA's mbarrier.
// The receiver arms its barrier with the bytes it expects per round and
// waits on the phase parity; no cluster-wide barrier and no memory fence
// on global memory are involved.
MSG_DI uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
MSG_DI void xbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
MSG_DI void xbar_arm(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
MSG_DI void xpush(void* dst, const uint4* src, int n16, unsigned rank, uint64_t* bar) {
    uint32_t ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(dst)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
    for (int i = 0; i < n16; ++i)
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                ra + 16u * (unsigned)i),
            "r"(src[i].x), "r"(src[i].y), "r"(src[i].z), "r"(src[i].w), "r"(rb)
            : "memory");
}
// use: how many times this barrier completed before (the emulation's
// counter); the device waits on the phase parity use & 1.
MSG_DI void xwait(uint64_t* bar, unsigned use, unsigned /*senders*/) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "XWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra XWAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(use & 1u)
        : "memory");
}
}  // namespace wp

#else  // host emulation (tests/emu)
#ifndef MSG_EMU_PRIMS
#error "engine_core.cuh outside nvcc requires the test-only warp emulation (tests/emu)"
#endif
#include MSG_EMU_PRIMS
#endif
