// TEST INFRASTRUCTURE ONLY — host-thread emulation of one warp.
//
// Provides the wp:: primitives of paper_2512_16099_b200/csrc/warp_prims.cuh
// so engine_core.cuh (the device code, unchanged) can be executed by 32
// std::threads on the CPU-only build box.  Every collective is a full
// barrier with double-buffered lane exchange; smem is plain shared host
// memory.  Used by tests/test_emu_parity.py to check the kernel logic against
// the reference before any GPU time is spent.  Never loaded by the product.
#pragma once
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <thread>

struct uint4 {
    unsigned x, y, z, w;
};

#define MSG_DI inline
#define MSG_DNI inline

namespace wp {

struct EmuWarp {
    std::atomic<unsigned> arrived{0};
    std::atomic<unsigned> gen{0};
    uint64_t buf[2][32];
};

inline thread_local EmuWarp* g_warp = nullptr;
inline thread_local unsigned g_lane = 0;
inline thread_local unsigned g_phase = 0;

// Block emulation (cluster_core.cuh): nthreads std::threads, one EmuWarp per
// 32 of them, plus a block-wide barrier.
struct EmuBlock {
    std::atomic<unsigned> arrived{0};
    std::atomic<unsigned> gen{0};
    unsigned n = 32;
};
inline thread_local EmuBlock* g_block = nullptr;
inline thread_local unsigned g_tid = 0;

// Cluster emulation (sharded block engine): S emulated blocks, a barrier
// over all their threads, and the base address of each block's scratch so
// cluster_map can translate a shared-memory pointer to another block's copy.
struct EmuCluster {
    std::atomic<unsigned> arrived{0};
    std::atomic<unsigned> gen{0};
    unsigned S = 1;
    unsigned n = 0;  // threads over all blocks
    char* base[64] = {};
};
inline thread_local EmuCluster* g_cluster = nullptr;
inline thread_local unsigned g_crank = 0;

inline void barrier() {
    EmuWarp* w = g_warp;
    const unsigned g = w->gen.load(std::memory_order_acquire);
    if (w->arrived.fetch_add(1, std::memory_order_acq_rel) == 31) {
        w->arrived.store(0, std::memory_order_relaxed);
        w->gen.fetch_add(1, std::memory_order_release);
    } else {
        unsigned spins = 0;
        while (w->gen.load(std::memory_order_acquire) == g) {
            if (++spins > 32) std::this_thread::yield();
        }
    }
}

inline const uint64_t* exchange(uint64_t v) {
    uint64_t* b = g_warp->buf[g_phase & 1u];
    b[g_lane] = v;
    ++g_phase;
    barrier();
    return b;
}

inline unsigned lane() { return g_lane; }
inline unsigned tid() { return g_tid; }
inline unsigned nthreads() { return g_block ? g_block->n : 32u; }
inline void bsync() {
    EmuBlock* b = g_block;
    const unsigned g = b->gen.load(std::memory_order_acquire);
    if (b->arrived.fetch_add(1, std::memory_order_acq_rel) == b->n - 1) {
        b->arrived.store(0, std::memory_order_relaxed);
        b->gen.fetch_add(1, std::memory_order_release);
    } else {
        unsigned spins = 0;
        while (b->gen.load(std::memory_order_acquire) == g) {
            if (++spins > 32) std::this_thread::yield();
        }
    }
}
inline void sync() { barrier(); }
inline unsigned cluster_rank() { return g_cluster ? g_crank : 0u; }
inline unsigned cluster_size() { return g_cluster ? g_cluster->S : 1u; }
inline unsigned cluster_id() { return 0u; }  // one cluster per emulated group
inline void cluster_sync() {
    EmuCluster* c = g_cluster;
    if (!c) {
        bsync();
        return;
    }
    const unsigned g = c->gen.load(std::memory_order_acquire);
    if (c->arrived.fetch_add(1, std::memory_order_acq_rel) == c->n - 1) {
        c->arrived.store(0, std::memory_order_relaxed);
        c->gen.fetch_add(1, std::memory_order_release);
    } else {
        unsigned spins = 0;
        while (c->gen.load(std::memory_order_acquire) == g) {
            if (++spins > 32) std::this_thread::yield();
        }
    }
}
template <class T>
inline const T* cluster_map(const T* p, unsigned rank) {
    if (!g_cluster) return p;
    const char* me = g_cluster->base[g_crank];
    return reinterpret_cast<const T*>(g_cluster->base[rank] + (reinterpret_cast<const char*>(p) - me));
}
inline void gfence() { std::atomic_thread_fence(std::memory_order_seq_cst); }
inline void gfence_sys() { std::atomic_thread_fence(std::memory_order_seq_cst); }
inline void st_release_sys(uint64_t* p, uint64_t v) { std::atomic_ref<uint64_t>(*p).store(v, std::memory_order_release); }
inline uint64_t ld_acquire_sys(const uint64_t* p) {
    return std::atomic_ref<uint64_t>(*const_cast<uint64_t*>(p)).load(std::memory_order_acquire);
}
inline uint64_t gtime_ns() {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
[[noreturn]] inline void fail_stop() { std::abort(); }
inline void spin_pause() { std::this_thread::yield(); }
// Cluster record push (device: st.async + mbarrier complete_tx): copy into
// the destination block's copy of `dst`, then count one record on its copy
// of `bar`; xwait spins until the barrier counted `senders` records for this use.
inline void xbar_init(uint64_t* bar) { std::atomic_ref<uint64_t>(*bar).store(0); }
inline void xbar_arm(uint64_t*, unsigned) {}
inline void xpush(void* dst, const uint4* src, int n16, unsigned rank, uint64_t* bar) {
    std::memcpy(const_cast<void*>(static_cast<const void*>(cluster_map(static_cast<const char*>(dst), rank))), src,
                16 * (size_t)n16);
    uint64_t* rb = const_cast<uint64_t*>(cluster_map(bar, rank));
    std::atomic_ref<uint64_t>(*rb).fetch_add(1, std::memory_order_acq_rel);
}
inline void xwait(uint64_t* bar, unsigned use, unsigned senders) {
    const uint64_t want = (uint64_t)senders * (use + 1);
    unsigned spins = 0;
    while (std::atomic_ref<uint64_t>(*bar).load(std::memory_order_acquire) < want)
        if (++spins > 32) std::this_thread::yield();
}
inline unsigned ballot(bool p) {
    const uint64_t* b = exchange(p ? 1u : 0u);
    unsigned m = 0;
    for (int i = 0; i < 32; ++i)
        if (b[i]) m |= 1u << i;
    return m;
}
inline unsigned rmin(unsigned x) {
    const uint64_t* b = exchange(x);
    unsigned m = 0xFFFFFFFFu;
    for (int i = 0; i < 32; ++i) m = (unsigned)b[i] < m ? (unsigned)b[i] : m;
    return m;
}
inline unsigned radd(unsigned x) {
    const uint64_t* b = exchange(x);
    unsigned m = 0;
    for (int i = 0; i < 32; ++i) m += (unsigned)b[i];
    return m;
}
inline unsigned rmax(unsigned x) {
    const uint64_t* b = exchange(x);
    unsigned m = 0;
    for (int i = 0; i < 32; ++i) m = (unsigned)b[i] > m ? (unsigned)b[i] : m;
    return m;
}
inline unsigned ror(unsigned x) {
    const uint64_t* b = exchange(x);
    unsigned m = 0;
    for (int i = 0; i < 32; ++i) m |= (unsigned)b[i];
    return m;
}
inline unsigned shfl(unsigned x, int src) { return (unsigned)exchange(x)[src & 31]; }
inline int shfl(int x, int src) { return (int)(unsigned)exchange((unsigned)x)[src & 31]; }
inline double shfl(double x, int src) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    const uint64_t r = exchange(u)[src & 31];
    double d;
    std::memcpy(&d, &r, 8);
    return d;
}
inline int popc(unsigned x) { return __builtin_popcount(x); }
inline int ffs(unsigned x) { return __builtin_ffs((int)x); }
// Built with -ffp-contract=off and no -march: plain SSE2 ops, one rounding each.
inline double dadd(double a, double b) { return a + b; }
inline double dsub(double a, double b) { return a - b; }
inline double dmul(double a, double b) { return a * b; }
inline double ddiv(double a, double b) { return a / b; }
inline uint64_t dbits(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}

}  // namespace wp
