// score.cu — the arrival scorer over large clusters, streamed from HBM.
//
// schedule() / first_fit_schedule() (scheduler.cpp:47-98) for snapshots of
// any size: each GPU is one packed 64-bit state word (busy compute, busy
// memory, blocked memory, 18 idle-exact placement bits; msg_pack_gpu_word).
// A block streams a 2048-word chunk of one snapshot with 128-bit loads
// (8 words per thread), scores every legal start of the job's profile with
// the 2 KiB cost-rank table in shared memory, reduces packed u64 keys
// [pass:1|cost rank:5|!reused:1|gpu:32|start:3] with REDUX.MIN (hi, then lo),
// and merges per snapshot with one 64-bit atomicMin.  Candidate counts feed
// evaluated_candidates (Lazy pass, Busy pass only when Lazy is empty).
//
// Bound: HBM bandwidth — 8 B per scored GPU.
#include <cuda_runtime.h>

#include "decide.h"
#include "dev_types.h"

namespace msgk {

constexpr int kScoreThreads = 256;
constexpr int kWordsPerThread = 8;
constexpr int kChunk = kScoreThreads * kWordsPerThread;  // words per block

__device__ __forceinline__ unsigned s_cs(int p) { return (kCsPack >> (4 * p)) & 0xFu; }
__device__ __forceinline__ unsigned s_ms(int p) { return (kMsPack >> (4 * p)) & 0xFu; }
__device__ __forceinline__ unsigned s_count(int p) { return (kCountPack >> (4 * p)) & 0xFu; }
__device__ __forceinline__ unsigned s_stride(int p) { return (kStridePack >> (4 * p)) & 0xFu; }
// first idle-exact bit of profile p (placements in profile-table order)
__device__ __forceinline__ unsigned s_pbase(int p) { return (0xB7420100u >> (4 * p)) & 0xFu; }

struct ScoreCtx {
    unsigned fm[7], st[7];  // memory footprints and start indexes of the profile's legal starts
    unsigned n, cs, pbase, lb, dyn, lazymask;
};

// All legal starts of the job's profile on one GPU word: candidate_starts
// (scheduler.cpp:19-28: avail, exact-idle when dynamic partitioning is off),
// post-placement cost rank, reuse flag, Lazy/Busy pass.
__device__ __forceinline__ void score_word(const ScoreCtx& c, const uint8_t* lut, uint64_t w, uint64_t g,
                                           uint64_t& best, unsigned& nl, unsigned& nb) {
    const unsigned lo = (unsigned)w;
    const unsigned bc = lo & 0x7Fu, bm = (lo >> 8) & 0xFFu, km = (lo >> 16) & 0xFFu;
    const unsigned exact = (unsigned)(w >> 24) >> c.pbase;
    const unsigned pc = __popc(bc);
    const unsigned lazy = (c.lazymask >> pc) & 1u;
    const uint64_t head = c.lb ? (((uint64_t)(lazy ^ 1u) << 41) | (g << 3)) : (g << 3);
    // popc(busy_c | fc) = pc + cs whenever the start is free
    const unsigned row = min(pc + c.cs, 7u) * 256u;
    unsigned cnt = 0;
#pragma unroll
    for (int j = 0; j < 7; ++j) {
        if ((unsigned)j < c.n) {
            const unsigned ex = (exact >> j) & 1u;
            if (!(c.fm[j] & km) && (c.dyn || ex)) {
                ++cnt;
                const uint64_t key = c.lb ? (head | ((uint64_t)lut[row + (bm | c.fm[j])] << 36) |
                                             ((uint64_t)(ex ^ 1u) << 35) | c.st[j])
                                          : (head | c.st[j]);
                best = key < best ? key : best;
            }
        }
    }
    nl += lazy ? cnt : 0u;
    nb += lazy ? 0u : cnt;
}

__global__ void __launch_bounds__(kScoreThreads) score_kernel(ScoreArgs a) {
    __shared__ __align__(16) uint8_t lut[8 * 256];
    __shared__ uint64_t wbest[kScoreThreads / 32];
    __shared__ unsigned wnl[kScoreThreads / 32], wnb[kScoreThreads / 32];
    for (unsigned i = threadIdx.x; i < 8 * 256 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(lut)[i] = reinterpret_cast<const uint4*>(a.tables->cost2rank)[i];
    const uint64_t chunks_per = (a.G + kChunk - 1) / kChunk;
    const uint64_t snap = blockIdx.x / chunks_per;
    const uint64_t c0 = (blockIdx.x % chunks_per) * kChunk;
    const int p = a.profile[snap];
    ScoreCtx c;
    c.n = s_count(p);
    c.cs = s_cs(p);
    c.pbase = s_pbase(p);
    c.lb = a.lb;
    c.dyn = a.dyn;
    c.lazymask = a.lazymask;
#pragma unroll
    for (int j = 0; j < 7; ++j) {
        const unsigned s = (unsigned)j < c.n ? (unsigned)j * s_stride(p) : 0u;
        c.st[j] = s;
        c.fm[j] = (unsigned)j < c.n ? (((1u << s_ms(p)) - 1u) << s) : 0xFFu;
    }
    __syncthreads();
    const uint64_t* words = a.words + snap * a.G;
    uint64_t best = ~0ull;
    unsigned nl = 0, nb = 0;
    const uint64_t base = c0 + (uint64_t)threadIdx.x * 2;
    if ((a.G & 1) == 0 && c0 + kChunk <= a.G) {
        // full chunk: 4 coalesced 16-byte loads per thread, issued together
        ulonglong2 v[kWordsPerThread / 2];
#pragma unroll
        for (int k = 0; k < kWordsPerThread / 2; ++k)
            v[k] = __ldcs(reinterpret_cast<const ulonglong2*>(words + base + (uint64_t)k * 2 * kScoreThreads));
#pragma unroll
        for (int k = 0; k < kWordsPerThread / 2; ++k) {
            const uint64_t g = base + (uint64_t)k * 2 * kScoreThreads;
            score_word(c, lut, v[k].x, g, best, nl, nb);
            score_word(c, lut, v[k].y, g + 1, best, nl, nb);
        }
    } else {
        for (uint64_t g = c0 + threadIdx.x; g < c0 + kChunk && g < a.G; g += kScoreThreads)
            score_word(c, lut, words[g], g, best, nl, nb);
    }
    // warp: u64 min as (hi, lo) REDUX pair; counts by REDUX.ADD
    const unsigned hi = (unsigned)(best >> 32);
    const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? (unsigned)best : 0xffffffffu);
    nl = __reduce_add_sync(0xffffffffu, nl);
    nb = __reduce_add_sync(0xffffffffu, nb);
    const unsigned w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        wbest[w] = ((uint64_t)mh << 32) | ml;
        wnl[w] = nl;
        wnb[w] = nb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t b = wbest[0];
        unsigned tl = wnl[0], tb = wnb[0];
        for (int k = 1; k < kScoreThreads / 32; ++k) {
            b = wbest[k] < b ? wbest[k] : b;
            tl += wnl[k];
            tb += wnb[k];
        }
        if (b != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(a.out + 2 * snap), (unsigned long long)b);
        if (tl | tb)
            atomicAdd(reinterpret_cast<unsigned long long*>(a.out + 2 * snap + 1),
                      ((unsigned long long)tl << 32) | tb);
    }
}

cudaError_t launch_score(const ScoreArgs& a, cudaStream_t stream) {
    if (!a.n || !a.G) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.out, 0, 16 * (size_t)a.n, stream);
    if (e != cudaSuccess) return e;
    // keys start at ~0 (no candidate); counts at 0
    e = cudaMemset2DAsync(a.out, 16, 0xFF, 8, a.n, stream);
    if (e != cudaSuccess) return e;
    const uint64_t chunks_per = (a.G + kChunk - 1) / kChunk;
    const uint64_t blocks = chunks_per * a.n;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidValue;
    score_kernel<<<(unsigned)blocks, kScoreThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace msgk
