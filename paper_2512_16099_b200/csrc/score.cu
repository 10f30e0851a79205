// score.cu — the arrival scorer over large clusters, streamed from HBM.
//
// schedule() / first_fit_schedule() (scheduler.cpp:47-98) for snapshots of
// any size: each GPU is one packed 64-bit state word (busy compute, busy
// memory, blocked memory, 18 idle-exact placement bits; msg_pack_gpu_word).
// A persistent grid streams 1024-word chunks of the snapshots with 128-bit
// loads (4 words per thread, the next chunk in flight), scores every legal
// start of the job's profile — the profile is block-uniform, so the scoring
// loop is specialised per profile with compile-time footprints — and keeps
// a 32-bit block-local key [pass:1|cost rank:5|!reused:1|word:11|start:3]
// reduced with one REDUX.MIN per warp.  Each warp's winner becomes a 64-bit
// global key [pass|rank|!reused|gpu:32|start] merged per snapshot with one
// atomicMin; candidate counts (Lazy << 16 | Busy) ride one REDUX.ADD.
//
// Bound: HBM bandwidth — 8 B per scored GPU.
#include <cuda_runtime.h>

#include <algorithm>

#include "decide.h"
#include "dev_types.h"

namespace msgk {

constexpr int kScoreThreads = 256;
#ifndef MSG_SCORE_WPT
#define MSG_SCORE_WPT 4
#endif
constexpr int kWordsPerThread = MSG_SCORE_WPT;  // 2 or 4 (one or two 128-bit loads)
constexpr int kChunk = kScoreThreads * kWordsPerThread;  // words per chunk (<= 2048: 11-bit local index)

template <int P>
struct Prof {
    static constexpr unsigned cs = (kCsPack >> (4 * P)) & 0xFu;
    static constexpr unsigned ms = (kMsPack >> (4 * P)) & 0xFu;
    static constexpr unsigned n = (kCountPack >> (4 * P)) & 0xFu;
    static constexpr unsigned stride = (kStridePack >> (4 * P)) & 0xFu;
    static constexpr unsigned pbase = (0x00B74210u >> (4 * P)) & 0xFu;  // first idle-exact bit
    __host__ __device__ static constexpr unsigned fm(unsigned j) { return ((1u << ms) - 1u) << (j * stride); }
};

struct ScoreCfg {
    unsigned lb, dyn, lazymask;
};

// candidate_starts (scheduler.cpp:19-28) of one GPU word, post-placement
// cost rank, reuse flag and Lazy/Busy pass, folded into the running minimum.
template <int P, bool LB>
__device__ __forceinline__ void score_word(const ScoreCfg& c, const uint8_t* lut, uint64_t w, unsigned local,
                                           unsigned& best, unsigned& cnt_lb) {
    using Q = Prof<P>;
    const unsigned lo = (unsigned)w;
    const unsigned bm = (lo >> 8) & 0xFFu, km = (lo >> 16) & 0xFFu;
    const unsigned exact = (unsigned)(w >> (24 + Q::pbase));
    const unsigned pc = __popc(lo & 0x7Fu);
    const unsigned lazy = (c.lazymask >> pc) & 1u;
    const unsigned head = LB ? (((lazy ^ 1u) << 31) | (local << 3)) : (local << 3);
    // LUT row of popc(busy_c | fc) = pc + cs (the start is free), | busy_m
    const unsigned rb = (min(pc + Q::cs, 7u) << 8) | bm;
    const unsigned allow = c.dyn ? 0x7Fu : exact;  // candidate_starts: exact-idle only without dyn
    unsigned cnt = 0;
    // Branch-free: every legal start is scored, unavailable ones are masked.
#pragma unroll
    for (unsigned j = 0; j < Q::n; ++j) {
        const unsigned ok = (((Q::fm(j) & km) == 0) ? 1u : 0u) & (allow >> j);
        const unsigned r = lut[rb | Q::fm(j)];
        const unsigned key = LB ? (head | (r << 26) | ((~exact >> j & 1u) << 25) | (j * Q::stride))
                                : (head | (j * Q::stride));
        best = min(best, ok ? key : 0xFFFFFFFFu);
        cnt += ok;
    }
    cnt_lb += lazy ? cnt << 16 : cnt;
}

// One chunk of one snapshot: every thread scores kWordsPerThread words it
// loaded (128-bit, evict-first) one grid-stride iteration earlier — the
// next chunk's load is in flight while this one is scored.  The warp's
// winner and candidate counts go straight to the snapshot's slots with one
// 64-bit atomicMin / atomicAdd (no block-level synchronisation).
struct ChunkData {
    ulonglong2 v[kWordsPerThread / 2];
};

__device__ __forceinline__ ChunkData load_chunk(const ScoreArgs& a, uint32_t snap, uint32_t c0) {
    ChunkData d;
    const uint64_t* words = a.words + (uint64_t)snap * a.G;
    const unsigned t2 = threadIdx.x * 2u;
#pragma unroll
    for (int k = 0; k < kWordsPerThread / 2; ++k) {
        const uint64_t g = (uint64_t)c0 + t2 + (unsigned)k * 2 * kScoreThreads;
        if ((a.G & 1) == 0 && g + 1 < a.G) {
            d.v[k] = __ldcs(reinterpret_cast<const ulonglong2*>(words + g));
        } else {
            d.v[k].x = g < a.G ? words[g] : 0ull;
            d.v[k].y = g + 1 < a.G ? words[g + 1] : 0ull;
        }
    }
    return d;
}

template <int P, bool LB>
__device__ __forceinline__ void score_chunk(const ScoreArgs& a, const ScoreCfg& c, const uint8_t* lut,
                                            const ChunkData& d, uint64_t snap, uint64_t c0) {
    unsigned best = 0xFFFFFFFFu, cnt = 0;
    const unsigned t2 = threadIdx.x * 2u;
    // words past the snapshot end score as fully occupied (no candidate)
    constexpr uint64_t kFull = 0xFFFF7Full;
#pragma unroll
    for (int k = 0; k < kWordsPerThread / 2; ++k) {
        const unsigned l = t2 + (unsigned)k * 2 * kScoreThreads;
        score_word<P, LB>(c, lut, c0 + l < a.G ? d.v[k].x : kFull, l, best, cnt);
        score_word<P, LB>(c, lut, c0 + l + 1 < a.G ? d.v[k].y : kFull, l + 1, best, cnt);
    }
    best = __reduce_min_sync(0xffffffffu, best);
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) {
        if (best != 0xFFFFFFFFu) {
            // local [pass|rank|!reused|word|start] -> global [pass|rank|!reused|gpu:32|start]
            const uint64_t gpu = c0 + ((best >> 3) & (kChunk - 1));
            const uint64_t g64 = ((uint64_t)(best >> 25) << 35) | (gpu << 3) | (best & 7u);
            atomicMin(reinterpret_cast<unsigned long long*>(a.out + 2 * snap), (unsigned long long)g64);
        }
        if (cnt)
            atomicAdd(reinterpret_cast<unsigned long long*>(a.out + 2 * snap + 1),
                      ((unsigned long long)(cnt >> 16) << 32) | (cnt & 0xFFFFu));
    }
}

// Persistent grid: each block walks chunks blockIdx.x, +gridDim.x, ...; the
// cost-rank table is staged into shared memory once per block.
template <bool LB>
__global__ void __launch_bounds__(kScoreThreads) score_kernel(ScoreArgs a) {
    __shared__ __align__(16) uint8_t lut[8 * 256];
    for (unsigned i = threadIdx.x; i < 8 * 256 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(lut)[i] = reinterpret_cast<const uint4*>(a.tables->cost2rank)[i];
    __syncthreads();
    const ScoreCfg c{a.lb, a.dyn, a.lazymask};
    // chunk ch = snap * chunks_per + j; advanced incrementally (no 64-bit divides)
    const uint32_t chunks_per = (uint32_t)((a.G + kChunk - 1) / kChunk);
    const uint32_t total = chunks_per * a.n;
    uint32_t ch = blockIdx.x;
    if (ch >= total) return;
    uint32_t snap = ch / chunks_per, j = ch - snap * chunks_per;
    const uint32_t step_s = gridDim.x / chunks_per, step_j = gridDim.x - step_s * chunks_per;
    ChunkData cur = load_chunk(a, snap, j * kChunk);
    for (; ch < total; ch += gridDim.x) {
        uint32_t nsnap = snap + step_s, nj = j + step_j;
        if (nj >= chunks_per) {
            nj -= chunks_per;
            ++nsnap;
        }
        ChunkData next;
        if (ch + gridDim.x < total) next = load_chunk(a, nsnap, nj * kChunk);
        const uint64_t c0 = (uint64_t)j * kChunk;
        switch (a.profile[snap]) {
            case 0: score_chunk<0, LB>(a, c, lut, cur, snap, c0); break;
            case 1: score_chunk<1, LB>(a, c, lut, cur, snap, c0); break;
            case 2: score_chunk<2, LB>(a, c, lut, cur, snap, c0); break;
            case 3: score_chunk<3, LB>(a, c, lut, cur, snap, c0); break;
            case 4: score_chunk<4, LB>(a, c, lut, cur, snap, c0); break;
            default: score_chunk<5, LB>(a, c, lut, cur, snap, c0); break;
        }
        cur = next;
        snap = nsnap;
        j = nj;
    }
}

__global__ void score_init_kernel(uint64_t* out, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        out[2 * i] = ~0ull;  // no candidate yet
        out[2 * i + 1] = 0;  // (lazy << 32 | busy) candidate counts
    }
}

cudaError_t launch_score(const ScoreArgs& a, cudaStream_t stream) {
    if (!a.n || !a.G) return cudaSuccess;
    score_init_kernel<<<(a.n + 255) / 256, 256, 0, stream>>>(a.out, a.n);
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const uint64_t chunks = ((a.G + kChunk - 1) / kChunk) * a.n;
    if (chunks > 0xFFFFFFFFull) return cudaErrorInvalidValue;
    const uint64_t blocks = std::min<uint64_t>(chunks, (uint64_t)sms * 8);  // 8 x 256 threads per SM
    if (a.lb) score_kernel<true><<<(unsigned)blocks, kScoreThreads, 0, stream>>>(a);
    else score_kernel<false><<<(unsigned)blocks, kScoreThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace msgk
