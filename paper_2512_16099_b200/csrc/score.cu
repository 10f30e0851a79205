// score.cu — the arrival scorer over large clusters, streamed from HBM.
//
// schedule() / first_fit_schedule() (scheduler.cpp:47-98) for snapshots of
// any size: each GPU is one packed 64-bit state word (busy compute, busy
// memory, blocked memory, 18 idle-exact placement bits; msg_pack_gpu_word).
// A persistent grid streams 1024-word chunks of the snapshots with 128-bit
// loads (4 words per thread, issued before use), scores every legal
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
constexpr int kWordsPerThread = 4;
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
template <int P>
__device__ __forceinline__ void score_word(const ScoreCfg& c, const uint8_t* lut, uint64_t w, unsigned local,
                                           unsigned& best, unsigned& cnt_lb) {
    using Q = Prof<P>;
    const unsigned lo = (unsigned)w;
    const unsigned bc = lo & 0x7Fu, bm = (lo >> 8) & 0xFFu, km = (lo >> 16) & 0xFFu;
    const unsigned exact = (unsigned)(w >> (24 + Q::pbase));
    const unsigned pc = __popc(bc);
    const unsigned lazy = (c.lazymask >> pc) & 1u;
    const unsigned head = c.lb ? (((lazy ^ 1u) << 31) | (local << 3)) : (local << 3);
    const unsigned row = min(pc + Q::cs, 7u) * 256u;  // popc(busy_c | fc) when the start is free
    unsigned cnt = 0;
#pragma unroll
    for (unsigned j = 0; j < Q::n; ++j) {
        const unsigned ex = (exact >> j) & 1u;
        if (!(Q::fm(j) & km) && (c.dyn || ex)) {
            ++cnt;
            const unsigned key = c.lb ? (head | ((unsigned)lut[row + (bm | Q::fm(j))] << 26) | ((ex ^ 1u) << 25) |
                                         (j * Q::stride))
                                      : (head | (j * Q::stride));
            best = min(best, key);
        }
    }
    cnt_lb += lazy ? cnt << 16 : cnt;
}

// One chunk of one snapshot: every thread scores kWordsPerThread words,
// loaded up front with 128-bit evict-first loads; the warp's winner and
// candidate counts go straight to the snapshot's slots with one 64-bit
// atomicMin / atomicAdd (no block-level synchronisation).
template <int P>
__device__ __forceinline__ void score_chunk(const ScoreArgs& a, const ScoreCfg& c, const uint8_t* lut,
                                            uint64_t snap, uint64_t c0) {
    const uint64_t* words = a.words + snap * a.G;
    unsigned best = 0xFFFFFFFFu, cnt = 0;
    const unsigned t2 = threadIdx.x * 2u;
    if ((a.G & 1) == 0 && c0 + kChunk <= a.G) {
        ulonglong2 v[kWordsPerThread / 2];
#pragma unroll
        for (int k = 0; k < kWordsPerThread / 2; ++k)
            v[k] = __ldcs(reinterpret_cast<const ulonglong2*>(words + c0 + t2 + (unsigned)k * 2 * kScoreThreads));
#pragma unroll
        for (int k = 0; k < kWordsPerThread / 2; ++k) {
            const unsigned l = t2 + (unsigned)k * 2 * kScoreThreads;
            score_word<P>(c, lut, v[k].x, l, best, cnt);
            score_word<P>(c, lut, v[k].y, l + 1, best, cnt);
        }
    } else {
        for (unsigned l = threadIdx.x; l < kChunk && c0 + l < a.G; l += kScoreThreads)
            score_word<P>(c, lut, words[c0 + l], l, best, cnt);
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
__global__ void __launch_bounds__(kScoreThreads) score_kernel(ScoreArgs a) {
    __shared__ __align__(16) uint8_t lut[8 * 256];
    for (unsigned i = threadIdx.x; i < 8 * 256 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(lut)[i] = reinterpret_cast<const uint4*>(a.tables->cost2rank)[i];
    __syncthreads();
    const ScoreCfg c{a.lb, a.dyn, a.lazymask};
    const uint64_t chunks_per = (a.G + kChunk - 1) / kChunk;
    const uint64_t total = chunks_per * a.n;
    for (uint64_t ch = blockIdx.x; ch < total; ch += gridDim.x) {
        const uint64_t snap = ch / chunks_per;
        const uint64_t c0 = (ch % chunks_per) * kChunk;
        switch (a.profile[snap]) {
            case 0: score_chunk<0>(a, c, lut, snap, c0); break;
            case 1: score_chunk<1>(a, c, lut, snap, c0); break;
            case 2: score_chunk<2>(a, c, lut, snap, c0); break;
            case 3: score_chunk<3>(a, c, lut, snap, c0); break;
            case 4: score_chunk<4>(a, c, lut, snap, c0); break;
            default: score_chunk<5>(a, c, lut, snap, c0); break;
        }
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
    const uint64_t blocks = std::min<uint64_t>(chunks, (uint64_t)sms * 8);  // 8 x 256 threads per SM
    score_kernel<<<(unsigned)blocks, kScoreThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace msgk
