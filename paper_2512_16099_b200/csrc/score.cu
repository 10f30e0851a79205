// score.cu — the arrival scorer over large clusters, streamed from HBM.
//
// schedule() / first_fit_schedule() (scheduler.cpp:47-98) for snapshots of
// any size: each GPU is one packed 64-bit state word (busy compute, busy
// memory, blocked memory, 18 idle-exact placement bits; msg_pack_gpu_word).
//
// Work is cut into ITEMS — up to kItemChunks chunks of one snapshot — so the
// job profile is uniform over an item and the scoring loop is specialised
// per profile with compile-time footprints.  A persistent grid (exactly the
// resident blocks) walks items blockIdx.x, +gridDim.x, ...; inside an item
// it streams kChunk-word chunks with 128-bit evict-first loads, the next
// chunk (or the next item's first chunk) always in flight while the current
// one is scored.  Each thread keeps a 32-bit item-local key
// [pass:1|cost rank:5|!reused:1|word:22|start:3]; at the end of the item
// the warp reduces it with one REDUX.MIN, rebases it to the 64-bit global
// key [pass|rank|!reused|gpu:32|start] and merges it per snapshot with one
// atomicMin; Lazy/all candidate counts ride two REDUX.ADD and one atomicAdd.
//
// Per word the hot path is table-driven (tables in shared memory, built
// once per block):
//   bct[p][busy_c]  byte offset of the post-placement LUT row
//                   (popc(busy_c) + cs, capped at 7) | !lazy << 31;
//   avail[p][km]    legal starts memory-disjoint from the blocked mask;
//   rank26[...]     cost rank of (row, busy_m | fm(start)), pre-shifted.
// So a word costs ~12 instructions plus LDS + LOP3 + predicated VIMNMX per
// legal start.  The reuse bit (idle instance of exactly this placement,
// scheduler.cpp:62-66) is resolved off the hot path: words are first scored
// as "not reused"; a warp whose chunk holds any idle-exact bit of the profile
// rescores that chunk with the bit (rare: an idle instance of the very
// profile requested).  Since the reuse-aware key of a candidate is never
// larger than its plain key, the minimum over both passes is exact.
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
#ifndef MSG_SCORE_MINB
#define MSG_SCORE_MINB 4
#endif
#ifndef MSG_SCORE_ITEM
#define MSG_SCORE_ITEM 4
#endif
constexpr int kWordsPerThread = MSG_SCORE_WPT;           // 2, 4 or 8 (1, 2 or 4 128-bit loads)
constexpr int kChunk = kScoreThreads * kWordsPerThread;  // words per chunk
constexpr int kItemChunks = MSG_SCORE_ITEM;              // chunks per item
static_assert((uint64_t)kChunk * kItemChunks <= (1u << 22), "item-local word index is 22 bits");

template <int P>
struct Prof {
    static constexpr unsigned cs = (kCsPack >> (4 * P)) & 0xFu;
    static constexpr unsigned ms = (kMsPack >> (4 * P)) & 0xFu;
    static constexpr unsigned n = (kCountPack >> (4 * P)) & 0xFu;
    static constexpr unsigned stride = (kStridePack >> (4 * P)) & 0xFu;
    static constexpr unsigned pbase = (0x00B74210u >> (4 * P)) & 0xFu;  // first idle-exact bit
    // idle-exact bits of this profile inside the word (bits 24 + pbase ...)
    static constexpr uint64_t xmask = (((1ull << n) - 1ull) << (24 + pbase));
    __host__ __device__ static constexpr unsigned fm(unsigned j) { return ((1u << ms) - 1u) << (j * stride); }
};

// Shared-memory tables of one block.
//  rank26[r * 256 + m]: cost rank of (popc busy_c = r, busy_m = m) pre-shifted
//    to its key position (bit 26); indexed as row + busy_m + fm(start) with an
//    ADD (an overlapping start is unavailable and masked, so the sum only has
//    to stay in bounds: 7 * 256 + 255 + 255 < 2304);
//  avail[p * 256 + km]: bit j set iff start j of profile p is memory-disjoint
//    from the blocked mask km (gpu.cpp:146-156: availability = disjointness);
//  bct[p * 128 + busy_c]: 4 * 256 * min(popc(busy_c) + cs_p, 7) | !lazy << 31
//    (classify, gpu.cpp:168-177, through the host-built lazy mask).
struct ScoreSmem {
    uint32_t rank26[2304];
    uint32_t bct[6 * 128];
    uint8_t avail[6 * 256];
};

__device__ __forceinline__ void score_smem_init(ScoreSmem& s, const DevTables* tb, unsigned lazymask) {
    for (unsigned i = threadIdx.x; i < 2304; i += blockDim.x)
        s.rank26[i] = i < 2048 ? (unsigned)tb->cost2rank[i] << 26 : 0u;
    for (unsigned i = threadIdx.x; i < 6 * 256; i += blockDim.x) {
        const unsigned p = i >> 8, km = i & 0xFFu;
        const unsigned ms = (kMsPack >> (4 * p)) & 0xFu, st = (kStridePack >> (4 * p)) & 0xFu;
        const unsigned n = (kCountPack >> (4 * p)) & 0xFu;
        unsigned a = 0;
        for (unsigned j = 0; j < n; ++j)
            if (!((((1u << ms) - 1u) << (j * st)) & km)) a |= 1u << j;
        s.avail[i] = (uint8_t)a;
    }
    for (unsigned i = threadIdx.x; i < 6 * 128; i += blockDim.x) {
        const unsigned p = i >> 7, pc = (unsigned)__popc(i & 0x7Fu);
        const unsigned cs = (kCsPack >> (4 * p)) & 0xFu;
        s.bct[i] = (min(pc + cs, 7u) << 10) | ((((lazymask >> pc) & 1u) ^ 1u) << 31);
    }
}

// Running per-thread state of one item.
struct ItemAcc {
    unsigned best;   // item-local key minimum
    unsigned all;    // candidates
    unsigned lazy;   // candidates on Lazy GPUs
    unsigned anyx;   // idle-exact bits of the profile seen in the current chunk
};

// candidate_starts (scheduler.cpp:19-28) of one GPU word folded into the
// running minimum.  With load balancing the key is
// [pass|cost rank|!reused|word|start] (scheduler.cpp:47-81); without it
// (first fit, scheduler.cpp:83-98) the lowest available start of the word
// is the word's candidate: one FFS.  REUSE selects the rescoring pass that
// clears !reused on idle-exact starts.
template <int P, bool LB, bool DYN, bool REUSE>
__device__ __forceinline__ void score_word(const ScoreSmem& sm, uint64_t w, unsigned local, ItemAcc& acc) {
    using Q = Prof<P>;
    const unsigned lo = (unsigned)w;
    unsigned A = sm.avail[P * 256 + ((lo >> 16) & 0xFFu)];
    if (!DYN) A &= (unsigned)(w >> (24 + Q::pbase));  // candidate_starts: exact idle instances only
    if (LB) {
        const unsigned v = sm.bct[P * 128 + (lo & 0x7Fu)];
        // row byte offset | busy_m * 4: the LUT row of popc(busy_c | fc), column busy_m
        const uint32_t* rp =
            reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(sm.rank26) + ((v & 0x1C00u) | ((lo >> 6) & 0x3FCu)));
        // without dynamic partitioning every candidate reuses (!reused = 0)
        const unsigned head = (v & 0x80000000u) | (DYN ? (1u << 25) : 0u) | (local << 3);
        if (REUSE) {
            const unsigned ex = (unsigned)(w >> (24 + Q::pbase));
#pragma unroll
            for (unsigned j = 0; j < Q::n; ++j) {
                const unsigned key = (rp[Q::fm(j)] | head | (j * Q::stride)) ^ (((ex >> j) & 1u) << 25);
                acc.best = ((A >> j) & 1u) ? min(acc.best, key) : acc.best;
            }
        } else {
#pragma unroll
            for (unsigned j = 0; j < Q::n; ++j) {
                const unsigned key = rp[Q::fm(j)] | head | (j * Q::stride);
                acc.best = ((A >> j) & 1u) ? min(acc.best, key) : acc.best;
            }
            const unsigned c = __popc(A);
            acc.all += c;
            acc.lazy += (int)v >= 0 ? c : 0u;
            if (DYN) acc.anyx |= (unsigned)((w & Q::xmask) >> 24);
        }
    } else if (!REUSE) {
        const unsigned key = (local << 3) | ((unsigned)(__ffs(A) - 1) * Q::stride);
        acc.best = A ? min(acc.best, key) : acc.best;
    }
}

struct ChunkData {
    ulonglong2 v[kWordsPerThread / 2];
};

// Words [c0, c0 + kChunk) of snapshot `snap`; words past the end read as a
// fully occupied GPU (no candidate).
__device__ __forceinline__ ChunkData load_chunk(const ScoreArgs& a, uint32_t snap, uint64_t c0) {
    constexpr uint64_t kFull = 0xFFFF7Full;
    ChunkData d;
    const uint64_t* words = a.words + (uint64_t)snap * a.G + c0;
    const unsigned t2 = threadIdx.x * 2u;
    if ((a.G & 1) == 0 && c0 + kChunk <= a.G) {  // whole, 16-byte aligned chunk
#pragma unroll
        for (int k = 0; k < kWordsPerThread / 2; ++k)
            d.v[k] = __ldcs(reinterpret_cast<const ulonglong2*>(words + t2 + (unsigned)k * 2 * kScoreThreads));
        return d;
    }
    const uint64_t rem = a.G - c0;
#pragma unroll
    for (int k = 0; k < kWordsPerThread / 2; ++k) {
        const uint64_t g = t2 + (unsigned)k * 2 * kScoreThreads;
        if ((a.G & 1) == 0 && g + 1 < rem) {
            d.v[k] = __ldcs(reinterpret_cast<const ulonglong2*>(words + g));
        } else {
            d.v[k].x = g < rem ? words[g] : kFull;
            d.v[k].y = g + 1 < rem ? words[g + 1] : kFull;
        }
    }
    return d;
}

template <int P, bool LB, bool DYN, bool REUSE>
__device__ __forceinline__ void score_chunk(const ScoreSmem& sm, const ChunkData& d, unsigned base, ItemAcc& acc) {
    const unsigned t2 = threadIdx.x * 2u;
#pragma unroll
    for (int k = 0; k < kWordsPerThread / 2; ++k) {
        const unsigned l = base + t2 + (unsigned)k * 2 * kScoreThreads;
        score_word<P, LB, DYN, REUSE>(sm, d.v[k].x, l, acc);
        score_word<P, LB, DYN, REUSE>(sm, d.v[k].y, l + 1, acc);
    }
}

// Work cursor over the flattened (item, chunk) sequence of one block.
struct Cursor {
    uint32_t item, snap, chunk, end;  // current item, its snapshot, chunk index, item end chunk
    uint32_t prof;                    // the snapshot's job profile (loaded with the item's first chunk)
};

// One item: its chunks are scored with the profile's specialised code while
// the following chunk (possibly the next item's first) is in flight.
template <int P, bool LB, bool DYN>
__device__ __forceinline__ void score_item(const ScoreArgs& a, const ScoreSmem& sm, ChunkData& cur, Cursor& cu,
                                           uint32_t chunks_per, uint32_t n_items, uint32_t items_per) {
    ItemAcc acc{0xFFFFFFFFu, 0u, 0u, 0u};
    const uint32_t snap = cu.snap, first = cu.chunk;
    for (;;) {
        // advance the cursor and prefetch
        Cursor nx = cu;
        bool more = true;
        if (++nx.chunk >= nx.end) {
            nx.item += gridDim.x;
            more = nx.item < n_items;
            if (more) {
                nx.snap = nx.item / items_per;
                nx.chunk = (nx.item - nx.snap * items_per) * kItemChunks;
                nx.end = min(nx.chunk + kItemChunks, chunks_per);
                nx.prof = a.profile[nx.snap];
            }
        }
        ChunkData next;
        if (more) next = load_chunk(a, nx.snap, (uint64_t)nx.chunk * kChunk);
        const unsigned base = (cu.chunk - first) * kChunk;
        acc.anyx = 0;
        score_chunk<P, LB, DYN, false>(sm, cur, base, acc);
        if (LB && DYN && __any_sync(0xffffffffu, acc.anyx != 0)) score_chunk<P, LB, DYN, true>(sm, cur, base, acc);
        const bool done = nx.item != cu.item;
        cur = next;
        cu = nx;
        if (done || !more) break;
    }
    const unsigned best = __reduce_min_sync(0xffffffffu, acc.best);
    unsigned all = 0, lazy = 0;
    if (LB) {
        all = __reduce_add_sync(0xffffffffu, acc.all);
        lazy = __reduce_add_sync(0xffffffffu, acc.lazy);
    }
    if ((threadIdx.x & 31) == 0) {
        if (best != 0xFFFFFFFFu) {
            // item-local [pass|rank|!reused|word|start] -> global [pass|rank|!reused|gpu:32|start]
            const uint64_t gpu = (uint64_t)first * kChunk + ((best >> 3) & ((1u << 22) - 1u));
            const uint64_t g64 = ((uint64_t)(best >> 25) << 35) | (gpu << 3) | (best & 7u);
            atomicMin(reinterpret_cast<unsigned long long*>(a.out + 2 * snap), (unsigned long long)g64);
        }
        if (LB && all)
            atomicAdd(reinterpret_cast<unsigned long long*>(a.out + 2 * snap + 1),
                      ((unsigned long long)lazy << 32) | (all - lazy));
    }
}

template <bool LB, bool DYN>
__global__ void __launch_bounds__(kScoreThreads, MSG_SCORE_MINB) score_kernel(ScoreArgs a) {
    __shared__ __align__(16) ScoreSmem sm;
    score_smem_init(sm, a.tables, a.lazymask);
    __syncthreads();
    const uint32_t chunks_per = (uint32_t)((a.G + kChunk - 1) / kChunk);
    const uint32_t items_per = (chunks_per + kItemChunks - 1) / kItemChunks;
    const uint32_t n_items = items_per * a.n;
    Cursor cu;
    cu.item = blockIdx.x;
    if (cu.item >= n_items) return;
    cu.snap = cu.item / items_per;
    cu.chunk = (cu.item - cu.snap * items_per) * kItemChunks;
    cu.end = min(cu.chunk + kItemChunks, chunks_per);
    cu.prof = a.profile[cu.snap];
    ChunkData cur = load_chunk(a, cu.snap, (uint64_t)cu.chunk * kChunk);
    while (cu.item < n_items) {
        switch (cu.prof) {
            case 0: score_item<0, LB, DYN>(a, sm, cur, cu, chunks_per, n_items, items_per); break;
            case 1: score_item<1, LB, DYN>(a, sm, cur, cu, chunks_per, n_items, items_per); break;
            case 2: score_item<2, LB, DYN>(a, sm, cur, cu, chunks_per, n_items, items_per); break;
            case 3: score_item<3, LB, DYN>(a, sm, cur, cu, chunks_per, n_items, items_per); break;
            case 4: score_item<4, LB, DYN>(a, sm, cur, cu, chunks_per, n_items, items_per); break;
            default: score_item<5, LB, DYN>(a, sm, cur, cu, chunks_per, n_items, items_per); break;
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
    static int sms = 0, per_sm[4] = {0, 0, 0, 0};
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], score_kernel<false, false>, kScoreThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], score_kernel<false, true>, kScoreThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[2], score_kernel<true, false>, kScoreThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[3], score_kernel<true, true>, kScoreThreads, 0);
    }
    const uint64_t chunks_per = (a.G + kChunk - 1) / kChunk;
    const uint64_t items = ((chunks_per + kItemChunks - 1) / kItemChunks) * a.n;
    if (chunks_per > 0xFFFFFFFFull || items > 0xFFFFFFFFull) return cudaErrorInvalidValue;
    // persistent grid: exactly the resident blocks (one wave)
    const int resident = std::max(1, per_sm[(a.lb ? 2 : 0) + (a.dyn ? 1 : 0)]);
    const uint64_t blocks = std::min<uint64_t>(items, (uint64_t)sms * resident);
    const dim3 grid((unsigned)blocks), block(kScoreThreads);
    if (a.lb) {
        if (a.dyn) score_kernel<true, true><<<grid, block, 0, stream>>>(a);
        else score_kernel<true, false><<<grid, block, 0, stream>>>(a);
    } else {
        if (a.dyn) score_kernel<false, true><<<grid, block, 0, stream>>>(a);
        else score_kernel<false, false><<<grid, block, 0, stream>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace msgk
