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
// Per word the hot path is one lookup.  With load balancing and dynamic
// partitioning (the schedule() default), a word whose blocked memory equals
// its busy memory (no draining instance — every word of a run without
// migration overlap) is scored from stab[profile][popc busy_c][busy_m]
// (build_score_table): the lowest post-placement cost rank over the
// available starts, which starts reach it, and how many starts are
// available.  The word's key is then assembled with a few ALU ops: the pass
// bit from the classification (classify, gpu.cpp:168-177: Lazy = 0, Busy =
// 1), the rank, !reused (an idle instance of exactly the profile at one of
// the minimum-rank starts, scheduler.cpp:62-66 — the idle-exact bits ride in
// the word), the word index and the start.  Since Lazy keys sort below Busy
// keys, ONE pass over the words yields schedule()'s two-pass answer
// (scheduler.cpp:57-80: Busy GPUs only when no Lazy GPU has a candidate);
// candidate counts are kept per class.  Words with a draining instance, and
// the !dyn / first-fit variants, take the per-start path (tables in shared
// memory, or in global memory for the rare draining word).
//
// The TMA kernel's default path keeps key-only item keys [pass|rank|
// !reused|word] (MSG_SCORE_KF): the start is recovered once per snapshot
// from the winning word (with_start), and a snapshot that is one item is
// finished by the block that scored it (no merge kernel).
//
// Bound: HBM bandwidth — 8 B per scored GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "decide.h"
#include "dev_types.h"

namespace msgk {

#ifndef MSG_SCORE_THREADS
#define MSG_SCORE_THREADS 512  // 2 blocks x 16 warps per SM: room for the key-form table (48 KiB) + a 64 KiB ring
#endif
constexpr int kScoreThreads = MSG_SCORE_THREADS;
#ifndef MSG_SCORE_WPT
#define MSG_SCORE_WPT 8
#endif
#ifndef MSG_SCORE_MINB
#define MSG_SCORE_MINB 2
#endif
#ifndef MSG_SCORE_KF
#define MSG_SCORE_KF 1  // key-only per-word keys, the start recovered once per snapshot (with_start)
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
//    from the blocked mask km (gpu.cpp:146-156: availability = disjointness),
//    and the number of such starts << 8;
//  bct[p * 128 + busy_c]: 4 * 256 * min(popc(busy_c) + cs_p, 7) | !lazy << 31
//    | (lazy ? 16 : 0) (classify, gpu.cpp:168-177, through the host-built lazy
//    mask; the low field is the shift that files the word's candidate count
//    under Lazy (high half) or Busy (low half) of a packed counter).
struct ScoreSmem {
    uint32_t rank26[2304];
    uint32_t bct[6 * 128];
    uint16_t avail[6 * 256];
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
        s.avail[i] = (uint16_t)(a | (unsigned)__popc(a) << 8);
    }
    for (unsigned i = threadIdx.x; i < 6 * 128; i += blockDim.x) {
        const unsigned p = i >> 7, pc = (unsigned)__popc(i & 0x7Fu);
        const unsigned cs = (kCsPack >> (4 * p)) & 0xFu;
        const unsigned lazy = (lazymask >> pc) & 1u;
        s.bct[i] = (min(pc + cs, 7u) << 10) | ((lazy ^ 1u) << 31) | (lazy << 4);
    }
}

// The per-word table of the default (load balancing + dynamic
// partitioning) path (host_tables.h, build_score_table), copied into shared
// memory once per block with the pass bit (bit 15: Busy) of each entry's
// popc(busy_c) set from this launch's threshold; NoTab for the other
// variants.  Keys at or above kNoCandKey mean "no candidate".
constexpr int kScoreTabEntries = 6 * 8 * 256;
constexpr unsigned kNoCandEntry = 0xFC08u;
constexpr unsigned kNoCandKey = 0xFC000000u;
struct FastTab {
    uint16_t t[kScoreTabEntries];
};
struct NoTab {};

__device__ __forceinline__ void fast_tab_init(FastTab& s, const uint16_t* g, unsigned lazymask) {
    const uint4* src = reinterpret_cast<const uint4*>(g);
    uint4* dst = reinterpret_cast<uint4*>(s.t);
    for (unsigned i = threadIdx.x; i < kScoreTabEntries / 8; i += blockDim.x) {
        // 8 entries of one (profile, pc) row: pc = (entry >> 8) & 7
        const unsigned pc = ((i * 8u) >> 8) & 7u;
        const unsigned pass = (((lazymask >> pc) & 1u) ^ 1u) * 0x80008000u;
        uint4 v = __ldg(src + i);
        // entries without a candidate (count 0) always carry the pass bit
        auto fix = [&](unsigned x) {
            unsigned y = x | pass;
            y |= ((x & 0x7u) == 0 ? 0x8000u : 0u) | (((x >> 16) & 0x7u) == 0 ? 0x80000000u : 0u);
            return y;
        };
        v.x = fix(v.x);
        v.y = fix(v.y);
        v.z = fix(v.z);
        v.w = fix(v.w);
        dst[i] = v;
    }
}

// Running per-thread state of one item.
struct ItemAcc {
    unsigned best;   // item-local key minimum
    unsigned cnt;    // candidates: Lazy << 16 | Busy
    unsigned anyx;   // idle-exact bits of the profile seen in the current chunk
};

// candidate_starts (scheduler.cpp:19-28) of one GPU word folded into the
// running minimum.  With load balancing the key is
// [pass|cost rank|!reused|word|start] (scheduler.cpp:47-81); without it
// (first fit, scheduler.cpp:83-98) the lowest available start of the word
// is the word's candidate: one FFS.  REUSE selects the rescoring pass that
// clears !reused on idle-exact starts.
template <int P, bool LB, bool DYN, bool REUSE>
__device__ __forceinline__ void score_word(const ScoreSmem& sm, uint64_t w, unsigned local, ItemAcc& acc,
                                           bool valid = true) {
    using Q = Prof<P>;
    const unsigned lo = (unsigned)w;
    unsigned A = sm.avail[P * 256 + ((lo >> 16) & 0xFFu)];  // starts | count << 8
    if (!valid) A = 0;  // a placeholder word: no candidate, no count
    if (!DYN) {  // candidate_starts: exact idle instances only
        A &= (unsigned)(w >> (24 + Q::pbase)) & ((1u << Q::n) - 1u);
        A |= (unsigned)__popc(A) << 8;
    }
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
            acc.cnt += __funnelshift_l(0u, A >> 8, v);  // (A >> 8) << (v & 31)
            if (DYN) acc.anyx |= (unsigned)((w & Q::xmask) >> 24);
        }
    } else if (!REUSE) {
        const unsigned a7 = A & 0x7Fu;
        const unsigned key = (local << 3) | ((unsigned)(__ffs(a7) - 1) * Q::stride);
        acc.best = a7 ? min(acc.best, key) : acc.best;
    }
}

// Per-start scoring of one word of profile P with load balancing and
// dynamic partitioning, tables read from global memory (L1): the rare words
// with a draining instance (blocked memory != busy memory).  Returns the
// word's minimum key (x) and its candidate count filed under Lazy << 16 or
// Busy (y).
template <int P>
__device__ __noinline__ uint2 score_word_generic(const DevTables* tb, uint64_t w, unsigned local, unsigned lazymask) {
    using Q = Prof<P>;
    const unsigned lo = (unsigned)w;
    const unsigned pc = (unsigned)__popc(lo & 0x7Fu), bm = (lo >> 8) & 0xFFu, km = (lo >> 16) & 0xFFu;
    const unsigned row = min(pc + Q::cs, 7u);
    const unsigned busy = ((lazymask >> pc) & 1u) ^ 1u;
    const unsigned ex = (unsigned)(w >> (24 + Q::pbase));
    unsigned best = 0xFFFFFFFFu, n = 0;
#pragma unroll
    for (unsigned j = 0; j < Q::n; ++j) {
        if (Q::fm(j) & km) continue;
        ++n;
        const unsigned r = __ldg(&tb->cost2rank[row * 256 + (bm | Q::fm(j))]);
        const unsigned key = (busy << 31) | (r << 26) | ((((ex >> j) & 1u) ^ 1u) << 25) | (local << 3) |
                             (j * Q::stride);
        best = min(best, key);
    }
    return make_uint2(best, n << (busy ? 0 : 16));
}

// One word of profile P with load balancing and dynamic partitioning: one
// lookup in the per-profile table T = shared table + P * 2048.
// Branch-free; returns false (and contributes nothing) for a word with a
// draining instance, which the caller rescores with score_word_generic.
// lk3 = the word's item-local index << 3.
template <int P>
__device__ __forceinline__ bool score_word_fast(const uint16_t* T, uint64_t w, unsigned lk3, ItemAcc& acc) {
    using Q = Prof<P>;
    const unsigned lo = (unsigned)w;
    const unsigned pc = (unsigned)__popc(lo & 0x7Fu);
    const unsigned bm = (lo >> 8) & 0xFFu;
    const bool plain = ((lo ^ (lo >> 8)) & 0xFF00u) == 0;  // blocked memory == busy memory: no draining
    unsigned e = T[pc * 256u + bm];
    e = plain ? e : kNoCandEntry;
    const unsigned mm = (e >> 3) & 0x7Fu;                      // minimum-rank starts
    const unsigned r = mm & (unsigned)(w >> (24 + Q::pbase));  // ... with an idle-exact instance
    const unsigned sel = r ? r : mm;
    const unsigned j = (unsigned)__ffs(sel) - 1u;
    const unsigned key = ((e >> 10) << 26) | (r ? 0u : 1u << 25) | lk3 | (j * Q::stride);
    acc.best = min(acc.best, key);
    acc.cnt += (e & 7u) << ((~e >> 11) & 16u);  // Lazy (pass 0) candidates in the high half
    return plain;
}

// The per-word table in key form (MSG_SCORE_T32, the TMA kernel's default
// path): one 32-bit entry per (profile, popc busy_c, busy_m), built per block
// from the 16-bit table and the launch's threshold.  Bits: 31 pass (Busy),
// 30..26 cost rank, 25 !reused, 2..0 the first minimum-rank start — i.e. the
// key of a word without an idle-exact instance, less its index; 21..15 the
// minimum-rank starts (reuse check); 14..9 / 8..3 the candidate count when
// the row is Busy / Lazy (summed per chunk in these fields).  A word then
// costs one LOP3 for its key and one AND + ADD for its counts.
constexpr int kScoreTab32Bytes = kScoreTabEntries * 4;
constexpr unsigned kNoCand32 = 0xFE000007u;  // key >= kNoCandKey, no counts, no starts

__device__ __forceinline__ void fast_tab32_init(uint32_t* t, const uint16_t* g, unsigned lazymask) {
    for (unsigned i = threadIdx.x; i < (unsigned)kScoreTabEntries; i += blockDim.x) {
        const unsigned e = __ldg(g + i);
        const unsigned p = i >> 11, pc = (i >> 8) & 7u;
        const unsigned cnt = e & 7u, mm = (e >> 3) & 0x7Fu, rank = (e >> 10) & 0x1Fu;
        const unsigned busy = ((lazymask >> pc) & 1u) ^ 1u;
        const unsigned stride = (kStridePack >> (4 * p)) & 0xFu;
        unsigned v = kNoCand32;
        if (cnt) {
            const unsigned j0 = (unsigned)__ffs(mm) - 1u;
            v = (busy << 31) | (rank << 26) | (1u << 25) | (mm << 15) | (cnt << (busy ? 9 : 3)) | (j0 * stride);
        }
        t[i] = v;
    }
}

template <int P>
__device__ __forceinline__ bool score_word_fast32(const uint32_t* T, uint64_t w, unsigned lk3, ItemAcc& acc,
                                                  unsigned& cnt) {
    using Q = Prof<P>;
    const unsigned lo = (unsigned)w;
    const unsigned pc = (unsigned)__popc(lo & 0x7Fu);
    const unsigned bm = (lo >> 8) & 0xFFu;
    const bool plain = ((lo ^ (lo >> 8)) & 0xFF00u) == 0;  // blocked memory == busy memory: no draining
    unsigned e = T[pc * 256u + bm];
    e = plain ? e : kNoCand32;
    unsigned key = (e & 0xFE000007u) | lk3;
    // minimum-rank starts with an idle-exact instance: reuse it (cleared
    // !reused bit, its lowest start; scheduler.cpp:62-66)
    const unsigned r = (e >> 15) & (unsigned)(w >> (24 + Q::pbase)) & 0x7Fu;
    if (r) key = (key & ~0x02000007u) | (((unsigned)__ffs(r) - 1u) * Q::stride);
    acc.best = min(acc.best, key);
    cnt += e & 0x7FF8u;
    return plain;
}

#if MSG_SCORE_KF
// The key-only form (MSG_SCORE_KF, default): the start is not carried in the
// key — the item keys hold [pass|rank|!reused|word] and the winning word's
// start is recovered once per snapshot (with_start: in the scoring grid when
// the snapshot is one item, else in score_reduce_kernel) — so a
// word costs fewer ALU ops: no start field, no per-word draining test (the
// busy/blocked XORs are ORed per thread and a thread that saw a draining
// word rescores its chunk), counts summed unmasked.  Entry bits: 31 pass
// (Busy), 30..26 cost rank, 25 !reused (the key, less the word index);
// 18..12 the minimum-rank starts (reuse check against the word's idle-exact
// bits shifted to 12); 11..6 / 5..0 the candidate count when the row is Lazy
// / Busy (a thread sums at most 8 words x 7 starts = 56 per field, so the
// fields never carry; the bits above them are don't-care in the sum).
constexpr unsigned kNoCandKf = 0xFE000000u;  // key >= kNoCandKey, no counts, no starts

__device__ __forceinline__ void fast_tabkf_init(uint32_t* t, const uint16_t* g, unsigned lazymask) {
    for (unsigned i = threadIdx.x; i < (unsigned)kScoreTabEntries; i += blockDim.x) {
        const unsigned e = __ldg(g + i);
        const unsigned pc = (i >> 8) & 7u;
        const unsigned cnt = e & 7u, mm = (e >> 3) & 0x7Fu, rank = (e >> 10) & 0x1Fu;
        const unsigned busy = ((lazymask >> pc) & 1u) ^ 1u;
        t[i] = cnt ? (busy << 31) | (rank << 26) | (1u << 25) | (mm << 12) | (cnt << (busy ? 0 : 6)) : kNoCandKf;
    }
}

template <int P>
__device__ __forceinline__ void score_word_kf(const uint32_t* T, uint64_t w, unsigned l, unsigned& best,
                                              unsigned& cnt, unsigned& dr) {
    using Q = Prof<P>;
    const unsigned lo = (unsigned)w;
    dr |= lo ^ (lo >> 8);  // bits 15..8: busy memory ^ blocked memory (a draining instance)
    const unsigned e = T[(unsigned)__popc(lo & 0x7Fu) * 256u + ((lo >> 8) & 0xFFu)];
    // a minimum-rank start with an idle-exact instance: reuse it (!reused
    // cleared; scheduler.cpp:62-66)
    const bool reuse = (e & (unsigned)(w >> (12 + Q::pbase)) & 0x7F000u) != 0;
    best = min(best, (e & (reuse ? 0xFC000000u : 0xFE000000u)) | l);
    cnt += e;
}

template <int P, int NW2>
__device__ __forceinline__ void score_words_fast32(const uint32_t* T, const DevTables* tb, const ulonglong2 (&x)[NW2],
                                                   unsigned l0, unsigned lazymask, ItemAcc& acc) {
    const unsigned best0 = acc.best;
    unsigned cnt = 0, dr = 0;
#pragma unroll
    for (int k = 0; k < NW2; ++k) {
        const unsigned l = l0 + (unsigned)k * 2 * kScoreThreads;
        score_word_kf<P>(T, x[k].x, l, acc.best, cnt, dr);
        score_word_kf<P>(T, x[k].y, l + 1u, acc.best, cnt, dr);
    }
    if (__builtin_expect(__any_sync(0xffffffffu, (dr & 0xFF00u) != 0), 0)) {
        if (dr & 0xFF00u) {  // this thread saw a draining word: rescore its words
            unsigned best = best0, c2 = 0, d2 = 0;
#pragma unroll
            for (int k = 0; k < 2 * NW2; ++k) {  // static indices: the words stay in registers
                const uint64_t w = (k & 1) ? x[k >> 1].y : x[k >> 1].x;
                const unsigned l = l0 + (unsigned)(k >> 1) * 2 * kScoreThreads + (unsigned)(k & 1);
                const unsigned lo = (unsigned)w;
                if (((lo ^ (lo >> 8)) & 0xFF00u) == 0) {
                    score_word_kf<P>(T, w, l, best, c2, d2);
                } else {
                    const uint2 g = score_word_generic<P>(tb, w, l, lazymask);
                    best = min(best, (g.x & 0xFE000000u) | l);
                    acc.cnt += g.y;
                }
            }
            acc.best = best;
            cnt = c2;
        }
    }
    acc.cnt += (((cnt >> 6) & 63u) << 16) + (cnt & 63u);  // Lazy in the high half
}
#else
template <int P, int NW2>
__device__ __forceinline__ void score_words_fast32(const uint32_t* T, const DevTables* tb, const ulonglong2 (&x)[NW2],
                                                   unsigned l0, unsigned lazymask, ItemAcc& acc) {
    unsigned slow = 0, cnt = 0;
#pragma unroll
    for (int k = 0; k < NW2; ++k) {
        const unsigned l3 = (l0 + (unsigned)k * 2 * kScoreThreads) << 3;
        slow |= (score_word_fast32<P>(T, x[k].x, l3, acc, cnt) ? 0u : 1u) << (2 * k);
        slow |= (score_word_fast32<P>(T, x[k].y, l3 + 8u, acc, cnt) ? 0u : 1u) << (2 * k + 1);
    }
    acc.cnt += (((cnt >> 3) & 63u) << 16) + ((cnt >> 9) & 63u);  // Lazy in the high half
    if (__builtin_expect(__any_sync(0xffffffffu, slow != 0), 0)) {
#pragma unroll
        for (int k = 0; k < 2 * NW2; ++k) {  // static indices: the words stay in registers
            if ((slow >> k) & 1u) {
                const uint64_t w = (k & 1) ? x[k >> 1].y : x[k >> 1].x;
                const uint2 g = score_word_generic<P>(tb, w, l0 + (unsigned)(k >> 1) * 2 * kScoreThreads + (k & 1),
                                                      lazymask);
                acc.best = min(acc.best, g.x);
                acc.cnt += g.y;
            }
        }
    }
}
#endif

// The thread's words of one chunk (x[k].x at local index l_k, x[k].y at
// l_k + 1), all through the table, then the draining ones (if any in the
// warp) through the per-start path.
template <int P, int NW2>
__device__ __forceinline__ void score_words_fast(const uint16_t* T, const DevTables* tb, const ulonglong2 (&x)[NW2],
                                                 unsigned l0, unsigned lazymask, ItemAcc& acc) {
    unsigned slow = 0;
#pragma unroll
    for (int k = 0; k < NW2; ++k) {
        const unsigned l3 = (l0 + (unsigned)k * 2 * kScoreThreads) << 3;
        slow |= (score_word_fast<P>(T, x[k].x, l3, acc) ? 0u : 1u) << (2 * k);
        slow |= (score_word_fast<P>(T, x[k].y, l3 + 8u, acc) ? 0u : 1u) << (2 * k + 1);
    }
    if (__builtin_expect(__any_sync(0xffffffffu, slow != 0), 0)) {
#pragma unroll
        for (int k = 0; k < 2 * NW2; ++k) {  // static indices: the words stay in registers
            if ((slow >> k) & 1u) {
                const uint64_t w = (k & 1) ? x[k >> 1].y : x[k >> 1].x;
                const uint2 g = score_word_generic<P>(tb, w, l0 + (unsigned)(k >> 1) * 2 * kScoreThreads + (k & 1),
                                                      lazymask);
                acc.best = min(acc.best, g.x);
                acc.cnt += g.y;
            }
        }
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

template <int P>
__device__ __forceinline__ void score_chunk_fast(const uint16_t* T, const ScoreArgs& a, const ChunkData& d,
                                                 unsigned base, ItemAcc& acc) {
    score_words_fast<P>(T, a.tables, d.v, base + threadIdx.x * 2u, a.lazymask, acc);
}

// Work cursor over the flattened (item, chunk) sequence of one block.
struct Cursor {
    uint32_t item, snap, chunk, end;  // current item, its snapshot, chunk index, item end chunk
    uint32_t prof;                    // the snapshot's job profile (loaded with the item's first chunk)
};

// End of an item: the warp's minimum key, rebased from the item-local word
// index to the global GPU index, and its candidate counts, merged into the
// snapshot's slots with one 64-bit atomicMin / atomicAdd.
template <bool LB>
__device__ __forceinline__ void flush_item(const ScoreArgs& a, const ItemAcc& acc, uint32_t snap, uint32_t first) {
    unsigned best = __reduce_min_sync(0xffffffffu, acc.best);
    best = best >= kNoCandKey ? 0xFFFFFFFFu : best;  // the table's no-candidate entries
    const unsigned cnt = LB ? __reduce_add_sync(0xffffffffu, acc.cnt) : 0u;
    if ((threadIdx.x & 31) == 0) {
        if (best != 0xFFFFFFFFu) {
            // item-local [pass|rank|!reused|word|start] -> global [pass|rank|!reused|gpu:32|start]
            const uint64_t gpu = (uint64_t)first * kChunk + ((best >> 3) & ((1u << 22) - 1u));
            const uint64_t g64 = ((uint64_t)(best >> 25) << 35) | (gpu << 3) | (best & 7u);
            atomicMin(reinterpret_cast<unsigned long long*>(a.out + 2 * snap), (unsigned long long)g64);
        }
        if (LB && cnt)
            atomicAdd(reinterpret_cast<unsigned long long*>(a.out + 2 * snap + 1),
                      ((unsigned long long)(cnt >> 16) << 32) | (cnt & 0xFFFFu));
    }
}

// Scores `c` (the cursor's chunk) while the following chunk loads into
// `n`; advances the cursor; true when the item is finished.
template <int P, bool LB, bool DYN>
__device__ __forceinline__ bool score_step(const ScoreArgs& a, const ScoreSmem& sm, const uint16_t* T,
                                           const ChunkData& c, ChunkData& n, Cursor& cu, ItemAcc& acc, uint32_t first,
                                           uint32_t chunks_per, uint32_t n_items, uint32_t items_per) {
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
    if (more) n = load_chunk(a, nx.snap, (uint64_t)nx.chunk * kChunk);
    const unsigned base = (cu.chunk - first) * kChunk;
    if constexpr (LB && DYN) {
        score_chunk_fast<P>(T + P * 2048, a, c, base, acc);
    } else {
        acc.anyx = 0;
        score_chunk<P, LB, DYN, false>(sm, c, base, acc);
    }
    const bool done = nx.item != cu.item || !more;
    cu = nx;
    return done;
}

// TMA path: the end of an item reduces each warp's key and counts into the
// block's per-warp slots (double-buffered by stage parity); thread 0 folds
// them after the stage barrier into the item's own output slot — no
// atomics, no output initialisation (score_reduce_kernel merges the items).
struct WarpPart {
    unsigned best, cnt;
};

template <bool LB>
__device__ __forceinline__ void stash_item(const ItemAcc& acc, WarpPart* wpart) {
    unsigned best = __reduce_min_sync(0xffffffffu, acc.best);
    best = best >= kNoCandKey ? 0xFFFFFFFFu : best;  // the table's no-candidate entries
    const unsigned cnt = LB ? __reduce_add_sync(0xffffffffu, acc.cnt) : 0u;
    if ((threadIdx.x & 31) == 0) wpart[threadIdx.x >> 5] = WarpPart{best, cnt};
}

// One item: its chunks are scored with the profile's specialised code while
// the following chunk (possibly the next item's first) is in flight.
template <int P, bool LB, bool DYN>
__device__ __forceinline__ void score_item(const ScoreArgs& a, const ScoreSmem& sm, const uint16_t* T, ChunkData& cur,
                                           Cursor& cu, uint32_t chunks_per, uint32_t n_items, uint32_t items_per) {
    ItemAcc acc{0xFFFFFFFFu, 0u, 0u};
    const uint32_t snap = cu.snap, first = cu.chunk;
    for (;;) {  // the following chunk loads while this one is scored
        ChunkData next;
        const bool done = score_step<P, LB, DYN>(a, sm, T, cur, next, cu, acc, first, chunks_per, n_items, items_per);
        cur = next;
        if (done) break;
    }
    flush_item<LB>(a, acc, snap, first);
}

// Register-streaming path: the fallback when the snapshot rows are not
// 16-byte aligned (odd G or an unaligned words pointer) — one pass with the
// full key, words in registers (the profile-specialised unrolled code needs
// the whole register file: one block per SM, no spills).
template <bool LB, bool DYN>
__global__ void __launch_bounds__(kScoreThreads, 1) score_kernel(ScoreArgs a) {
    __shared__ __align__(16) ScoreSmem sm;
    __shared__ __align__(16) std::conditional_t<LB && DYN, FastTab, NoTab> ft;
    const uint16_t* T = nullptr;
    if constexpr (LB && DYN) {
        fast_tab_init(ft, a.stab, a.lazymask);
        T = ft.t;
    } else {
        score_smem_init(sm, a.tables, a.lazymask);
    }
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
            case 0: score_item<0, LB, DYN>(a, sm, T, cur, cu, chunks_per, n_items, items_per); break;
            case 1: score_item<1, LB, DYN>(a, sm, T, cur, cu, chunks_per, n_items, items_per); break;
            case 2: score_item<2, LB, DYN>(a, sm, T, cur, cu, chunks_per, n_items, items_per); break;
            case 3: score_item<3, LB, DYN>(a, sm, T, cur, cu, chunks_per, n_items, items_per); break;
            case 4: score_item<4, LB, DYN>(a, sm, T, cur, cu, chunks_per, n_items, items_per); break;
            default: score_item<5, LB, DYN>(a, sm, T, cur, cu, chunks_per, n_items, items_per); break;
        }
    }
}

// ---------------------------------------------------------------------------
// TMA-fed variant (the default when the snapshot rows are 16-byte aligned:
// even G, 16-byte aligned words).  One elected thread streams the block's
// chunk sequence into a kStages-deep ring of shared-memory buffers with 1-D
// bulk async copies (cp.async.bulk ... mbarrier::complete_tx), so each SM
// keeps kStages x 8 KiB x blocks of HBM reads in flight without holding them
// in registers; the block consumes a stage after its mbarrier phase
// completes (LDS.128 per two words) and hands it back with one
// __syncthreads.  Per-stage metadata (snapshot, item base, valid words,
// profile, item end) travels with the copy.
#ifndef MSG_SCORE_STAGES
#define MSG_SCORE_STAGES 2
#endif
constexpr int kStages = MSG_SCORE_STAGES;

struct StageMeta {
    uint32_t snap;    // 0xFFFFFFFF: end of the block's sequence
    uint32_t base;    // item-local index of the chunk's first word
    uint32_t nvalid;  // words copied (< kChunk only in a snapshot's last chunk)
    uint32_t prof;    // the snapshot's job profile
    uint32_t first;   // first chunk of the item
    uint32_t last;    // chunk ends its item
    uint32_t pad[2];
};

// The stage ring lives in dynamic shared memory (beyond the 48 KiB static limit).
struct TmaSmem {
    const ScoreSmem* t;       // static: the per-start scoring tables (generic variants)
    const uint16_t* ft;       // static: the per-word table (load balancing + dynamic partitioning)
    const uint32_t* ft32;     // dynamic: the same in key form (MSG_SCORE_T32)
    uint64_t (*buf)[kChunk];  // [kStages][kChunk]
    uint64_t* full;           // [kStages]
    StageMeta* meta;          // [kStages]
};
constexpr size_t kTmaDynBytes = sizeof(uint64_t) * kChunk * kStages + 8 * kStages + sizeof(StageMeta) * kStages;
#ifndef MSG_SCORE_T32
#define MSG_SCORE_T32 1
#endif
// the default-path kernel (load balancing + dynamic partitioning) keeps the
// key-form table in front of its ring
constexpr size_t kTmaDynBytesFast = kTmaDynBytes + (MSG_SCORE_T32 ? (size_t)kScoreTab32Bytes : 0);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Producer cursor over the block's (item, chunk) sequence (thread 0 only).
struct Producer {
    uint32_t item, snap, chunk, first, end, prof;
    bool done;
};

__device__ __forceinline__ void prod_start_item(const ScoreArgs& a, Producer& p, uint32_t chunks_per,
                                                uint32_t items_per, uint32_t n_items) {
    if (p.item >= n_items) {
        p.done = true;
        return;
    }
    p.snap = p.item / items_per;
    p.first = p.chunk = (p.item - p.snap * items_per) * kItemChunks;
    p.end = min(p.first + kItemChunks, chunks_per);
    p.prof = a.profile[p.snap];
}

// Issue the next chunk of the sequence into `stage` (or the end marker).
__device__ __forceinline__ void prod_issue(const ScoreArgs& a, TmaSmem& sm, Producer& p, int stage,
                                           uint32_t chunks_per, uint32_t items_per, uint32_t n_items) {
    StageMeta& m = sm.meta[stage];
    if (p.done) {
        m.snap = 0xFFFFFFFFu;
        mbar_arrive(&sm.full[stage]);
        return;
    }
    const uint64_t c0 = (uint64_t)p.chunk * kChunk;
    const uint64_t rem = a.G - c0;
    const uint32_t nvalid = rem < (uint64_t)kChunk ? (uint32_t)rem : (uint32_t)kChunk;
    m.snap = p.snap;
    m.base = (p.chunk - p.first) * kChunk;
    m.nvalid = nvalid;
    m.prof = p.prof;
    m.first = p.first;
    m.last = p.chunk + 1 >= p.end;
    if (nvalid < (uint32_t)kChunk) {  // a snapshot's last chunk: the tail reads as fully occupied GPUs
        for (uint32_t i = nvalid; i < (uint32_t)kChunk; ++i) sm.buf[stage][i] = 0xFFFF7Full;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the stage's previous reads precede the copy
    mbar_arrive_tx(&sm.full[stage], nvalid * 8u);
    bulk_load(sm.buf[stage], a.words + (uint64_t)p.snap * a.G + c0, nvalid * 8u, &sm.full[stage]);
    if (++p.chunk >= p.end) {
        p.item += gridDim.x;
        prod_start_item(a, p, chunks_per, items_per, n_items);
    }
}

template <int P, bool LB, bool DYN, bool REUSE>
__device__ __forceinline__ void score_stage(const TmaSmem& sm, int stage, const StageMeta& m, ItemAcc& acc) {
    constexpr uint64_t kFull = 0xFFFF7Full;
    const ulonglong2* v = reinterpret_cast<const ulonglong2*>(sm.buf[stage]);
    const unsigned t2 = threadIdx.x * 2u;
    const bool whole = m.nvalid == (uint32_t)kChunk;
#pragma unroll
    for (int k = 0; k < kWordsPerThread / 2; ++k) {
        const unsigned l = t2 + (unsigned)k * 2 * kScoreThreads;
        const ulonglong2 x = v[threadIdx.x + (unsigned)k * kScoreThreads];
        score_word<P, LB, DYN, REUSE>(*sm.t, whole || l < m.nvalid ? x.x : kFull, m.base + l, acc);
        score_word<P, LB, DYN, REUSE>(*sm.t, whole || l + 1 < m.nvalid ? x.y : kFull, m.base + l + 1, acc);
    }
}

template <int P, bool LB, bool DYN>
__device__ __forceinline__ void consume_stage(const TmaSmem& sm, int stage, const StageMeta& m, ItemAcc& acc,
                                              WarpPart* wpart) {
    acc.anyx = 0;
    score_stage<P, LB, DYN, false>(sm, stage, m, acc);
    if (m.last) {
        stash_item<LB>(acc, wpart);
        acc = ItemAcc{0xFFFFFFFFu, 0u, 0u};
    }
}

// The default path (load balancing + dynamic partitioning): every word of
// the stage scored with one table lookup, Lazy and Busy together in one
// pass (module comment).
template <int P>
__device__ __forceinline__ void consume_fast(const ScoreArgs& a, const TmaSmem& sm, int stage, const StageMeta& m,
                                             ItemAcc& acc, WarpPart* wpart) {
    // a snapshot's last chunk was padded with full-GPU words by the producer
    const ulonglong2* v = reinterpret_cast<const ulonglong2*>(sm.buf[stage]);
    ulonglong2 x[kWordsPerThread / 2];
#pragma unroll
    for (int k = 0; k < kWordsPerThread / 2; ++k) x[k] = v[threadIdx.x + (unsigned)k * kScoreThreads];
#if MSG_SCORE_T32
    score_words_fast32<P>(sm.ft32 + P * 2048, a.tables, x, m.base + threadIdx.x * 2u, a.lazymask, acc);
#else
    score_words_fast<P>(sm.ft + P * 2048, a.tables, x, m.base + threadIdx.x * 2u, a.lazymask, acc);
#endif
    if (m.last) {
        stash_item<true>(acc, wpart);
        acc = ItemAcc{0xFFFFFFFFu, 0u, 0u};
    }
}

// With key-only item keys (MSG_SCORE_KF) the winning word's start is
// recovered here, once per snapshot: the lowest start among the word's
// available starts with the key's cost rank and reuse flag
// (candidate_starts + Candidate::better_than, scheduler.cpp:19-43).
__device__ __forceinline__ unsigned word_start(const DevTables* tb, uint64_t w, unsigned p, unsigned key7) {
    const unsigned lo = (unsigned)w;
    const unsigned cs = (kCsPack >> (4 * p)) & 0xFu, ms = (kMsPack >> (4 * p)) & 0xFu;
    const unsigned n = (kCountPack >> (4 * p)) & 0xFu, st = (kStridePack >> (4 * p)) & 0xFu;
    const unsigned pbase = (0x00B74210u >> (4 * p)) & 0xFu;
    const unsigned pc = (unsigned)__popc(lo & 0x7Fu), bm = (lo >> 8) & 0xFFu, km = (lo >> 16) & 0xFFu;
    const unsigned row = min(pc + cs, 7u);
    const unsigned ex = (unsigned)(w >> (24 + pbase));
    for (unsigned j = 0; j < n; ++j) {
        const unsigned fm = ((1u << ms) - 1u) << (j * st);
        if (fm & km) continue;
        const unsigned r = tb->cost2rank[row * 256 + (bm | fm)];
        if (((r << 1) | (((ex >> j) & 1u) ^ 1u)) == (key7 & 0x3Fu)) return j * st;
    }
    return 0;
}

// The snapshot's merged key with its start filled in (key-only item keys).
__device__ __forceinline__ uint64_t with_start(const ScoreArgs& a, uint32_t s, uint64_t best) {
    const uint64_t gpu = (best >> 3) & 0xFFFFFFFFull;
    const uint64_t w = a.words[(uint64_t)s * a.G + gpu];
    const unsigned p = a.profile[s], lo = (unsigned)w;
    if (((lo ^ (lo >> 8)) & 0xFF00u) == 0) {  // no draining instance: the per-word table's starts
        const unsigned e = a.stab[p * 2048u + (unsigned)__popc(lo & 0x7Fu) * 256u + ((lo >> 8) & 0xFFu)];
        const unsigned mm = (e >> 3) & 0x7Fu, pbase = (0x00B74210u >> (4 * p)) & 0xFu;
        const unsigned sel = ((best >> 35) & 1u) ? mm : mm & (unsigned)(w >> (24 + pbase));
        return best | (uint64_t)(((unsigned)__ffs(sel) - 1u) * ((kStridePack >> (4 * p)) & 0xFu));
    }
    return best | word_start(a.tables, w, p, (unsigned)(best >> 35));
}

template <bool LB, bool DYN>
__global__ void __launch_bounds__(kScoreThreads, MSG_SCORE_MINB) score_tma_kernel(ScoreArgs a) {
    constexpr bool kFast = LB && DYN;
    constexpr bool kT32 = kFast && MSG_SCORE_T32;
    __shared__ __align__(16) std::conditional_t<kT32, NoTab, std::conditional_t<kFast, FastTab, ScoreSmem>> tabs;
    __shared__ WarpPart wpart[2][kScoreThreads / 32];  // item ends, by stage parity
    extern __shared__ __align__(128) unsigned char dyn_smem[];
    unsigned char* ring = dyn_smem + (kT32 ? kScoreTab32Bytes : 0);
    TmaSmem sm{nullptr, nullptr, nullptr, reinterpret_cast<uint64_t(*)[kChunk]>(ring),
               reinterpret_cast<uint64_t*>(ring + sizeof(uint64_t) * kChunk * kStages),
               reinterpret_cast<StageMeta*>(ring + sizeof(uint64_t) * kChunk * kStages + 8 * kStages)};
    // the merge kernel may launch now: it waits for this grid (griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;");
    if constexpr (kT32) {
        uint32_t* t32 = reinterpret_cast<uint32_t*>(dyn_smem);
#if MSG_SCORE_KF
        fast_tabkf_init(t32, a.stab, a.lazymask);
#else
        fast_tab32_init(t32, a.stab, a.lazymask);
#endif
        sm.ft32 = t32;
    } else if constexpr (kFast) {
        fast_tab_init(tabs, a.stab, a.lazymask);
        sm.ft = tabs.t;
    } else {
        score_smem_init(tabs, a.tables, a.lazymask);
        sm.t = &tabs;
    }
    const uint32_t chunks_per = (uint32_t)((a.G + kChunk - 1) / kChunk);
    const uint32_t items_per = (chunks_per + kItemChunks - 1) / kItemChunks;
    const uint32_t n_items = items_per * a.n;
    Producer p;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&sm.full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        p.item = blockIdx.x;
        p.done = false;
        prod_start_item(a, p, chunks_per, items_per, n_items);
        for (int s = 0; s < kStages; ++s) prod_issue(a, sm, p, s, chunks_per, items_per, n_items);
    }
    __syncthreads();
    ItemAcc acc{0xFFFFFFFFu, 0u, 0u};
    for (uint32_t n = 0;; ++n) {
        const int stage = (int)(n % kStages);
        mbar_wait(&sm.full[stage], (n / kStages) & 1u);
        const StageMeta m = sm.meta[stage];
        if (m.snap == 0xFFFFFFFFu) break;
        WarpPart* wp = wpart[n & 1u];
        if constexpr (kFast) {
            switch (m.prof) {
                case 0: consume_fast<0>(a, sm, stage, m, acc, wp); break;
                case 1: consume_fast<1>(a, sm, stage, m, acc, wp); break;
                case 2: consume_fast<2>(a, sm, stage, m, acc, wp); break;
                case 3: consume_fast<3>(a, sm, stage, m, acc, wp); break;
                case 4: consume_fast<4>(a, sm, stage, m, acc, wp); break;
                default: consume_fast<5>(a, sm, stage, m, acc, wp); break;
            }
        } else {
            switch (m.prof) {
                case 0: consume_stage<0, LB, DYN>(sm, stage, m, acc, wp); break;
                case 1: consume_stage<1, LB, DYN>(sm, stage, m, acc, wp); break;
                case 2: consume_stage<2, LB, DYN>(sm, stage, m, acc, wp); break;
                case 3: consume_stage<3, LB, DYN>(sm, stage, m, acc, wp); break;
                case 4: consume_stage<4, LB, DYN>(sm, stage, m, acc, wp); break;
                default: consume_stage<5, LB, DYN>(sm, stage, m, acc, wp); break;
            }
        }
        __syncthreads();  // every thread is done with the stage
        if (threadIdx.x == 0) {
            prod_issue(a, sm, p, stage, chunks_per, items_per, n_items);
            if (m.last) {  // the item's result: min key (rebased to the global GPU index), counts
                unsigned best = 0xFFFFFFFFu, cnt = 0;
                for (int w = 0; w < kScoreThreads / 32; ++w) {
                    best = min(best, wp[w].best);
                    cnt += wp[w].cnt;
                }
                uint64_t g64 = ~0ull;
                if (best != 0xFFFFFFFFu) {
                    if constexpr (kT32 && MSG_SCORE_KF) {  // [pass|rank|!reused|word]; the start: the merge
                        const uint64_t gpu = (uint64_t)m.first * kChunk + (best & ((1u << 22) - 1u));
                        g64 = ((uint64_t)(best >> 25) << 35) | (gpu << 3);
                    } else {
                        const uint64_t gpu = (uint64_t)m.first * kChunk + ((best >> 3) & ((1u << 22) - 1u));
                        g64 = ((uint64_t)(best >> 25) << 35) | (gpu << 3) | (best & 7u);
                    }
                }
                uint64_t* it = a.items + 2 * ((uint64_t)m.snap * items_per + m.first / kItemChunks);
                it[0] = g64;
                it[1] = ((uint64_t)(cnt >> 16) << 32) | (cnt & 0xFFFFu);
            }
        }
    }
    if (items_per == 1) {
        // every snapshot is one item (G <= one item's words): the block
        // finishes the snapshots it scored — no merge kernel; the key-only
        // keys get their start here, one dependent lookup per snapshot,
        // all of the block's snapshots in parallel
        __syncthreads();  // thread 0's item results are visible to the block
        for (uint64_t it = blockIdx.x + (uint64_t)threadIdx.x * gridDim.x; it < n_items;
             it += (uint64_t)blockDim.x * gridDim.x) {
            uint64_t best = a.items[2 * it];
            if (kT32 && MSG_SCORE_KF && best != ~0ull) best = with_start(a, (uint32_t)it, best);
            a.out[2 * it] = best;
            a.out[2 * it + 1] = a.items[2 * it + 1];
        }
    }
}

// After the scoring grid (TMA path): each snapshot's items merge into its
// output — minimum key, summed Lazy/Busy candidate counts.
__global__ void score_reduce_kernel(ScoreArgs a, uint32_t items_per, uint32_t kf) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the scoring grid
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= a.n) return;
    uint64_t best = ~0ull, cnt = 0;
    const uint64_t* it = a.items + 2 * (uint64_t)s * items_per;
    for (uint32_t i = 0; i < items_per; ++i) {
        best = it[2 * i] < best ? it[2 * i] : best;
        cnt += it[2 * i + 1];
    }
    if (kf && best != ~0ull) best = with_start(a, s, best);
    a.out[2 * s] = best;
    a.out[2 * s + 1] = cnt;
}

__global__ void score_init_kernel(uint64_t* out, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        out[2 * i] = ~0ull;  // no candidate yet
        out[2 * i + 1] = 0;  // (lazy << 32 | busy) candidate counts
    }
}

size_t score_items_bytes(uint32_t n, uint64_t G) {
    const uint64_t chunks_per = (G + kChunk - 1) / kChunk;
    return (size_t)n * ((chunks_per + kItemChunks - 1) / kItemChunks) * 2 * sizeof(uint64_t);
}

cudaError_t launch_score(const ScoreArgs& a, cudaStream_t stream) {
    if (!a.n || !a.G) return cudaSuccess;
    static int sms = 0, per_sm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int dyn = (int)kTmaDynBytes;
        cudaFuncSetAttribute(score_tma_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        cudaFuncSetAttribute(score_tma_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        cudaFuncSetAttribute(score_tma_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        cudaFuncSetAttribute(score_tma_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kTmaDynBytesFast);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], score_kernel<false, false>, kScoreThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], score_kernel<false, true>, kScoreThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[2], score_kernel<true, false>, kScoreThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[3], score_kernel<true, true>, kScoreThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[4], score_tma_kernel<false, false>, kScoreThreads, dyn);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[5], score_tma_kernel<false, true>, kScoreThreads, dyn);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[6], score_tma_kernel<true, false>, kScoreThreads, dyn);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[7], score_tma_kernel<true, true>, kScoreThreads,
                                                      kTmaDynBytesFast);
    }
    const uint64_t chunks_per = (a.G + kChunk - 1) / kChunk;
    const uint64_t items = ((chunks_per + kItemChunks - 1) / kItemChunks) * a.n;
    if (chunks_per > 0xFFFFFFFFull || items > 0xFFFFFFFFull) return cudaErrorInvalidValue;
    // bulk copies need 16-byte aligned rows; MSG_SCORE_REG forces the register-streaming kernel
    static const bool force_reg = std::getenv("MSG_SCORE_REG") != nullptr;
    const bool tma = !force_reg && (a.G & 1) == 0 && (reinterpret_cast<uintptr_t>(a.words) & 15) == 0;
    const int v = (tma ? 4 : 0) + (a.lb ? 2 : 0) + (a.dyn ? 1 : 0);
    // persistent grid: exactly the resident blocks (one wave)
    const uint64_t blocks = std::min<uint64_t>(items, (uint64_t)sms * std::max(1, per_sm[v]));
    const dim3 grid((unsigned)blocks), block(kScoreThreads);
    if (!tma) score_init_kernel<<<(a.n + 255) / 256, 256, 0, stream>>>(a.out, a.n);  // register path: atomics
    switch (v) {
        case 0: score_kernel<false, false><<<grid, block, 0, stream>>>(a); break;
        case 1: score_kernel<false, true><<<grid, block, 0, stream>>>(a); break;
        case 2: score_kernel<true, false><<<grid, block, 0, stream>>>(a); break;
        case 3: score_kernel<true, true><<<grid, block, 0, stream>>>(a); break;
        case 4: score_tma_kernel<false, false><<<grid, block, kTmaDynBytes, stream>>>(a); break;
        case 5: score_tma_kernel<false, true><<<grid, block, kTmaDynBytes, stream>>>(a); break;
        case 6: score_tma_kernel<true, false><<<grid, block, kTmaDynBytes, stream>>>(a); break;
        default: score_tma_kernel<true, true><<<grid, block, kTmaDynBytesFast, stream>>>(a); break;
    }
    if (!tma || items / a.n == 1) return cudaGetLastError();  // one item per snapshot: merged in the grid
    // The merge launches as a programmatic dependent: its launch overlaps
    // the scoring grid's tail; griddepcontrol.wait holds its reads until the
    // scoring grid has completed.
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t lc{};
    lc.stream = stream;
    lc.attrs = at;
    lc.numAttrs = 1;
    lc.gridDim = dim3((a.n + 255) / 256);
    lc.blockDim = dim3(256);
    const uint32_t kf = (MSG_SCORE_T32 && MSG_SCORE_KF && a.lb && a.dyn) ? 1u : 0u;
    cudaError_t e = cudaLaunchKernelEx(&lc, score_reduce_kernel, a, (uint32_t)(items / a.n), kf);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace msgk
