// Exact-rational fragmentation metric → lookup tables for the kernels.
//
// Restates frag.cpp:12-58 in integer arithmetic over the 7 compute / 8 memory
// slice masks and tabulates it: the 2-mask decision cost
// (frag_cost_masks(busy_c, busy_m), frag.hpp:46-48) depends only on
// (popcount(busy_c), busy_m), and its 2048 values take 31 distinct rationals,
// all integral over 25200 = 420 * 60 (420 = lcm(1..7), 60 = lcm(1..6)).  The
// kernels compare costs by their rank among those values (order-isomorphic
// to Frac's cross-multiplication, frag.hpp:20-25).
#pragma once
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "dev_types.h"

namespace msgk {

inline int host_cs(int p) { return (kCsPack >> (4 * p)) & 0xF; }
inline int host_ms(int p) { return (kMsPack >> (4 * p)) & 0xF; }
inline unsigned host_startmask(int p) { return (unsigned)(kStartMask >> (8 * p)) & 0xFF; }
inline unsigned host_fpm(int p, int s) { return ((1u << host_ms(p)) - 1u) << s; }
inline unsigned host_fpc(int p, int s) { return ((1u << host_cs(p)) - 1u) << s; }

// ideal_from_masks (frag.cpp:12-16)
inline int host_ideal(int pc, int pm, int p) {
    return std::min((7 - pc) / host_cs(p), (8 - pm) / host_ms(p));
}
// feasible_from_masks (frag.cpp:18-26); the compute test is implied by the
// memory test because every footprint has compute ⊆ memory.
inline int host_feasible(unsigned blocked_m, int p) {
    int n = 0;
    for (int s = 0; s < 8; ++s)
        if (((host_startmask(p) >> s) & 1u) && !(host_fpm(p, s) & blocked_m)) ++n;
    return n;
}
// frag_cost_masks (frag.cpp:44-58) as a numerator over 25200.
inline int host_cost_k(int pc, int pm, unsigned blocked_m) {
    long ratio = 0;
    int counted = 0;
    for (int p = 0; p < 6; ++p) {
        const int ideal = host_ideal(pc, pm, p);
        if (ideal == 0) continue;
        ratio += (long)host_feasible(blocked_m, p) * (420 / ideal);
        ++counted;
    }
    if (counted == 0) return 0;
    const long den = 420L * counted;
    return (int)((den - ratio) * (25200 / den));
}

// Every (busy_c, busy_m) produced by a slice-disjoint set of legal
// placements (the states the engine can ever hold), by recursion over the 18
// placements.  mark[pc*256 + bm] = 1 for each reachable pair.
inline void enumerate_reachable(int first, unsigned bc, unsigned bm, std::vector<uint8_t>& mark) {
    mark[__builtin_popcount(bc) * 256 + bm] = 1;
    int idx = 0;
    for (int p = 0; p < 6; ++p)
        for (int s = 0; s < 8; ++s) {
            if (!((host_startmask(p) >> s) & 1u)) continue;
            if (idx++ < first) continue;
            if (host_fpm(p, s) & bm) continue;
            enumerate_reachable(idx, bc | host_fpc(p, s), bm | host_fpm(p, s), mark);
        }
}

// Ranks are assigned over the reachable pairs only (31 distinct costs, the
// survey's exhaustive count); unreachable table entries get rank 31, which
// no engine state can look up.
// The arrival scorer's per-word table (score.cu): for job profile p and a
// GPU word with popc(busy_c) = pc and busy memory = blocked memory = bm (no
// draining instance), candidate_starts + the per-start cost of schedule()
// (scheduler.cpp:19-28,57-66) folded into one u16 entry:
//   bits 10-14  the lowest post-placement cost rank over the available
//               starts (cost2rank[min(pc + cs, 7)][bm | fm(start)])
//   bits 3-9    which starts (ordinals j, start = j * stride) reach it
//   bits 0-2    how many starts are available (the candidate count, <= 7)
// Bit 15 (the Lazy/Busy pass) is filled in per launch from the threshold
// (score.cu, fast_tab_init).  A word without an available start gets
// kScoreNoCand: rank field 31 and, with the pass bit, a key above every
// real one; minimum-start mask 1 keeps the start decode in range; count 0.
constexpr int kScoreTab = 6 * 8 * 256;
constexpr uint16_t kScoreNoCand = 0x7C08;
inline void build_score_table(const DevTables& t, uint16_t* out) {
    for (int p = 0; p < 6; ++p)
        for (int pc = 0; pc < 8; ++pc)
            for (unsigned bm = 0; bm < 256; ++bm) {
                const int row = std::min(pc + host_cs(p), 7);
                unsigned best = 32, mm = 0, cnt = 0, j = 0;
                for (int s = 0; s < 8; ++s) {
                    if (!((host_startmask(p) >> s) & 1u)) continue;
                    const unsigned fm = host_fpm(p, s);
                    if (!(fm & bm)) {
                        const unsigned r = t.cost2rank[row * 256 + (bm | fm)];
                        if (r < best) {
                            best = r;
                            mm = 0;
                        }
                        if (r == best) mm |= 1u << j;
                        ++cnt;
                    }
                    ++j;
                }
                out[(p * 8 + pc) * 256 + bm] = cnt ? (uint16_t)(best << 10 | mm << 3 | cnt) : kScoreNoCand;
            }
}

inline int build_tables(DevTables* t) {
    std::memset(t, 0, sizeof(*t));
    std::vector<uint8_t> mark(8 * 256, 0);
    enumerate_reachable(0, 0, 0, mark);
    std::vector<int> distinct;
    for (int pc = 0; pc < 8; ++pc)
        for (unsigned bm = 0; bm < 256; ++bm)
            if (mark[pc * 256 + bm]) distinct.push_back(host_cost_k(pc, __builtin_popcount(bm), bm));
    std::sort(distinct.begin(), distinct.end());
    distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
    if (distinct.size() > 31) return -1;
    for (int pc = 0; pc < 8; ++pc)
        for (unsigned bm = 0; bm < 256; ++bm) {
            uint8_t r = 31;
            if (mark[pc * 256 + bm]) {
                const int k = host_cost_k(pc, __builtin_popcount(bm), bm);
                r = (uint8_t)(std::lower_bound(distinct.begin(), distinct.end(), k) - distinct.begin());
            }
            t->cost2rank[pc * 256 + bm] = r;
        }
    for (size_t r = 0; r < 32; ++r) t->rank2k[r] = r < distinct.size() ? (uint16_t)distinct[r] : 0xFFFFu;
    // Feasibility vectors (feasible_from_masks per profile, frag.cpp:18-26) of
    // every blocked mask, and ideal vectors (ideal_from_masks, :12-16) of
    // every (popc busy_c, popc busy_m): 32 and 18 distinct values.
    std::vector<uint32_t> fvecs, ivecs;
    auto intern = [](std::vector<uint32_t>& v, uint32_t x) {
        auto it = std::find(v.begin(), v.end(), x);
        if (it != v.end()) return (int)(it - v.begin());
        v.push_back(x);
        return (int)v.size() - 1;
    };
    for (unsigned km = 0; km < 256; ++km) {
        uint32_t f = 0;
        uint8_t pl = 0;
        for (int p = 0; p < 6; ++p) {
            const int n = host_feasible(km, p);
            f |= (uint32_t)n << (3 * p);
            if (n) pl |= (uint8_t)(1u << p);
        }
        t->feasid[km] = (uint8_t)intern(fvecs, f);
        t->placeable[km] = pl;
    }
    for (int pc = 0; pc < 8; ++pc)
        for (int pm = 0; pm < 9; ++pm) {
            uint32_t v = 0;
            for (int p = 0; p < 6; ++p) v |= (uint32_t)std::max(0, host_ideal(pc, pm, p)) << (3 * p);
            t->idealid[pc * 9 + pm] = (uint8_t)intern(ivecs, v);
        }
    if (fvecs.size() > 32 || ivecs.size() > 32) return -3;
    // 4-mask cost (frag_cost_exact, frag.cpp:60-63) of each (ideal, feasible)
    // vector pair; doubles are the correctly rounded k/25200, equal to the
    // reference's Frac::to_double (num/den of the same rational).
    std::vector<int> k4(32 * 32, 0);
    for (size_t i = 0; i < ivecs.size(); ++i)
        for (size_t f = 0; f < fvecs.size(); ++f) {
            long ratio = 0;
            int counted = 0;
            for (int p = 0; p < 6; ++p) {
                const int ideal = (ivecs[i] >> (3 * p)) & 7, feas = (fvecs[f] >> (3 * p)) & 7;
                if (ideal == 0) continue;
                ratio += (long)feas * (420 / ideal);
                ++counted;
            }
            k4[i * 32 + f] = counted ? (int)((420L * counted - ratio) * (60 / counted)) : 0;
        }
    std::vector<int> d4 = k4;
    std::sort(d4.begin(), d4.end());
    d4.erase(std::unique(d4.begin(), d4.end()), d4.end());
    if (d4.size() > 256) return -2;
    for (size_t i = 0; i < k4.size(); ++i)
        t->cost4pair[i] = (uint8_t)(std::lower_bound(d4.begin(), d4.end(), k4[i]) - d4.begin());
    for (int p = 0; p < 6; ++p)
        for (int s = 0; s < 8; ++s) {
            const unsigned m = host_fpm(p, s) & 0xFFu;
            t->share_run[p * 8 + s] = (host_fpc(p, s) & 0x7Fu) | (m << 8) | (m << 16) | (1u << 24);
        }
    for (size_t i = 0; i < 256; ++i) {
        t->cost4val[i] = i < d4.size() ? (double)d4[i] / 25200.0 : 0.0;
        t->cost4k[i] = i < d4.size() ? (uint16_t)d4[i] : 0;
    }
    return (int)distinct.size();
}

inline int n_reachable_pairs() {
    std::vector<uint8_t> mark(8 * 256, 0);
    enumerate_reachable(0, 0, 0, mark);
    int n = 0;
    for (uint8_t m : mark) n += m;
    return n;
}

}  // namespace msgk
