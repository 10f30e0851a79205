// staging.h — host-side validation, staging and decoding shared by the
// product runtime (host_runtime.cpp) and the CPU-side unit-test harness of
// the kernel logic (tests/emu).  No CUDA, no scheduling logic.
#pragma once
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "dev_types.h"
#include "host_tables.h"
#include "migsched_b200.h"

namespace msgk {

inline constexpr uint32_t kMaxGpusEnsemble = 32;          // WarpSmem<8>
inline constexpr uint64_t kMaxJobsPerTrace = 1ull << 22;  // key layout (engine_core.cuh)

inline constexpr const char* kProfileNames[] = {"7g.40gb", "4g.20gb", "3g.20gb",  // profiles.cpp:8-15
                                                "2g.10gb", "1g.10gb", "1g.5gb"};
inline constexpr const char* kStatusNames[] = {"Ok",          "InvalidPlacement", "SlicesBusy",   "UnknownJob", "UnknownGpu",
                              "NotLazy",     "UnknownProfile",   "BadThreshold", "BadConfig",  "BadSpec",
                              "TraceUnsorted", "BadConcurrency", "JobsPending",  "ParseError"};

struct CfgState {
    int32_t status = MSG_OK;
    std::string message;
    DevConfig dev{};
    std::vector<uint32_t> init;
    double overlap = 0.0;
    int32_t gpu_count = 0;
};

// Engine::Engine's configuration checks (sim.cpp:73-95) in the reference's
// order, then this engine's envelope (G <= 32 for the ensemble kernel).
inline CfgState validate_config(const msg_config& c) {
    CfgState s;
    s.gpu_count = c.gpu_count;
    s.overlap = c.migration_overlap_s;
    auto fail = [&](int st, const std::string& m) {
        s.status = st;
        s.message = std::string(kStatusNames[st]) + ": " + m;
        return s;
    };
    if (c.gpu_count < 1) return fail(MSG_ERR_BAD_CONFIG, "cluster must contain at least one GPU");
    if (c.threshold < 0.0 || c.threshold > 1.0)
        return fail(MSG_ERR_BAD_THRESHOLD, "load-balancing threshold must be in [0,1]");
    if (!c.dynamic_partitioning && !c.has_static_layout)
        return fail(MSG_ERR_BAD_CONFIG, "dynamic partitioning is off but no static layout is configured");
    if (!c.dynamic_partitioning) {
        if (c.layout_gpus != c.gpu_count)
            return fail(MSG_ERR_BAD_CONFIG, "static layout must list every GPU in the cluster");
        for (int g = 0; g < c.layout_gpus; ++g) {
            unsigned used = 0;
            for (int i = c.layout_offsets[g]; i < c.layout_offsets[g + 1]; ++i) {
                const int p = c.layout_profile[i], st = c.layout_start[i];
                if (p < 0 || p >= MSG_PROFILE_COUNT)
                    return fail(MSG_ERR_UNKNOWN_PROFILE, "static layout references an unknown profile");
                // add_idle_instance -> slice_footprint (profiles.cpp:49-57)
                if (st < 0 || st > 7 || !((host_startmask(p) >> st) & 1u))
                    return fail(MSG_ERR_INVALID_PLACEMENT, "placement (" + std::to_string(st) + "," +
                                                               std::to_string(host_ms(p)) + ") is not valid for profile " +
                                                               kProfileNames[p]);
                if (host_fpm(p, st) & used)  // gpu.cpp:103-113
                    return fail(MSG_ERR_SLICES_BUSY,
                                "layout instance overlaps an existing instance on GPU " + std::to_string(g));
                used |= host_fpm(p, st);
                s.init.push_back((uint32_t)(g * 8 + st) | ((uint32_t)p << 24));  // slot:24 | profile:8
            }
        }
    }
    if (c.gpu_count >= (1 << 16))  // 16-bit GPU ids in the event records
        return fail(MSG_ERR_UNSUPPORTED, "at most 65535 GPUs per cluster");
    s.dev.alpha = c.contention_alpha;
    s.dev.overlap = c.migration_overlap_s;
    s.dev.latency = c.reconfig_latency_s;
    s.dev.G = c.gpu_count;
    s.dev.flags = (c.load_balancing ? CF_LB : 0u) | (c.dynamic_partitioning ? CF_DYN : 0u) | (c.migration ? CF_MIG : 0u);
    uint32_t lm = 0;
    for (int pc = 0; pc <= 7; ++pc)
        if ((double)pc / 7.0 < c.threshold) lm |= 1u << pc;  // classify (gpu.cpp:168-177)
    s.dev.lazymask = lm;
    s.dev.n_init = (uint32_t)s.init.size();
    return s;
}

// Per-trace validation (sim.cpp:97-116) + rank/permutation staging.
struct TraceCheck {
    int32_t status = MSG_OK;
    std::string message;
    bool identity = true;
};

inline TraceCheck check_trace(const msg_trace_batch* b, uint32_t t) {
    TraceCheck r;
    const uint64_t lo = b->offsets[t], hi = b->offsets[t + 1];
    const uint64_t n = hi - lo;
    {
        // Fast pass, no early exit (vectorisable): any bad profile, unsorted
        // or NaN arrival, non-positive or NaN service, non-increasing ids.
        // A clean trace returns here; anything else takes the exact pass
        // below, which finds the first failure and its message.
        const int32_t* pf = b->profile + lo;
        const double* ar = b->arrival_s + lo;
        const double* sv = b->service_s + lo;
        const int64_t* id = b->job_id + lo;
        unsigned bad = 0, dec = 0;
        if (n) bad |= (unsigned)pf[0] >= (unsigned)MSG_PROFILE_COUNT || !(ar[0] >= -1.0) || !(sv[0] > 0.0);
        for (uint64_t i = 1; i < n; ++i) {
            bad |= ((unsigned)pf[i] >= (unsigned)MSG_PROFILE_COUNT) | !(ar[i] >= ar[i - 1]) | !(sv[i] > 0.0);
            dec |= id[i] <= id[i - 1];
        }
        if (!bad && !dec) {
            if (n >= kMaxJobsPerTrace) {
                r.status = MSG_ERR_UNSUPPORTED;
                r.message = "Unsupported: at most 2^22 - 1 jobs per trace";
            }
            return r;
        }
    }
    // First failing job in trace order; at one job the checks run in the
    // reference's order: profile, sortedness, service, duplicate id.
    uint64_t bad_idx = n;
    int bad_status = MSG_OK;
    std::string bad_msg;
    double prev = -1.0;
    bool increasing = true;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t k = lo + i;
        const int p = b->profile[k];
        const int64_t id = b->job_id[k];
        if (p < 0 || p >= MSG_PROFILE_COUNT) {
            bad_idx = i, bad_status = MSG_ERR_UNKNOWN_PROFILE;
            bad_msg = "job " + std::to_string(id) + " requests an unknown profile";
            break;
        }
        if (b->arrival_s[k] < prev) {
            bad_idx = i, bad_status = MSG_ERR_TRACE_UNSORTED;
            bad_msg = "job " + std::to_string(id) + " arrives out of order";
            break;
        }
        if (b->service_s[k] <= 0.0) {
            bad_idx = i, bad_status = MSG_ERR_BAD_SPEC;
            bad_msg = "job " + std::to_string(id) + " has non-positive service demand";
            break;
        }
        if (std::isnan(b->arrival_s[k]) || std::isnan(b->service_s[k])) {
            // The reference accepts NaN times and then orders its heap
            // inconsistently; this engine rejects them.
            bad_idx = i, bad_status = MSG_ERR_BAD_SPEC;
            bad_msg = "job " + std::to_string(id) + " has a NaN time";
            break;
        }
        if (i > 0 && id <= b->job_id[k - 1]) increasing = false;
        prev = b->arrival_s[k];
    }
    // Duplicate ids (only possible when ids are not strictly increasing).
    if (!increasing) {
        r.identity = false;
        std::vector<std::pair<int64_t, uint64_t>> v(n);
        for (uint64_t i = 0; i < n; ++i) v[i] = {b->job_id[lo + i], i};
        std::sort(v.begin(), v.end());
        uint64_t dup_idx = n;
        for (uint64_t i = 1; i < n; ++i)
            if (v[i].first == v[i - 1].first) dup_idx = std::min(dup_idx, v[i].second);
        if (dup_idx < bad_idx) {
            bad_idx = dup_idx;
            bad_status = MSG_ERR_BAD_SPEC;
            bad_msg = "duplicate job id " + std::to_string(b->job_id[lo + dup_idx]);
        }
    }
    if (bad_status != MSG_OK) {
        r.status = bad_status;
        r.message = std::string(kStatusNames[bad_status]) + ": " + bad_msg;
        return r;
    }
    if (n >= kMaxJobsPerTrace) {
        r.status = MSG_ERR_UNSUPPORTED;
        r.message = "Unsupported: at most 2^22 - 1 jobs per trace";
    }
    return r;
}

// Copy one validated trace into the rank-order (job-id order) arrays; for
// traces whose ids are not increasing, also the arrival-order permutation
// (arrivals pop in (time, job id) order, TimerLater sim.cpp:49-56).
// copy_ids = false: an identity-order trace's ids are not copied (the caller
// reads them from the batch itself, which outlives its use).
inline void stage_trace_arrays(const msg_trace_batch* b, uint32_t t, const DevTrace& tr, double* ha, double* hs,
                               uint8_t* hp, int64_t* hid, uint32_t* hperm, bool copy_ids = true) {
    const uint64_t lo = b->offsets[t];
    const uint64_t o = tr.job_off;
    const uint32_t n = tr.n_jobs;
    if (!tr.has_perm) {
        std::memcpy(ha + o, b->arrival_s + lo, n * sizeof(double));
        std::memcpy(hs + o, b->service_s + lo, n * sizeof(double));
        if (copy_ids) std::memcpy(hid + o, b->job_id + lo, n * sizeof(int64_t));
        for (uint32_t i = 0; i < n; ++i) hp[o + i] = (uint8_t)b->profile[lo + i];
        return;
    }
    std::vector<uint32_t> by_id(n);
    std::iota(by_id.begin(), by_id.end(), 0u);
    std::sort(by_id.begin(), by_id.end(),
              [&](uint32_t x, uint32_t y) { return b->job_id[lo + x] < b->job_id[lo + y]; });
    std::vector<uint32_t> rank(n);
    for (uint32_t r = 0; r < n; ++r) {
        const uint32_t i = by_id[r];
        rank[i] = r;
        ha[o + r] = b->arrival_s[lo + i];
        hs[o + r] = b->service_s[lo + i];
        hp[o + r] = (uint8_t)b->profile[lo + i];
        hid[o + r] = b->job_id[lo + i];
    }
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
        const double ax = b->arrival_s[lo + x], ay = b->arrival_s[lo + y];
        if (ax != ay) return ax < ay;
        return b->job_id[lo + x] < b->job_id[lo + y];
    });
    for (uint32_t k = 0; k < n; ++k) hperm[o + k] = rank[order[k]];
}

inline void decode_event(const EventRec& r, const int64_t* ids, double overlap, msg_event* out) {
    std::memset(out, 0, sizeof(*out));
    out->time_s = r.t;
    out->kind = r.kind;
    uint32_t pr = 0;
    auto set_job = [&]() {
        out->job = ids[r.job];
        pr |= MSG_HAS_JOB;
    };
    const int size = host_ms(r.profile < 6 ? r.profile : 0);
    switch (r.kind) {
        case 0:  // Arrival (sim.cpp:226-249 / :254-256)
            set_job();
            out->profile = r.profile;
            pr |= MSG_HAS_PROFILE;
            if (r.flags & EF_PLACED) {
                out->gpu = r.gpu;
                out->start = r.start;
                out->size = size;
                out->reused = (r.flags & EF_REUSED) ? 1 : 0;
                std::memcpy(&out->scheduled_s, &r.aux, sizeof(double));
                pr |= MSG_HAS_GPU | MSG_HAS_START | MSG_HAS_SIZE | MSG_HAS_REUSED | MSG_HAS_SCHEDULED;
            }
            break;
        case 1:  // Completion
        case 3:  // MigrationEnd
            set_job();
            out->gpu = r.gpu;
            pr |= MSG_HAS_GPU;
            break;
        case 2: {  // MigrationStart (sim.cpp:366-381)
            set_job();
            out->profile = r.profile;
            out->from_gpu = r.gpu;
            out->from_start = r.start;
            out->to_gpu = r.gpu2;
            out->to_start = r.start2;
            out->move_kind = (r.flags & EF_INTER) ? 1 : 0;
            out->overlap_s = overlap;
            // Frac::to_double (frag.hpp:18) of num/den equals k/25200.0:
            // both are correctly rounded quotients of the same rational.
            out->from_cost_before = (double)(r.aux & 0xFFFF) / 25200.0;
            out->from_cost_after = (double)((r.aux >> 16) & 0xFFFF) / 25200.0;
            out->to_cost_before = (double)((r.aux >> 32) & 0xFFFF) / 25200.0;
            out->to_cost_after = (double)((r.aux >> 48) & 0xFFFF) / 25200.0;
            pr |= MSG_HAS_PROFILE | MSG_HAS_FROM_GPU | MSG_HAS_FROM_START | MSG_HAS_TO_GPU | MSG_HAS_TO_START |
                  MSG_HAS_MOVE_KIND | MSG_HAS_OVERLAP | MSG_HAS_COSTS;
            break;
        }
        case 4:  // Reconfig (sim.cpp:183-195)
            out->gpu = r.gpu;
            out->action = (r.flags & EF_DESTROY) ? 1 : 0;
            out->profile = r.profile;
            out->start = r.start;
            out->size = size;
            pr |= MSG_HAS_GPU | MSG_HAS_ACTION | MSG_HAS_PROFILE | MSG_HAS_START | MSG_HAS_SIZE;
            break;
        case 5:  // Enqueue
            set_job();
            break;
        case 6:  // Dequeue (sim.cpp:332-341)
            set_job();
            out->gpu = r.gpu;
            out->start = r.start;
            out->size = size;
            out->reused = (r.flags & EF_REUSED) ? 1 : 0;
            std::memcpy(&out->scheduled_s, &r.aux, sizeof(double));
            pr |= MSG_HAS_GPU | MSG_HAS_START | MSG_HAS_SIZE | MSG_HAS_REUSED | MSG_HAS_SCHEDULED;
            break;
    }
    out->present = pr;
}

// ---- decision-level snapshots (host_decide.cpp) ---------------------------
inline int placement_index(int p, int s) {  // idle-exact bit (profile-table order)
    static const int base[6] = {0, 1, 2, 4, 7, 11};
    const int stride = (kStridePack >> (4 * p)) & 0xF;
    return base[p] + s / stride;
}

inline uint32_t lazymask_of(double threshold) {
    uint32_t m = 0;
    for (int pc = 0; pc <= 7; ++pc)
        if ((double)pc / 7.0 < threshold) m |= 1u << pc;
    return m;
}

// A snapshot must be representable as the reference's GpuState: valid
// (profile, start) per instance, pairwise slice-disjoint (gpu.cpp:146-156).
inline msg_status check_gpu(const msg_instance* s8, std::string* err) {
    unsigned used = 0;
    for (int s = 0; s < 8; ++s) {
        const msg_instance& x = s8[s];
        if (x.state == MSG_SLOT_EMPTY) continue;
        if (x.state > MSG_SLOT_DRAINING) {
            *err = "InvalidArgument: bad slot state";
            return MSG_ERR_INVALID_ARGUMENT;
        }
        if (x.profile < 0 || x.profile >= MSG_PROFILE_COUNT) {
            *err = "UnknownProfile: snapshot instance with an unknown profile";
            return MSG_ERR_UNKNOWN_PROFILE;
        }
        if (!((host_startmask(x.profile) >> s) & 1u)) {
            *err = "InvalidPlacement: instance at an illegal start";
            return MSG_ERR_INVALID_PLACEMENT;
        }
        if (host_fpm(x.profile, s) & used) {
            *err = "SlicesBusy: overlapping instances in a snapshot";
            return MSG_ERR_SLICES_BUSY;
        }
        used |= host_fpm(x.profile, s);
    }
    return MSG_OK;
}

inline uint32_t to_st(uint8_t state) {
    return state == MSG_SLOT_IDLE ? ST_IDLE : state == MSG_SLOT_BUSY ? ST_RUN : state == MSG_SLOT_DRAINING ? ST_DRAIN
                                                                                                          : ST_EMPTY;
}

struct Staged {
    std::vector<uint32_t> words;
    std::vector<int32_t> jobs;
    std::vector<std::vector<int64_t>> ids;  // per snapshot: rank -> job id
};

// Slot words + per-snapshot job ranks (dense, id order) over the busy jobs and
// any extra ids (queued requests).
inline msg_status stage_snapshots(uint32_t n, int G, const msg_instance* slots, const uint64_t* qoff, const int64_t* qjob,
                           Staged* st, std::string* err) {
    const size_t per = (size_t)G * 8;
    st->words.resize(n * per);
    st->jobs.resize(n * per);
    st->ids.assign(n, {});
    for (uint32_t i = 0; i < n; ++i) {
        const msg_instance* sn = slots + i * per;
        for (int g = 0; g < G; ++g) {
            msg_status e = check_gpu(sn + g * 8, err);
            if (e != MSG_OK) return e;
        }
        std::vector<int64_t>& ids = st->ids[i];
        for (size_t k = 0; k < per; ++k)
            if (sn[k].state == MSG_SLOT_BUSY) ids.push_back(sn[k].job);
        if (qoff)
            for (uint64_t k = qoff[i]; k < qoff[i + 1]; ++k) ids.push_back(qjob[k]);
        std::sort(ids.begin(), ids.end());
        if (std::adjacent_find(ids.begin(), ids.end()) != ids.end()) {
            *err = "InvalidArgument: a job id appears twice in one snapshot";
            return MSG_ERR_INVALID_ARGUMENT;
        }
        if (ids.size() >= (1u << 22)) {
            *err = "Unsupported: too many jobs in one snapshot";
            return MSG_ERR_UNSUPPORTED;
        }
        for (size_t k = 0; k < per; ++k) {
            const msg_instance& x = sn[k];
            st->words[i * per + k] = to_st(x.state) | ((uint32_t)(x.state ? x.profile : 0) << 4) | (x.seq << 8);
            st->jobs[i * per + k] =
                x.state == MSG_SLOT_BUSY
                    ? (int32_t)(std::lower_bound(ids.begin(), ids.end(), x.job) - ids.begin())
                    : -1;
        }
    }
    return MSG_OK;
}

// Write the kernel's slot words back as msg_instance, renumbering `seq`
// densely per GPU in creation order.
inline void unstage_snapshots(uint32_t n, int G, const std::vector<uint32_t>& w, const std::vector<int32_t>& j,
                       const Staged& st, msg_instance* slots) {
    const size_t per = (size_t)G * 8;
    for (uint32_t i = 0; i < n; ++i)
        for (int g = 0; g < G; ++g) {
            const size_t b = i * per + g * 8;
            int order[8], m = 0;
            for (int s = 0; s < 8; ++s)
                if ((w[b + s] & 0xF) != ST_EMPTY) order[m++] = s;
            for (int x = 1; x < m; ++x)  // insertion sort by creation sequence
                for (int y = x; y > 0 && (w[b + order[y]] >> 8) < (w[b + order[y - 1]] >> 8); --y)
                    std::swap(order[y], order[y - 1]);
            for (int s = 0; s < 8; ++s) slots[b + s] = msg_instance{-1, 0, -1, MSG_SLOT_EMPTY, 0};
            for (int r = 0; r < m; ++r) {
                const int s = order[r];
                const uint32_t v = w[b + s];
                const uint32_t stt = v & 0xF;
                msg_instance& o = slots[b + s];
                o.seq = (uint32_t)r;
                o.profile = (int8_t)((v >> 4) & 0xF);
                o.state = stt == ST_IDLE ? MSG_SLOT_IDLE : stt == ST_DRAIN ? MSG_SLOT_DRAINING : MSG_SLOT_BUSY;
                o.job = (o.state == MSG_SLOT_BUSY && j[b + s] >= 0) ? st.ids[i][j[b + s]] : -1;
            }
        }
}

}  // namespace msgk
