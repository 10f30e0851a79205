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
                                                               std::to_string(host_ms(p)) + ") is not valid");
                if (host_fpm(p, st) & used)  // gpu.cpp:103-113
                    return fail(MSG_ERR_SLICES_BUSY,
                                "layout instance overlaps an existing instance on GPU " + std::to_string(g));
                used |= host_fpm(p, st);
                s.init.push_back((uint32_t)(g * 8 + st) | ((uint32_t)p << 16));
            }
        }
    }
    if ((uint32_t)c.gpu_count > kMaxGpusEnsemble)
        return fail(MSG_ERR_UNSUPPORTED, "the ensemble engine supports at most 32 GPUs per cluster");
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
inline void stage_trace_arrays(const msg_trace_batch* b, uint32_t t, const DevTrace& tr, double* ha, double* hs,
                               uint8_t* hp, int64_t* hid, uint32_t* hperm) {
    const uint64_t lo = b->offsets[t];
    const uint64_t o = tr.job_off;
    const uint32_t n = tr.n_jobs;
    if (!tr.has_perm) {
        std::memcpy(ha + o, b->arrival_s + lo, n * sizeof(double));
        std::memcpy(hs + o, b->service_s + lo, n * sizeof(double));
        std::memcpy(hid + o, b->job_id + lo, n * sizeof(int64_t));
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

}  // namespace msgk
