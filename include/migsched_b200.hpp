// migsched_b200.hpp — header-only C++ façade over include/migsched_b200.h.
//
// Re-exports the reference's own value types and entry points so a C++
// caller of the reference library (the CLI's `run(trace, cfg)`,
// proj/tools/migsched.cpp:85,165; the test suite) switches by changing the
// namespace: migsched::run -> migsched_b200::run.  Types mirror
// proj/include/migsched/sim.hpp:13-114 and scheduler.hpp:12-29 field for
// field; errors are rethrown as migsched_b200::Error carrying the
// reference's code string (error.hpp:10-19).
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "migsched_b200.h"

namespace migsched_b200 {

using JobId = std::int64_t;

enum class ProfileId : std::uint8_t { p7g40gb = 0, p4g20gb = 1, p3g20gb = 2, p2g10gb = 3, p1g10gb = 4, p1g5gb = 5 };

inline const char* profile_name(int p) {
    static const char* names[] = {"7g.40gb", "4g.20gb", "3g.20gb", "2g.10gb", "1g.10gb", "1g.5gb"};
    return (p >= 0 && p < 6) ? names[p] : "";
}

class Error : public std::runtime_error {
public:
    Error(std::string code, const std::string& what) : std::runtime_error(code + ": " + what), code_(std::move(code)) {}
    const std::string& code() const noexcept { return code_; }

    // From a library message, which is already the reference's what() text
    // ("Code: message"): what() of the result equals the reference's.
    static Error from_library(int status, const char* text) {
        std::string code = msg_status_name(status), m = text ? text : "";
        const std::string prefix = code + ": ";
        if (m.rfind(prefix, 0) == 0) m.erase(0, prefix.size());
        return Error(std::move(code), m);
    }

private:
    std::string code_;
};

struct Job {  // sim.hpp:13-18
    JobId id = 0;
    double arrival_s = 0.0;
    ProfileId profile{};
    double service_s = 0.0;
};

struct FeatureFlags {  // scheduler.hpp:12-16
    bool load_balancing = true;
    bool dynamic_partitioning = true;
    bool migration = true;
};

struct StaticLayoutEntry {
    ProfileId profile{};
    int start = 0;
};
using StaticLayout = std::vector<std::vector<StaticLayoutEntry>>;

struct SchedulerConfig {  // scheduler.hpp:25-29
    double threshold = 0.4;
    FeatureFlags features;
    std::optional<StaticLayout> static_layout;
};

struct SimConfig {  // sim.hpp:88-95
    SchedulerConfig sched;
    double contention_alpha = 0.15;
    double migration_overlap_s = 0.0;
    double reconfig_latency_s = 0.0;
    int gpu_count = 4;
    std::uint64_t seed = 0;
};

enum class EventKind { Arrival, Completion, MigrationStart, MigrationEnd, Reconfig, Enqueue, Dequeue };

struct SimEvent {  // sim.hpp:33-52
    double time_s = 0.0;
    EventKind kind{};
    std::optional<JobId> job;
    std::optional<int> gpu;
    std::optional<std::string> profile;
    std::optional<int> start;
    std::optional<int> size;
    std::optional<bool> reused;
    std::optional<double> scheduled_s;
    std::optional<std::string> action;
    std::optional<int> from_gpu;
    std::optional<int> from_start;
    std::optional<int> to_gpu;
    std::optional<int> to_start;
    std::optional<std::string> move_kind;
    std::optional<double> overlap_s;
    std::optional<double> from_cost_before, from_cost_after;
    std::optional<double> to_cost_before, to_cost_after;
};
using EventLog = std::vector<SimEvent>;

struct JobMetrics {  // sim.hpp:56-67
    JobId id = 0;
    std::string profile;
    double arrival_s = 0.0, scheduled_s = 0.0, completed_s = 0.0;
    double wait_s = 0.0, execution_s = 0.0, turnaround_s = 0.0;
    int gpu = -1;
    int migrations = 0;
};

struct ComplexityStats {
    int max_arrival_frag_evals = 0;
    int max_intra_iter_frag_evals = 0;
    int max_inter_iter_frag_evals = 0;
};

struct SimReport {  // sim.hpp:75-86
    std::vector<JobMetrics> per_job;
    double mean_wait_s = 0.0, mean_execution_s = 0.0, mean_turnaround_s = 0.0, workload_makespan_s = 0.0;
    long migration_count = 0;
    long reconfig_op_count = 0;
    int gpu_count = 0;
    ComplexityStats complexity;
    std::vector<std::pair<double, double>> frag_timeline;
};

struct SimResult {
    SimReport report;
    EventLog events;
};

namespace detail {

inline SimEvent to_event(const msg_event& e) {
    SimEvent o;
    o.time_s = e.time_s;
    o.kind = static_cast<EventKind>(e.kind);
    const uint32_t p = e.present;
    if (p & MSG_HAS_JOB) o.job = e.job;
    if (p & MSG_HAS_GPU) o.gpu = e.gpu;
    if (p & MSG_HAS_PROFILE) o.profile = profile_name(e.profile);
    if (p & MSG_HAS_START) o.start = e.start;
    if (p & MSG_HAS_SIZE) o.size = e.size;
    if (p & MSG_HAS_REUSED) o.reused = e.reused != 0;
    if (p & MSG_HAS_SCHEDULED) o.scheduled_s = e.scheduled_s;
    if (p & MSG_HAS_ACTION) o.action = e.action ? "destroy" : "create";
    if (p & MSG_HAS_FROM_GPU) o.from_gpu = e.from_gpu;
    if (p & MSG_HAS_FROM_START) o.from_start = e.from_start;
    if (p & MSG_HAS_TO_GPU) o.to_gpu = e.to_gpu;
    if (p & MSG_HAS_TO_START) o.to_start = e.to_start;
    if (p & MSG_HAS_MOVE_KIND) o.move_kind = e.move_kind ? "inter" : "intra";
    if (p & MSG_HAS_OVERLAP) o.overlap_s = e.overlap_s;
    if (p & MSG_HAS_COSTS) {
        o.from_cost_before = e.from_cost_before;
        o.from_cost_after = e.from_cost_after;
        o.to_cost_before = e.to_cost_before;
        o.to_cost_after = e.to_cost_after;
    }
    return o;
}

struct ConfigHolder {
    msg_config c{};
    std::vector<int32_t> off, prof, start;
    explicit ConfigHolder(const SimConfig& s) {
        c.threshold = s.sched.threshold;
        c.contention_alpha = s.contention_alpha;
        c.migration_overlap_s = s.migration_overlap_s;
        c.reconfig_latency_s = s.reconfig_latency_s;
        c.seed = s.seed;
        c.gpu_count = s.gpu_count;
        c.load_balancing = s.sched.features.load_balancing;
        c.dynamic_partitioning = s.sched.features.dynamic_partitioning;
        c.migration = s.sched.features.migration;
        if (s.sched.static_layout) {
            c.has_static_layout = 1;
            off.push_back(0);
            for (const auto& g : *s.sched.static_layout) {
                for (const auto& e : g) {
                    prof.push_back(static_cast<int32_t>(e.profile));
                    start.push_back(e.start);
                }
                off.push_back(static_cast<int32_t>(prof.size()));
            }
            c.layout_gpus = static_cast<int32_t>(s.sched.static_layout->size());
            c.layout_offsets = off.data();
            c.layout_profile = prof.data();
            c.layout_start = start.data();
        }
    }
};

}  // namespace detail

// One CUDA device; msg_engine underneath.
class Engine {
public:
    explicit Engine(int device = 0) {
        msg_engine* e = nullptr;
        const msg_status st = msg_engine_create(device, &e);
        if (st != MSG_OK) throw Error(msg_status_name(st), "cannot create the CUDA engine");
        eng_.reset(e);
    }

    // migsched::run (sim.hpp:114, sim.cpp:504-507) for many traces at once.
    std::vector<SimResult> run_batch(const std::vector<std::vector<Job>>& traces, const SimConfig& cfg,
                                     bool with_events = true) {
        std::vector<uint64_t> off{0};
        std::vector<int64_t> ids;
        std::vector<double> arr, svc;
        std::vector<int32_t> prof;
        for (const auto& t : traces) {
            for (const Job& j : t) {
                ids.push_back(j.id);
                arr.push_back(j.arrival_s);
                prof.push_back(static_cast<int32_t>(j.profile));
                svc.push_back(j.service_s);
            }
            off.push_back(ids.size());
        }
        msg_trace_batch b{};
        b.n_traces = static_cast<uint32_t>(traces.size());
        b.offsets = off.data();
        b.job_id = ids.data();
        b.arrival_s = arr.data();
        b.profile = prof.data();
        b.service_s = svc.data();
        detail::ConfigHolder ch(cfg);
        msg_batch_result* r = nullptr;
        const uint32_t flags = MSG_OUT_JOBS | (with_events ? MSG_OUT_EVENTS | MSG_OUT_TIMELINE : 0u);
        const msg_status st = msg_run_batch(eng_.get(), &b, &ch.c, 1, flags, &r);
        if (st != MSG_OK) throw Error::from_library(st, msg_engine_last_error(eng_.get()));
        std::unique_ptr<msg_batch_result, void (*)(msg_batch_result*)> hold(r, msg_result_free);
        std::vector<SimResult> out(traces.size());
        for (uint32_t t = 0; t < b.n_traces; ++t) {
            const msg_trace_summary* s = msg_result_summary(r, t);
            if (s->status != MSG_OK) throw Error::from_library(s->status, msg_result_message(r, t));
            SimReport& rep = out[t].report;
            rep.mean_wait_s = s->mean_wait_s;
            rep.mean_execution_s = s->mean_execution_s;
            rep.mean_turnaround_s = s->mean_turnaround_s;
            rep.workload_makespan_s = s->workload_makespan_s;
            rep.migration_count = static_cast<long>(s->migration_count);
            rep.reconfig_op_count = static_cast<long>(s->reconfig_op_count);
            rep.gpu_count = s->gpu_count;
            rep.complexity = {s->max_arrival_frag_evals, s->max_intra_iter_frag_evals, s->max_inter_iter_frag_evals};
            uint64_t n = 0;
            const msg_job_row* jr = msg_result_jobs(r, t, &n);
            for (uint64_t k = 0; k < n; ++k) {
                const msg_job_row& j = jr[k];
                rep.per_job.push_back({j.id, profile_name(j.profile), j.arrival_s, j.scheduled_s, j.completed_s,
                                       j.wait_s, j.execution_s, j.turnaround_s, j.gpu, j.migrations});
            }
            if (with_events) {
                const msg_event* ev = msg_result_events(r, t, &n);
                for (uint64_t k = 0; k < n; ++k) out[t].events.push_back(detail::to_event(ev[k]));
                const msg_timeline_point* tl = msg_result_timeline(r, t, &n);
                for (uint64_t k = 0; k < n; ++k) rep.frag_timeline.emplace_back(tl[k].time_s, tl[k].mean_frag_cost);
            }
        }
        return out;
    }

    SimResult run(const std::vector<Job>& trace, const SimConfig& cfg) { return std::move(run_batch({trace}, cfg)[0]); }

    msg_engine* handle() const { return eng_.get(); }

private:
    std::unique_ptr<msg_engine, void (*)(msg_engine*)> eng_{nullptr, msg_engine_destroy};
};

// Drop-in for migsched::run(trace, cfg): uses a process-wide engine on
// device 0.
inline SimResult run(const std::vector<Job>& trace, const SimConfig& cfg) {
    static Engine engine(0);
    return engine.run(trace, cfg);
}

// Drop-in for migsched::load_trace(path) (workload.hpp:53): the native
// parallel JSONL reader, same validation, codes and messages; jobs
// stable-sorted by arrival.
inline std::vector<Job> load_trace(const std::string& path) {
    msg_trace_file* f = nullptr;
    char msg[512];
    const msg_status st = msg_trace_load(path.c_str(), &f, msg, sizeof msg);
    if (st != MSG_OK) throw Error::from_library(st, msg);
    const uint64_t n = msg_trace_file_jobs(f);
    std::vector<Job> jobs(n);
    const int64_t* id = msg_trace_file_ids(f);
    const double* a = msg_trace_file_arrival(f);
    const int32_t* p = msg_trace_file_profile(f);
    const double* sv = msg_trace_file_service(f);
    for (uint64_t i = 0; i < n; ++i) jobs[i] = Job{id[i], a[i], static_cast<ProfileId>(p[i]), sv[i]};
    msg_trace_file_free(f);
    return jobs;
}

}  // namespace migsched_b200
