// ORACLE / TEST INFRASTRUCTURE — never linked into the product.
//
// C ABI over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libmigsched_ref.so).  Used only by tests/, by
// __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
// --impl reference leg.  It converts between the reference's C++ types and
// the shared record formats of include/migsched_b200.h so results of the two
// engines can be compared bit for bit.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "migsched/error.hpp"
#include "migsched/frag.hpp"
#include "migsched/gpu.hpp"
#include "migsched/migration.hpp"
#include "migsched/oracle.hpp"
#include "migsched/reports.hpp"
#include "migsched/scheduler.hpp"
#include "migsched/sim.hpp"
#include "migsched/workload.hpp"
#include "migsched_b200.h"

using namespace migsched;

namespace {

int status_of(const std::string& code) {
    static const std::map<std::string, int> m = {
        {"InvalidPlacement", MSG_ERR_INVALID_PLACEMENT}, {"SlicesBusy", MSG_ERR_SLICES_BUSY},
        {"UnknownJob", MSG_ERR_UNKNOWN_JOB},             {"UnknownGpu", MSG_ERR_UNKNOWN_GPU},
        {"NotLazy", MSG_ERR_NOT_LAZY},                   {"UnknownProfile", MSG_ERR_UNKNOWN_PROFILE},
        {"BadThreshold", MSG_ERR_BAD_THRESHOLD},         {"BadConfig", MSG_ERR_BAD_CONFIG},
        {"BadSpec", MSG_ERR_BAD_SPEC},                   {"TraceUnsorted", MSG_ERR_TRACE_UNSORTED},
        {"BadConcurrency", MSG_ERR_BAD_CONCURRENCY},     {"JobsPending", MSG_ERR_JOBS_PENDING},
        {"ParseError", MSG_ERR_PARSE_ERROR}};
    auto it = m.find(code);
    return it == m.end() ? MSG_ERR_INVALID_ARGUMENT : it->second;
}

int profile_index(const std::string& name) {
    auto p = find_profile(name);
    return p ? static_cast<int>(*p) : -1;
}

SimConfig to_sim_config(const msg_config& c) {
    SimConfig cfg;
    cfg.sched.threshold = c.threshold;
    cfg.sched.features.load_balancing = c.load_balancing != 0;
    cfg.sched.features.dynamic_partitioning = c.dynamic_partitioning != 0;
    cfg.sched.features.migration = c.migration != 0;
    if (c.has_static_layout) {
        StaticLayout layout;
        for (int g = 0; g < c.layout_gpus; ++g) {
            std::vector<StaticLayoutEntry> entries;
            for (int i = c.layout_offsets[g]; i < c.layout_offsets[g + 1]; ++i) {
                entries.push_back({static_cast<ProfileId>(c.layout_profile[i]), c.layout_start[i]});
            }
            layout.push_back(std::move(entries));
        }
        cfg.sched.static_layout = std::move(layout);
    }
    cfg.contention_alpha = c.contention_alpha;
    cfg.migration_overlap_s = c.migration_overlap_s;
    cfg.reconfig_latency_s = c.reconfig_latency_s;
    cfg.gpu_count = c.gpu_count;
    cfg.seed = c.seed;
    return cfg;
}

msg_event to_msg_event(const SimEvent& ev) {
    msg_event out;
    std::memset(&out, 0, sizeof(out));
    out.time_s = ev.time_s;
    out.kind = static_cast<int32_t>(ev.kind);
    uint32_t present = 0;
    if (ev.job) { out.job = *ev.job; present |= MSG_HAS_JOB; }
    if (ev.gpu) { out.gpu = *ev.gpu; present |= MSG_HAS_GPU; }
    if (ev.profile) { out.profile = profile_index(*ev.profile); present |= MSG_HAS_PROFILE; }
    if (ev.start) { out.start = *ev.start; present |= MSG_HAS_START; }
    if (ev.size) { out.size = *ev.size; present |= MSG_HAS_SIZE; }
    if (ev.reused) { out.reused = *ev.reused ? 1 : 0; present |= MSG_HAS_REUSED; }
    if (ev.scheduled_s) { out.scheduled_s = *ev.scheduled_s; present |= MSG_HAS_SCHEDULED; }
    if (ev.action) { out.action = *ev.action == "destroy" ? 1 : 0; present |= MSG_HAS_ACTION; }
    if (ev.from_gpu) { out.from_gpu = *ev.from_gpu; present |= MSG_HAS_FROM_GPU; }
    if (ev.from_start) { out.from_start = *ev.from_start; present |= MSG_HAS_FROM_START; }
    if (ev.to_gpu) { out.to_gpu = *ev.to_gpu; present |= MSG_HAS_TO_GPU; }
    if (ev.to_start) { out.to_start = *ev.to_start; present |= MSG_HAS_TO_START; }
    if (ev.move_kind) { out.move_kind = *ev.move_kind == "inter" ? 1 : 0; present |= MSG_HAS_MOVE_KIND; }
    if (ev.overlap_s) { out.overlap_s = *ev.overlap_s; present |= MSG_HAS_OVERLAP; }
    if (ev.from_cost_before) {
        out.from_cost_before = *ev.from_cost_before;
        out.from_cost_after = ev.from_cost_after.value_or(0.0);
        out.to_cost_before = ev.to_cost_before.value_or(0.0);
        out.to_cost_after = ev.to_cost_after.value_or(0.0);
        present |= MSG_HAS_COSTS;
    }
    out.present = present;
    return out;
}

// Handler events (the metric's unit) recovered from the log: every Arrival
// and Completion event is one timer pop; MigrationEnd events are timer pops
// only when overlap > 0 (otherwise logged inline, sim.cpp:384-394);
// ServiceStart pops happen for placements with ops*latency > 0
// (sim.cpp:199-210).
uint64_t count_handler_events(const EventLog& log, const SimConfig& cfg) {
    uint64_t n = 0;
    for (std::size_t i = 0; i < log.size(); ++i) {
        const SimEvent& ev = log[i];
        switch (ev.kind) {
            case EventKind::Arrival:
            case EventKind::Completion: ++n; break;
            case EventKind::MigrationEnd:
                if (cfg.migration_overlap_s > 0.0) ++n;
                break;
            default: break;
        }
        const bool placement = (ev.kind == EventKind::Arrival && ev.gpu) || ev.kind == EventKind::Dequeue;
        if (placement) {
            std::size_t ops = 0;
            for (std::size_t j = i + 1; j < log.size() && log[j].kind == EventKind::Reconfig; ++j) ++ops;
            if (static_cast<double>(ops) * cfg.reconfig_latency_s > 0.0) ++n;
        }
    }
    return n;
}

void fill_summary(const SimResult& r, const SimConfig& cfg, msg_trace_summary* s) {
    std::memset(s, 0, sizeof(*s));
    s->status = MSG_OK;
    s->gpu_count = r.report.gpu_count;
    s->n_jobs = r.report.per_job.size();
    s->handler_events = count_handler_events(r.events, cfg);
    s->n_events = r.events.size();
    s->timeline_samples = r.report.frag_timeline.size();
    s->migration_count = r.report.migration_count;
    s->reconfig_op_count = r.report.reconfig_op_count;
    for (const SimEvent& ev : r.events) {
        if (ev.kind == EventKind::Enqueue) ++s->enqueue_count;
        if (ev.kind == EventKind::Dequeue) ++s->dequeue_count;
    }
    s->max_arrival_frag_evals = r.report.complexity.max_arrival_frag_evals;
    s->max_intra_iter_frag_evals = r.report.complexity.max_intra_iter_frag_evals;
    s->max_inter_iter_frag_evals = r.report.complexity.max_inter_iter_frag_evals;
    s->mean_wait_s = r.report.mean_wait_s;
    s->mean_execution_s = r.report.mean_execution_s;
    s->mean_turnaround_s = r.report.mean_turnaround_s;
    s->workload_makespan_s = r.report.workload_makespan_s;
    double sum = 0.0;
    for (const auto& [t, v] : r.report.frag_timeline) sum += v;
    s->timeline_sum = sum;
}

std::vector<Job> to_trace(const msg_trace_batch* b, uint32_t t) {
    std::vector<Job> jobs;
    const uint64_t lo = b->offsets[t], hi = b->offsets[t + 1];
    jobs.reserve(hi - lo);
    for (uint64_t i = lo; i < hi; ++i) {
        Job j;
        j.id = b->job_id[i];
        j.arrival_s = b->arrival_s[i];
        j.profile = static_cast<ProfileId>(static_cast<std::uint8_t>(b->profile[i]));
        if (b->profile[i] < 0 || b->profile[i] >= kProfileCount) j.profile = static_cast<ProfileId>(200);
        j.service_s = b->service_s[i];
        jobs.push_back(j);
    }
    return jobs;
}

struct RefResult {
    int status = MSG_OK;
    std::string message;
    SimConfig cfg;
    SimResult result;
    std::vector<msg_event> events;
    std::vector<msg_job_row> jobs;
    std::vector<msg_timeline_point> timeline;
    msg_trace_summary summary{};
    std::string jsonl, report_json, report_csv, timeline_csv;
};

void copy_msg(const std::string& m, char* buf, size_t len) {
    if (!buf || len == 0) return;
    std::strncpy(buf, m.c_str(), len - 1);
    buf[len - 1] = 0;
}

}  // namespace

extern "C" {

// ---- whole-trace run (sim.cpp:504-507) ------------------------------------
void* ref_run(const msg_trace_batch* batch, uint32_t trace, const msg_config* c) {
    auto* out = new RefResult();
    out->cfg = to_sim_config(*c);
    try {
        const std::vector<Job> jobs = to_trace(batch, trace);
        out->result = run(jobs, out->cfg);
        for (const SimEvent& ev : out->result.events) out->events.push_back(to_msg_event(ev));
        for (const JobMetrics& m : out->result.report.per_job) {
            msg_job_row r;
            std::memset(&r, 0, sizeof(r));
            r.id = m.id;
            r.arrival_s = m.arrival_s;
            r.scheduled_s = m.scheduled_s;
            r.completed_s = m.completed_s;
            r.wait_s = m.wait_s;
            r.execution_s = m.execution_s;
            r.turnaround_s = m.turnaround_s;
            r.profile = profile_index(m.profile);
            r.gpu = m.gpu;
            r.migrations = m.migrations;
            out->jobs.push_back(r);
        }
        for (const auto& [t, v] : out->result.report.frag_timeline) out->timeline.push_back({t, v});
        fill_summary(out->result, out->cfg, &out->summary);
        out->jsonl = events_to_jsonl(out->result.events);
        out->report_json = report_to_json(out->result.report, out->cfg);
        out->report_csv = report_to_csv(out->result.report);
        out->timeline_csv = frag_timeline_to_csv(out->result.report);
    } catch (const Error& e) {
        out->status = status_of(e.code());
        out->message = e.what();
        out->summary.status = out->status;
    }
    return out;
}

int ref_result_status(void* h) { return static_cast<RefResult*>(h)->status; }
const char* ref_result_message(void* h) { return static_cast<RefResult*>(h)->message.c_str(); }
const msg_trace_summary* ref_result_summary(void* h) { return &static_cast<RefResult*>(h)->summary; }
const msg_event* ref_result_events(void* h, uint64_t* n) {
    auto* r = static_cast<RefResult*>(h);
    *n = r->events.size();
    return r->events.data();
}
const msg_job_row* ref_result_jobs(void* h, uint64_t* n) {
    auto* r = static_cast<RefResult*>(h);
    *n = r->jobs.size();
    return r->jobs.data();
}
const msg_timeline_point* ref_result_timeline(void* h, uint64_t* n) {
    auto* r = static_cast<RefResult*>(h);
    *n = r->timeline.size();
    return r->timeline.data();
}
// Text outputs of the reference's own serializers (reports.cpp:39-116).
const char* ref_result_text(void* h, int which) {
    auto* r = static_cast<RefResult*>(h);
    switch (which) {
        case 0: return r->jsonl.c_str();
        case 1: return r->report_json.c_str();
        case 2: return r->report_csv.c_str();
        default: return r->timeline_csv.c_str();
    }
}
void ref_result_free(void* h) { delete static_cast<RefResult*>(h); }

// ---- batched summaries on a std::thread pool (CPU baseline) -------------
// Returns wall seconds of the batch.
double ref_run_batch(const msg_trace_batch* batch, const msg_config* cfgs, uint32_t n_cfgs,
                     int32_t threads, msg_trace_summary* out) {
    if (threads <= 0) threads = static_cast<int32_t>(std::max(1u, std::thread::hardware_concurrency()));
    std::vector<SimConfig> sims;
    for (uint32_t i = 0; i < n_cfgs; ++i) sims.push_back(to_sim_config(cfgs[i]));
    std::atomic<uint32_t> next{0};
    const auto t0 = std::chrono::steady_clock::now();
    auto worker = [&]() {
        for (;;) {
            const uint32_t t = next.fetch_add(1);
            if (t >= batch->n_traces) return;
            const uint32_t ci = batch->config_index ? batch->config_index[t] : 0;
            try {
                const SimResult r = run(to_trace(batch, t), sims[ci]);
                fill_summary(r, sims[ci], &out[t]);
            } catch (const Error& e) {
                std::memset(&out[t], 0, sizeof(out[t]));
                out[t].status = status_of(e.code());
            }
        }
    };
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int32_t ref_hardware_threads() { return static_cast<int32_t>(std::thread::hardware_concurrency()); }

// ---- workload generation (workload.cpp:98-147) ---------------------------
int ref_generate(const msg_workload_spec* s, int64_t* id, double* arrival, int32_t* profile,
                 double* service) {
    WorkloadSpec spec;
    spec.mean_interarrival_s = s->mean_interarrival_s;
    spec.query_type = s->query_type ? QueryType::Long : QueryType::Normal;
    for (int i = 0; i < 4; ++i) spec.profile_mix[i] = s->profile_mix[i];
    spec.service.family = static_cast<ServiceFamily>(s->service_family);
    spec.service.median_s = s->median_s;
    spec.service.sigma = s->sigma;
    spec.service.mean_s = s->mean_s;
    spec.service.value_s = s->value_s;
    spec.job_count = s->job_count;
    spec.seed = s->seed;
    try {
        const auto jobs = generate(spec);
        for (std::size_t i = 0; i < jobs.size(); ++i) {
            id[i] = jobs[i].id;
            arrival[i] = jobs[i].arrival_s;
            profile[i] = static_cast<int32_t>(jobs[i].profile);
            service[i] = jobs[i].service_s;
        }
    } catch (const Error& e) {
        return status_of(e.code());
    }
    return MSG_OK;
}

// ---- decision-level bridges ------------------------------------------------
namespace {

// Rebuild one GpuState from 8 slots, creating instances in `seq` order so
// the instance vector order matches the snapshot's creation order.
GpuState build_gpu(const msg_instance* slots8, int id) {
    GpuState gpu(id);
    std::vector<int> order;
    for (int s = 0; s < 8; ++s)
        if (slots8[s].state != MSG_SLOT_EMPTY) order.push_back(s);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return slots8[a].seq < slots8[b].seq; });
    for (int s : order) {
        const auto pid = static_cast<ProfileId>(slots8[s].profile);
        const Placement pl{s, profile(pid).size};
        switch (slots8[s].state) {
            case MSG_SLOT_IDLE: gpu.add_idle_instance(pid, pl); break;
            case MSG_SLOT_BUSY: gpu.create_instance(pid, pl, slots8[s].job); break;
            case MSG_SLOT_DRAINING:
                gpu.create_instance(pid, pl, slots8[s].job);
                gpu.start_draining(slots8[s].job);
                break;
        }
    }
    return gpu;
}

void dump_gpu(const GpuState& gpu, msg_instance* slots8) {
    for (int s = 0; s < 8; ++s) {
        slots8[s] = msg_instance{-1, 0, -1, MSG_SLOT_EMPTY, 0};
    }
    uint32_t seq = 0;
    for (const Instance& inst : gpu.instances()) {
        msg_instance& o = slots8[inst.placement.start];
        o.job = inst.job ? *inst.job : -1;
        o.seq = seq++;
        o.profile = static_cast<int8_t>(inst.profile);
        o.state = inst.busy() ? MSG_SLOT_BUSY : (inst.draining ? MSG_SLOT_DRAINING : MSG_SLOT_IDLE);
    }
}

}  // namespace

int ref_schedule(int32_t op, int32_t G, const msg_instance* slots, int32_t prof,
                 const msg_sched_config* c, msg_decision* out) {
    std::vector<GpuState> gpus;
    for (int g = 0; g < G; ++g) gpus.push_back(build_gpu(slots + 8 * g, g));
    SchedulerConfig cfg;
    cfg.threshold = c->threshold;
    cfg.features.load_balancing = c->load_balancing != 0;
    cfg.features.dynamic_partitioning = c->dynamic_partitioning != 0;
    const JobRequest job{999999999, static_cast<ProfileId>(static_cast<std::uint8_t>(prof))};
    std::memset(out, 0, sizeof(*out));
    try {
        ScheduleDecision d;
        if (op == MSG_OP_SCHEDULE) d = schedule(job, gpus, cfg);
        else if (op == MSG_OP_FIRST_FIT) d = first_fit_schedule(job, gpus, cfg);
        else d = dispatch_schedule(job, gpus, cfg);
        out->evaluated_candidates = d.evaluated_candidates;
        if (d.placed) {
            out->placed = 1;
            out->gpu = d.placed->gpu;
            out->start = d.placed->placement.start;
            out->size = d.placed->placement.size;
            out->reused = d.placed->reused ? 1 : 0;
        }
    } catch (const Error& e) {
        return status_of(e.code());
    }
    return MSG_OK;
}

int ref_plan(int32_t op, int32_t G, msg_instance* slots, int32_t gpu, double threshold,
             int32_t enabled, double overlap_s, uint32_t max_moves, msg_move* moves,
             msg_plan_summary* sum) {
    std::vector<GpuState> gpus;
    for (int g = 0; g < G; ++g) gpus.push_back(build_gpu(slots + 8 * g, g));
    std::memset(sum, 0, sizeof(*sum));
    sum->kind = -1;
    try {
        MigrationPlan plan;
        MigrationConfig cfg{threshold, enabled != 0, overlap_s};
        if (op == MSG_PLAN_ON_DEPARTURE) plan = on_departure(gpus, gpu, cfg);
        else if (op == MSG_PLAN_INTRA) plan = plan_intra(gpus, gpu, overlap_s);
        else plan = plan_inter(gpus, gpu, cfg);
        sum->kind = plan.kind ? static_cast<int32_t>(*plan.kind) : -1;
        sum->n_moves = static_cast<int32_t>(plan.moves.size());
        sum->n_iterations = static_cast<int32_t>(plan.frag_evals_per_iteration.size());
        for (int e : plan.frag_evals_per_iteration) sum->max_evals = std::max(sum->max_evals, e);
        for (std::size_t i = 0; i < plan.moves.size() && i < max_moves; ++i) {
            const MigrationMove& m = plan.moves[i];
            msg_move& o = moves[i];
            std::memset(&o, 0, sizeof(o));
            o.job = m.job;
            o.profile = static_cast<int32_t>(m.profile);
            o.from_gpu = m.from_gpu;
            o.from_start = m.from_placement.start;
            o.to_gpu = m.to_gpu;
            o.to_start = m.to_placement.start;
            o.move_kind = m.kind == MoveKind::InterGpu ? 1 : 0;
            o.reused = m.create.reused ? 1 : 0;
            int destroyed = 0;
            for (const ReconfigOp& op2 : m.create.ops) destroyed += op2.action == ReconfigAction::Destroy;
            o.n_destroyed = destroyed;
            o.from_cost_before = m.from_cost_before;
            o.from_cost_after = m.from_cost_after;
            o.to_cost_before = m.to_cost_before;
            o.to_cost_after = m.to_cost_after;
        }
        for (int g = 0; g < G; ++g) dump_gpu(gpus[g], slots + 8 * g);
    } catch (const Error& e) {
        sum->status = status_of(e.code());
        return sum->status;
    }
    return MSG_OK;
}

// try_dequeue (scheduler.cpp:106-121) on one snapshot.
int ref_try_dequeue(int32_t G, msg_instance* slots, uint32_t nq, const int64_t* qjob, const int32_t* qprof,
                    const msg_sched_config* c, msg_dequeue_item* placed, uint32_t* n_placed) {
    std::vector<GpuState> gpus;
    for (int g = 0; g < G; ++g) gpus.push_back(build_gpu(slots + 8 * g, g));
    SchedulerConfig cfg;
    cfg.threshold = c->threshold;
    cfg.features.load_balancing = c->load_balancing != 0;
    cfg.features.dynamic_partitioning = c->dynamic_partitioning != 0;
    std::deque<JobRequest> q;
    for (uint32_t i = 0; i < nq; ++i) q.push_back({qjob[i], static_cast<ProfileId>(static_cast<std::uint8_t>(qprof[i]))});
    try {
        const auto res = try_dequeue(q, gpus, cfg);
        *n_placed = static_cast<uint32_t>(res.size());
        for (std::size_t i = 0; i < res.size(); ++i) {
            msg_dequeue_item& o = placed[i];
            o.job = res[i].job.id;
            o.gpu = res[i].outcome.gpu;
            o.start = res[i].outcome.placement.start;
            o.size = res[i].outcome.placement.size;
            o.reused = res[i].create.reused ? 1 : 0;
            o.evaluated_candidates = res[i].evaluated_candidates;
            int d = 0;
            for (const ReconfigOp& op : res[i].create.ops) d += op.action == ReconfigAction::Destroy;
            o.n_destroyed = d;
        }
        for (int g = 0; g < G; ++g) dump_gpu(gpus[g], slots + 8 * g);
    } catch (const Error& e) {
        return status_of(e.code());
    }
    return MSG_OK;
}

// Frag cost of a state word (busy_c, busy_m, blocked_c, blocked_m) as the
// exact Frac pair (frag.cpp:44-58).
void ref_frag_cost(uint8_t bc, uint8_t bm, uint8_t kc, uint8_t km, int64_t* num, int64_t* den) {
    const Frac f = frag_cost_masks(bc, bm, kc, km);
    *num = f.num;
    *den = f.den;
}

// The reference's own brute-force oracle (oracle.cpp:103-340).
int ref_oracle_run_all(int depth) { return static_cast<int>(oracle::run_all(depth).size()); }

// enumerate_states(depth) flattened: per state, a count then (profile,start) pairs.
int64_t ref_enumerate_states(int depth, int32_t* out, int64_t cap) {
    const auto states = oracle::enumerate_states(depth);
    int64_t n = 0;
    for (const auto& st : states) {
        if (n + 1 + 2 * static_cast<int64_t>(st.busy.size()) > cap) return -1;
        out[n++] = static_cast<int32_t>(st.busy.size());
        for (const auto& u : st.busy) {
            out[n++] = u.profile_index;
            out[n++] = u.start;
        }
    }
    return n;
}

// ---- trace files: migsched::load_trace / save_trace (workload.cpp:151-213)
struct RefTrace {
    std::vector<Job> jobs;
    std::string code, message;
};
void* ref_load_trace(const char* path) {
    auto* t = new RefTrace();
    try {
        t->jobs = load_trace(path);
    } catch (const Error& e) {
        t->code = e.code();
        t->message = e.what();
    } catch (const std::exception& e) {  // e.g. nlohmann type_error escaping load_trace
        t->code = "Exception";
        t->message = e.what();
    }
    return t;
}
const char* ref_trace_code(void* h) { return static_cast<RefTrace*>(h)->code.c_str(); }
const char* ref_trace_message(void* h) { return static_cast<RefTrace*>(h)->message.c_str(); }
int64_t ref_trace_jobs(void* h) { return (int64_t) static_cast<RefTrace*>(h)->jobs.size(); }
void ref_trace_get(void* h, int64_t* id, double* arrival, int32_t* profile, double* service) {
    const auto& j = static_cast<RefTrace*>(h)->jobs;
    for (size_t i = 0; i < j.size(); ++i) {
        id[i] = j[i].id;
        arrival[i] = j[i].arrival_s;
        profile[i] = (int32_t)j[i].profile;
        service[i] = j[i].service_s;
    }
}
void ref_trace_free(void* h) { delete static_cast<RefTrace*>(h); }
int ref_save_trace(const char* path, int64_t n, const int64_t* id, const double* arrival, const int32_t* profile,
                   const double* service) {
    std::vector<Job> jobs((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        jobs[(size_t)i].id = id[i];
        jobs[(size_t)i].arrival_s = arrival[i];
        jobs[(size_t)i].profile = static_cast<ProfileId>(profile[i]);
        jobs[(size_t)i].service_s = service[i];
    }
    try {
        save_trace(jobs, path);
    } catch (const std::exception&) {
        return 1;
    }
    return 0;
}

// ---- the CLI's ablation (tools/migsched.cpp:64-99, reports.cpp:137-168) on
// the reference library, for the CLI parity test: writes ablation.json and
// the table (NUL-terminated, truncated to the buffer sizes); 0 on success.
int ref_ablation(const msg_trace_batch* batch, const msg_config* base, char* json, size_t jlen, char* table,
                 size_t tlen) {
    try {
        const std::vector<Job> trace = to_trace(batch, 0);
        const SimConfig cfg0 = to_sim_config(*base);
        struct Step {
            const char* name;
            FeatureFlags features;
        };
        const Step steps[] = {{"baseline", {false, false, false}},
                              {"lb", {true, false, false}},
                              {"lb+dyn", {true, true, false}},
                              {"lb+dyn+migr", {true, true, true}}};
        std::vector<AblationRow> rows;
        double base_turn = 0.0;
        for (const Step& st : steps) {
            SimConfig cfg = cfg0;
            cfg.sched.features = st.features;
            if (!cfg.sched.features.dynamic_partitioning && !cfg.sched.static_layout)
                cfg.sched.static_layout = static_layout_preset("static-a");
            const SimResult r = run(trace, cfg);
            AblationRow row;
            row.name = st.name;
            row.features = st.features;
            row.mean_turnaround_s = r.report.mean_turnaround_s;
            row.mean_wait_s = r.report.mean_wait_s;
            row.mean_execution_s = r.report.mean_execution_s;
            row.workload_makespan_s = r.report.workload_makespan_s;
            if (rows.empty()) base_turn = row.mean_turnaround_s;
            row.normalized_turnaround = base_turn > 0.0 ? row.mean_turnaround_s / base_turn : 1.0;
            rows.push_back(row);
        }
        std::snprintf(json, jlen, "%s", ablation_to_json(rows).c_str());
        std::snprintf(table, tlen, "%s", ablation_to_table(rows).c_str());
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// ---- brute-force scheduler oracle over clusters of enumerated states
// (oracle.cpp:233-296, check_cluster_against_search): for every cluster of
// G states (indices into enumerate_states(depth)) and every profile, the
// placement the exact-fraction search picks — Lazy GPUs first (threshold
// 0.4), per GPU best_placement_search (lower start on ties), then the
// lowest cost, lower GPU on ties; (-1, -1) when nothing fits.  Threaded.
void ref_oracle_clusters(int depth, int G, const int32_t* idx, int64_t n, int32_t* out_gpu, int32_t* out_start,
                         int threads) {
    const auto states = oracle::enumerate_states(depth);
    std::vector<int> used(states.size(), 0);
    for (size_t i = 0; i < states.size(); ++i)
        for (const auto& u : states[i].busy) used[i] += profiles()[(size_t)u.profile_index].compute_slices;
    // per state and profile: the best single-GPU placement (start, cost)
    std::vector<std::optional<oracle::BestPlacement>> best(states.size() * kProfileCount);
    for (size_t i = 0; i < states.size(); ++i)
        for (int p = 0; p < kProfileCount; ++p)
            best[i * kProfileCount + p] = oracle::best_placement_search(states[i], profiles()[(size_t)p]);
    std::atomic<int64_t> next{0};
    auto work = [&]() {
        for (;;) {
            const int64_t c0 = next.fetch_add(256);
            if (c0 >= n) return;
            for (int64_t c = c0; c < std::min<int64_t>(n, c0 + 256); ++c) {
                for (int p = 0; p < kProfileCount; ++p) {
                    int bg = -1, bs = -1;
                    double bc = 0.0;
                    for (int pass = 0; pass < 2 && bg < 0; ++pass) {
                        for (int g = 0; g < G; ++g) {
                            const int st = idx[c * G + g];
                            const bool lazy = used[(size_t)st] / 7.0 < 0.4;
                            if ((pass == 0) != lazy) continue;
                            const auto& b = best[(size_t)st * kProfileCount + p];
                            if (b && (bg < 0 || b->cost < bc)) {
                                bg = g;
                                bs = b->start;
                                bc = b->cost;
                            }
                        }
                    }
                    out_gpu[c * kProfileCount + p] = bg;
                    out_start[c * kProfileCount + p] = bs;
                }
            }
        }
    };
    std::vector<std::thread> pool;
    const int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
}

}  // extern "C"
