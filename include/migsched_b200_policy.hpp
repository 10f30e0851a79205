// migsched_b200_policy.hpp — the reference's C++ policy interface over its
// own value types, decided on the B200.
//
// For a C++ caller of the reference library that keeps its types
// (migsched::GpuState, JobRequest, SchedulerConfig, MigrationConfig, Job,
// SimConfig — include/migsched/*.hpp), this header offers every hot-path
// function of that interface with the same signature in namespace
// migsched_b200, so a call site switches by changing the namespace
// (migsched::schedule -> migsched_b200::schedule):
//
//   schedule / first_fit_schedule / dispatch_schedule  scheduler.hpp:59-70
//   try_dequeue                                        scheduler.hpp:81-83
//   apply_move / plan_intra / plan_inter / on_departure migration.hpp:55-63
//   frag_cost / frag_cost_exact                        frag.hpp:50-51
//   run                                                sim.hpp:114
//
// Every decision (placement search, planners, costs, the whole event loop
// of run) is computed by the sm_100a kernels behind the C ABI
// (include/migsched_b200.h).  The caller owns its std::vector<GpuState>;
// where the reference mutates it (try_dequeue, the planners, apply_move)
// the decided placements and moves are applied to the caller's objects
// through GpuState's own methods (create_instance, start_draining,
// finish_draining), in the reference's order, so instance ids, reuse flags
// and reconfiguration ops come out exactly as the reference's.  Errors are
// thrown as migsched::Error with the reference's code and what() text.
//
// Include the reference's headers (the caller's tree) before or through
// this one; link libmigsched_b200.so.  One process-wide engine on device
// MSG_DEVICE (default 0) serves the calls; calls are serialised on it.
//
// Known deviation: MigrationPlan::frag_evals_per_iteration holds a single
// entry, the maximum over the plan's iterations — the only quantity the
// reference consumes (sim.cpp:347-349, ComplexityStats).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <deque>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "migsched/error.hpp"
#include "migsched/frag.hpp"
#include "migsched/migration.hpp"
#include "migsched/scheduler.hpp"
#include "migsched/sim.hpp"
#include "migsched_b200.h"

namespace migsched_b200 {

namespace policy_detail {

struct EngineBox {
    msg_engine* eng = nullptr;
    std::mutex mu;
    ~EngineBox() {
        if (eng) msg_engine_destroy(eng);
    }
};

inline EngineBox& box() {
    static EngineBox b;
    return b;
}

// The process-wide engine (created on first use; no CPU fallback: a missing
// device throws CudaError).
inline msg_engine* engine() {
    EngineBox& b = box();
    if (!b.eng) {
        const char* d = std::getenv("MSG_DEVICE");
        msg_engine* e = nullptr;
        const msg_status st = msg_engine_create(d ? std::atoi(d) : 0, &e);
        if (st != MSG_OK) throw migsched::Error(msg_status_name(st), "cannot create the CUDA engine");
        b.eng = e;
    }
    return b.eng;
}

// migsched::Error from a library status: the engine's message is the
// reference's what() text ("Code: message"); the code is stripped once.
[[noreturn]] inline void raise(msg_engine* eng, msg_status st) {
    std::string code = msg_status_name(st), m = eng ? msg_engine_last_error(eng) : "";
    const std::string prefix = code + ": ";
    if (m.rfind(prefix, 0) == 0) m.erase(0, prefix.size());
    throw migsched::Error(code, m);
}

// One GPU as 8 instance slots keyed by start index, seq = position in the
// instance vector (= creation order, gpu.cpp:88-111).
inline void to_slots(const migsched::GpuState& g, msg_instance* s8) {
    for (int k = 0; k < 8; ++k) s8[k] = msg_instance{-1, 0, -1, MSG_SLOT_EMPTY, 0};
    uint32_t seq = 0;
    for (const migsched::Instance& inst : g.instances()) {
        const int st = inst.placement.start;
        if (st < 0 || st > 7) throw migsched::Error("InvalidPlacement", "instance start outside 0..7");
        msg_instance& x = s8[st];
        x.job = inst.job ? *inst.job : -1;
        x.seq = seq++;
        x.profile = static_cast<int8_t>(inst.profile);
        x.state = inst.job ? MSG_SLOT_BUSY : inst.draining ? MSG_SLOT_DRAINING : MSG_SLOT_IDLE;
    }
}

// A cluster snapshot whose busy jobs carry surrogate ids gpu * 8 + (rank of
// the job id among the GPU's busy jobs).  The reference's decisions compare
// job ids only between jobs of one GPU (plan_intra: (cost, job, start)) or
// after the GPU index (plan_inter: (cost, gpu, job)); schedule and
// try_dequeue never compare them.  So the surrogates give the same
// decisions while the reference's callers may reuse ids across GPUs (its
// oracle suites do, oracle.cpp:117-125).  `orig` maps surrogate -> id.
inline std::vector<msg_instance> to_slots(std::span<const migsched::GpuState> gpus, std::vector<int64_t>* orig) {
    std::vector<msg_instance> s(gpus.size() * 8 + 8);
    if (orig) orig->assign(gpus.size() * 8, -1);
    for (size_t g = 0; g < gpus.size(); ++g) {
        msg_instance* s8 = s.data() + 8 * g;
        to_slots(gpus[g], s8);
        int64_t ids[8];
        int n = 0;
        for (int k = 0; k < 8; ++k)
            if (s8[k].state == MSG_SLOT_BUSY) ids[n++] = s8[k].job;
        std::sort(ids, ids + n);
        for (int k = 0; k < 8; ++k) {
            if (s8[k].state != MSG_SLOT_BUSY) continue;
            const int64_t r = std::lower_bound(ids, ids + n, s8[k].job) - ids;
            const int64_t sur = static_cast<int64_t>(g) * 8 + r;
            if (orig) (*orig)[static_cast<size_t>(sur)] = s8[k].job;
            s8[k].job = sur;
        }
    }
    return s;
}

// The busy instances only: their 4-mask cost is the 2-mask "end state"
// cost apply_move records (migration.cpp:52-54).
inline void to_busy_slots(const migsched::GpuState& g, msg_instance* s8) {
    to_slots(g, s8);
    for (int k = 0; k < 8; ++k)
        if (s8[k].state != MSG_SLOT_BUSY) s8[k] = msg_instance{-1, 0, -1, MSG_SLOT_EMPTY, 0};
}

inline msg_sched_config sched_config(const migsched::SchedulerConfig& c) {
    msg_sched_config m{};
    m.threshold = c.threshold;
    m.load_balancing = c.features.load_balancing ? 1 : 0;
    m.dynamic_partitioning = c.features.dynamic_partitioning ? 1 : 0;
    return m;
}

inline migsched::ScheduleDecision decide(int32_t op, const migsched::JobRequest& job,
                                         std::span<const migsched::GpuState> gpus,
                                         const migsched::SchedulerConfig& cfg) {
    const int p = static_cast<int>(job.profile);
    if (p < 0 || p >= MSG_PROFILE_COUNT)  // scheduler.cpp:11-15
        throw migsched::Error("UnknownProfile", "job " + std::to_string(job.id) + " requests an unknown profile");
    std::lock_guard<std::mutex> lk(box().mu);
    msg_engine* eng = engine();
    const std::vector<msg_instance> slots = to_slots(gpus, nullptr);
    const int32_t prof = p;
    const msg_sched_config c = sched_config(cfg);
    msg_decision d{};
    const msg_status st =
        msg_schedule_batch(eng, op, 1, static_cast<int32_t>(gpus.size()), slots.data(), &prof, &c, &d);
    if (st != MSG_OK) raise(eng, st);
    migsched::ScheduleDecision out;
    out.evaluated_candidates = d.evaluated_candidates;
    if (d.placed) out.placed = migsched::PlacedOutcome{d.gpu, migsched::Placement{d.start, d.size}, d.reused != 0};
    return out;
}

inline migsched::GpuState& gpu_at(std::vector<migsched::GpuState>& gpus, int id, const char* ctx) {
    if (id < 0 || static_cast<size_t>(id) >= gpus.size())  // migration.cpp:12-17
        throw migsched::Error("UnknownGpu", std::string(ctx) + ": no GPU with id " + std::to_string(id));
    return gpus[static_cast<size_t>(id)];
}

// frag_cost of n GPU snapshots on the device (numerators over 25200 and
// doubles).
inline void frag_costs(const std::vector<msg_instance>& slots, uint32_t n, int32_t* num, double* cost) {
    msg_engine* eng = engine();
    const msg_status st = msg_frag_cost_batch(eng, n, slots.data(), num, cost);
    if (st != MSG_OK) raise(eng, st);
}

// Applies a move the device decided to the caller's GpuStates in
// apply_move's order (migration.cpp:58-64): source replica drains, the
// destination instance is created (reusing an exact idle one or destroying
// overlapping idle ones), the source is freed at once when overlap <= 0.
inline migsched::MigrationMove replay_move(std::vector<migsched::GpuState>& gpus, migsched::MigrationMove mv) {
    migsched::GpuState& from = gpus[static_cast<size_t>(mv.from_gpu)];
    migsched::GpuState& to = gpus[static_cast<size_t>(mv.to_gpu)];
    mv.source_instance = from.start_draining(mv.job);
    mv.create = to.create_instance(mv.profile, mv.to_placement, mv.job);
    if (mv.overlap_s <= 0.0) from.finish_draining(mv.source_instance);
    return mv;
}

inline migsched::MigrationPlan plan(int32_t op, std::vector<migsched::GpuState>& gpus, int gpu_id, double threshold,
                                    bool enabled, double overlap_s, const char* ctx) {
    gpu_at(gpus, gpu_id, ctx);
    if (!enabled) return {};
    std::lock_guard<std::mutex> lk(box().mu);
    msg_engine* eng = engine();
    std::vector<int64_t> orig;
    const std::vector<msg_instance> before = to_slots(std::span<const migsched::GpuState>(gpus), &orig);
    const int32_t G = static_cast<int32_t>(gpus.size());
    const int32_t g = gpu_id;
    uint32_t cap = 64;
    std::vector<msg_move> moves;
    msg_plan_summary s{};
    for (;;) {
        std::vector<msg_instance> slots = before;
        moves.assign(cap, msg_move{});
        const msg_status st =
            msg_plan_batch(eng, op, 1, G, slots.data(), &g, threshold, enabled ? 1 : 0, overlap_s, cap, moves.data(), &s);
        if (st != MSG_OK) raise(eng, st);
        if (s.status == MSG_ERR_NOT_LAZY)  // migration.cpp:127-129
            throw migsched::Error("NotLazy", "GPU " + std::to_string(gpu_id) + " is not below the threshold");
        if (s.status == MSG_ERR_UNKNOWN_GPU)
            throw migsched::Error("UnknownGpu", std::string(ctx) + ": no GPU with id " + std::to_string(gpu_id));
        if (s.status != MSG_OK) {
            throw migsched::Error(msg_status_name(s.status), std::string(ctx) + ": rejected by the engine");
        }
        if (static_cast<uint32_t>(s.n_moves) <= cap) break;
        cap = static_cast<uint32_t>(s.n_moves);
    }
    migsched::MigrationPlan out;
    if (s.kind >= 0) out.kind = s.kind == 0 ? migsched::MoveKind::IntraGpu : migsched::MoveKind::InterGpu;
    out.frag_evals_per_iteration.push_back(s.max_evals);
    for (int32_t k = 0; k < s.n_moves; ++k) {
        const msg_move& m = moves[static_cast<size_t>(k)];
        migsched::MigrationMove mv;
        mv.job = orig[static_cast<size_t>(m.job)];
        mv.profile = static_cast<migsched::ProfileId>(m.profile);
        const int size = migsched::profile(mv.profile).size;
        mv.from_gpu = m.from_gpu;
        mv.from_placement = migsched::Placement{m.from_start, size};
        mv.to_gpu = m.to_gpu;
        mv.to_placement = migsched::Placement{m.to_start, size};
        mv.kind = m.move_kind ? migsched::MoveKind::InterGpu : migsched::MoveKind::IntraGpu;
        mv.overlap_s = overlap_s;
        mv = replay_move(gpus, mv);
        mv.from_cost_before = m.from_cost_before;
        mv.from_cost_after = m.from_cost_after;
        mv.to_cost_before = m.to_cost_before;
        mv.to_cost_after = m.to_cost_after;
        out.moves.push_back(std::move(mv));
    }
    return out;
}

inline migsched::SimEvent to_event(const msg_event& e) {
    static const char* names[] = {"7g.40gb", "4g.20gb", "3g.20gb", "2g.10gb", "1g.10gb", "1g.5gb"};
    migsched::SimEvent o;
    o.time_s = e.time_s;
    o.kind = static_cast<migsched::EventKind>(e.kind);
    const uint32_t p = e.present;
    if (p & MSG_HAS_JOB) o.job = e.job;
    if (p & MSG_HAS_GPU) o.gpu = e.gpu;
    if (p & MSG_HAS_PROFILE) o.profile = names[e.profile];
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

}  // namespace policy_detail

// ---- scheduler.hpp:59-83 ----------------------------------------------------
inline migsched::ScheduleDecision schedule(const migsched::JobRequest& job, std::span<const migsched::GpuState> gpus,
                                           const migsched::SchedulerConfig& cfg) {
    return policy_detail::decide(MSG_OP_SCHEDULE, job, gpus, cfg);
}

inline migsched::ScheduleDecision first_fit_schedule(const migsched::JobRequest& job,
                                                     std::span<const migsched::GpuState> gpus,
                                                     const migsched::SchedulerConfig& cfg) {
    return policy_detail::decide(MSG_OP_FIRST_FIT, job, gpus, cfg);
}

inline migsched::ScheduleDecision dispatch_schedule(const migsched::JobRequest& job,
                                                    std::span<const migsched::GpuState> gpus,
                                                    const migsched::SchedulerConfig& cfg) {
    return policy_detail::decide(MSG_OP_DISPATCH, job, gpus, cfg);
}

// Strict FCFS (scheduler.cpp:106-121): the device places heads until the
// first that would queue; each placement is applied to the caller's GPU
// with create_instance, and the placed heads leave the queue.
inline std::vector<migsched::DequeueResult> try_dequeue(std::deque<migsched::JobRequest>& queue,
                                                        std::vector<migsched::GpuState>& gpus,
                                                        const migsched::SchedulerConfig& cfg) {
    std::vector<migsched::DequeueResult> placed;
    if (queue.empty()) return placed;
    std::vector<msg_dequeue_item> items(queue.size());
    uint32_t n_placed = 0;
    {
        std::lock_guard<std::mutex> lk(policy_detail::box().mu);
        msg_engine* eng = policy_detail::engine();
        std::vector<msg_instance> slots =
            policy_detail::to_slots(std::span<const migsched::GpuState>(gpus), nullptr);
        const uint64_t qoff[2] = {0, queue.size()};
        std::vector<int64_t> qjob;  // surrogate ids past the busy ones (placement never compares ids)
        std::vector<int32_t> qprof;
        for (const auto& j : queue) {
            qjob.push_back(static_cast<int64_t>(gpus.size() * 8 + qjob.size()));
            qprof.push_back(static_cast<int32_t>(j.profile));
        }
        const msg_sched_config c = policy_detail::sched_config(cfg);
        const msg_status st = msg_try_dequeue_batch(eng, 1, static_cast<int32_t>(gpus.size()), slots.data(), qoff,
                                                    qjob.data(), qprof.data(), &c, items.data(), &n_placed);
        if (st != MSG_OK) policy_detail::raise(eng, st);
    }
    for (uint32_t k = 0; k < n_placed; ++k) {
        const msg_dequeue_item& it = items[k];
        const migsched::JobRequest head = queue.front();
        queue.pop_front();
        const migsched::PlacedOutcome outcome{it.gpu, migsched::Placement{it.start, it.size}, it.reused != 0};
        migsched::CreateResult create =
            gpus[static_cast<size_t>(it.gpu)].create_instance(head.profile, outcome.placement, head.id);
        placed.push_back({head, outcome, std::move(create), it.evaluated_candidates});
    }
    return placed;
}

// ---- migration.hpp:55-63 ----------------------------------------------------
// apply_move (migration.cpp:35-69): the reference's validation order, the
// four end-state costs from the device cost tables.
inline migsched::MigrationMove apply_move(std::vector<migsched::GpuState>& gpus, migsched::MigrationMove move) {
    migsched::GpuState& from = policy_detail::gpu_at(gpus, move.from_gpu, "apply_move");
    migsched::GpuState& to = policy_detail::gpu_at(gpus, move.to_gpu, "apply_move");
    const migsched::Instance* source = from.find_job(move.job);
    if (source == nullptr)
        throw migsched::Error("UnknownJob", "job " + std::to_string(move.job) + " is not running on GPU " +
                                                std::to_string(move.from_gpu));
    if (source->profile != move.profile)
        throw migsched::Error("InvalidPlacement", "migration profile does not match the job's instance");
    if (!migsched::avail(to, move.profile, move.to_placement))
        throw migsched::Error("SlicesBusy", "migration destination is occupied on GPU " + std::to_string(move.to_gpu));
    std::lock_guard<std::mutex> lk(policy_detail::box().mu);
    std::vector<msg_instance> s(16);
    double c[2];
    policy_detail::to_busy_slots(from, s.data());
    policy_detail::to_busy_slots(to, s.data() + 8);
    policy_detail::frag_costs(s, 2, nullptr, c);
    move.from_cost_before = c[0];
    move.to_cost_before = c[1];
    move = policy_detail::replay_move(gpus, move);
    policy_detail::to_busy_slots(from, s.data());
    policy_detail::to_busy_slots(to, s.data() + 8);
    policy_detail::frag_costs(s, 2, nullptr, c);
    move.from_cost_after = c[0];
    move.to_cost_after = c[1];
    return move;
}

inline migsched::MigrationPlan plan_intra(std::vector<migsched::GpuState>& gpus, int gpu, double overlap_s) {
    return policy_detail::plan(MSG_PLAN_INTRA, gpus, gpu, 0.4, true, overlap_s, "plan_intra");
}

inline migsched::MigrationPlan plan_inter(std::vector<migsched::GpuState>& gpus, int lazy_gpu,
                                          const migsched::MigrationConfig& cfg) {
    return policy_detail::plan(MSG_PLAN_INTER, gpus, lazy_gpu, cfg.threshold, true, cfg.overlap_s, "plan_inter");
}

inline migsched::MigrationPlan on_departure(std::vector<migsched::GpuState>& gpus, int departed_gpu,
                                            const migsched::MigrationConfig& cfg) {
    return policy_detail::plan(MSG_PLAN_ON_DEPARTURE, gpus, departed_gpu, cfg.threshold, cfg.enabled, cfg.overlap_s,
                               "on_departure");
}

// ---- frag.hpp:50-51 ---------------------------------------------------------
// The device's exact cost tables: every reachable cost is k/25200.
inline migsched::Frac frag_cost_exact(const migsched::GpuState& gpu) {
    std::lock_guard<std::mutex> lk(policy_detail::box().mu);
    std::vector<msg_instance> s(8);
    policy_detail::to_slots(gpu, s.data());
    int32_t k = 0;
    policy_detail::frag_costs(s, 1, &k, nullptr);
    return migsched::Frac{k, 25200};
}

inline double frag_cost(const migsched::GpuState& gpu) {
    std::lock_guard<std::mutex> lk(policy_detail::box().mu);
    std::vector<msg_instance> s(8);
    policy_detail::to_slots(gpu, s.data());
    double c = 0.0;
    policy_detail::frag_costs(s, 1, nullptr, &c);
    return c;
}

// ---- sim.hpp:114 ------------------------------------------------------------
// migsched::run for many traces in one launch (one warp per trace).
inline std::vector<migsched::SimResult> run_batch(const std::vector<std::vector<migsched::Job>>& traces,
                                                  const migsched::SimConfig& cfg) {
    std::vector<uint64_t> off{0};
    std::vector<int64_t> ids;
    std::vector<double> arr, svc;
    std::vector<int32_t> prof;
    for (const auto& t : traces) {
        for (const migsched::Job& j : t) {
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
    msg_config c{};
    c.threshold = cfg.sched.threshold;
    c.contention_alpha = cfg.contention_alpha;
    c.migration_overlap_s = cfg.migration_overlap_s;
    c.reconfig_latency_s = cfg.reconfig_latency_s;
    c.seed = cfg.seed;
    c.gpu_count = cfg.gpu_count;
    c.load_balancing = cfg.sched.features.load_balancing;
    c.dynamic_partitioning = cfg.sched.features.dynamic_partitioning;
    c.migration = cfg.sched.features.migration;
    std::vector<int32_t> loff, lprof, lstart;
    if (cfg.sched.static_layout) {
        c.has_static_layout = 1;
        loff.push_back(0);
        for (const auto& g : *cfg.sched.static_layout) {
            for (const auto& e : g) {
                lprof.push_back(static_cast<int32_t>(e.profile));
                lstart.push_back(e.start);
            }
            loff.push_back(static_cast<int32_t>(lprof.size()));
        }
        c.layout_gpus = static_cast<int32_t>(cfg.sched.static_layout->size());
        c.layout_offsets = loff.data();
        c.layout_profile = lprof.data();
        c.layout_start = lstart.data();
    }
    std::lock_guard<std::mutex> lk(policy_detail::box().mu);
    msg_engine* eng = policy_detail::engine();
    msg_batch_result* r = nullptr;
    const msg_status st = msg_run_batch(eng, &b, &c, 1, MSG_OUT_JOBS | MSG_OUT_EVENTS | MSG_OUT_TIMELINE, &r);
    if (st != MSG_OK) policy_detail::raise(eng, st);
    std::unique_ptr<msg_batch_result, void (*)(msg_batch_result*)> hold(r, msg_result_free);
    static const char* names[] = {"7g.40gb", "4g.20gb", "3g.20gb", "2g.10gb", "1g.10gb", "1g.5gb"};
    std::vector<migsched::SimResult> out(traces.size());
    for (uint32_t t = 0; t < b.n_traces; ++t) {
        const msg_trace_summary* s = msg_result_summary(r, t);
        if (s->status != MSG_OK) {
            std::string code = msg_status_name(s->status), m = msg_result_message(r, t);
            if (m.rfind(code + ": ", 0) == 0) m.erase(0, code.size() + 2);
            throw migsched::Error(code, m);
        }
        migsched::SimReport& rep = out[t].report;
        rep.mean_wait_s = s->mean_wait_s;
        rep.mean_execution_s = s->mean_execution_s;
        rep.mean_turnaround_s = s->mean_turnaround_s;
        rep.workload_makespan_s = s->workload_makespan_s;
        rep.migration_count = static_cast<long>(s->migration_count);
        rep.reconfig_op_count = static_cast<long>(s->reconfig_op_count);
        rep.gpu_count = s->gpu_count;
        rep.complexity.max_arrival_frag_evals = s->max_arrival_frag_evals;
        rep.complexity.max_intra_iter_frag_evals = s->max_intra_iter_frag_evals;
        rep.complexity.max_inter_iter_frag_evals = s->max_inter_iter_frag_evals;
        uint64_t n = 0;
        const msg_job_row* rows = msg_result_jobs(r, t, &n);
        rep.per_job.reserve(n);
        for (uint64_t k = 0; k < n; ++k) {
            const msg_job_row& x = rows[k];
            migsched::JobMetrics m;
            m.id = x.id;
            m.profile = names[x.profile];
            m.arrival_s = x.arrival_s;
            m.scheduled_s = x.scheduled_s;
            m.completed_s = x.completed_s;
            m.wait_s = x.wait_s;
            m.execution_s = x.execution_s;
            m.turnaround_s = x.turnaround_s;
            m.gpu = x.gpu;
            m.migrations = x.migrations;
            rep.per_job.push_back(std::move(m));
        }
        const msg_timeline_point* tl = msg_result_timeline(r, t, &n);
        rep.frag_timeline.reserve(n);
        for (uint64_t k = 0; k < n; ++k) rep.frag_timeline.emplace_back(tl[k].time_s, tl[k].mean_frag_cost);
        const msg_event* ev = msg_result_events(r, t, &n);
        out[t].events.reserve(n);
        for (uint64_t k = 0; k < n; ++k) out[t].events.push_back(policy_detail::to_event(ev[k]));
    }
    return out;
}

inline migsched::SimResult run(const std::vector<migsched::Job>& trace, const migsched::SimConfig& cfg) {
    return std::move(run_batch({trace}, cfg)[0]);
}

}  // namespace migsched_b200
