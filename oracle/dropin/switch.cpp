// TEST INFRASTRUCTURE (never part of the product): the link-time form of the
// namespace switch INTEGRATION.md describes.  The reference's hot-path
// policy functions are defined here, in namespace migsched with the
// reference's signatures, as calls into the B200 façade
// (include/migsched_b200_policy.hpp).  oracle/Makefile weakens the same
// symbols in copies of the reference's scheduler.o / migration.o / frag.o /
// sim.o, so the reference's OWN unit tests and acceptance suite, compiled
// unchanged, link against these definitions and exercise the GPU engine.
// (The reference's oracle.o also calls schedule(): its differential suites
// compare the GPU's decisions with its brute-force search.)
#include <cstdio>

#include "migsched_b200_policy.hpp"

namespace migsched {

ScheduleDecision schedule(const JobRequest& job, std::span<const GpuState> gpus, const SchedulerConfig& cfg) {
    return migsched_b200::schedule(job, gpus, cfg);
}
ScheduleDecision first_fit_schedule(const JobRequest& job, std::span<const GpuState> gpus,
                                    const SchedulerConfig& cfg) {
    return migsched_b200::first_fit_schedule(job, gpus, cfg);
}
ScheduleDecision dispatch_schedule(const JobRequest& job, std::span<const GpuState> gpus,
                                   const SchedulerConfig& cfg) {
    return migsched_b200::dispatch_schedule(job, gpus, cfg);
}
std::vector<DequeueResult> try_dequeue(std::deque<JobRequest>& queue, std::vector<GpuState>& gpus,
                                       const SchedulerConfig& cfg) {
    return migsched_b200::try_dequeue(queue, gpus, cfg);
}
MigrationMove apply_move(std::vector<GpuState>& gpus, MigrationMove move) {
    return migsched_b200::apply_move(gpus, std::move(move));
}
MigrationPlan plan_intra(std::vector<GpuState>& gpus, int gpu, double overlap_s) {
    return migsched_b200::plan_intra(gpus, gpu, overlap_s);
}
MigrationPlan plan_inter(std::vector<GpuState>& gpus, int lazy_gpu, const MigrationConfig& cfg) {
    return migsched_b200::plan_inter(gpus, lazy_gpu, cfg);
}
MigrationPlan on_departure(std::vector<GpuState>& gpus, int departed_gpu, const MigrationConfig& cfg) {
    return migsched_b200::on_departure(gpus, departed_gpu, cfg);
}
Frac frag_cost_exact(const GpuState& gpu) { return migsched_b200::frag_cost_exact(gpu); }
double frag_cost(const GpuState& gpu) { return migsched_b200::frag_cost(gpu); }
SimResult run(const std::vector<Job>& trace, const SimConfig& cfg) { return migsched_b200::run(trace, cfg); }

}  // namespace migsched

namespace {
// Evidence that the switch took: how many device launches the engine made.
struct LaunchReport {
    ~LaunchReport() {
        msg_engine* e = migsched_b200::policy_detail::box().eng;
        std::printf("[b200-dropin] device launches: %llu\n",
                    static_cast<unsigned long long>(e ? msg_engine_launch_count(e) : 0));
    }
} report_at_exit;
}  // namespace
