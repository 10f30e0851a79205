// ORACLE / TEST INFRASTRUCTURE — C++ drop-in check.
//
// Calls the reference's migsched::run and the GPU engine's
// migsched_b200::run (include/migsched_b200.hpp) on the same traces, converts
// the GPU's SimEvents into the reference's type and serializes BOTH with the
// reference's own events_to_jsonl / report_to_json / report_to_csv /
// frag_timeline_to_csv (reports.cpp:14-116).  Exit 0 iff every output file is
// byte-identical.  Built by oracle/Makefile (needs the reference headers),
// run on the GPU box by tests/test_gpu_dropin.py.
#include <cstdio>
#include <string>

#include "migsched/reports.hpp"
#include "migsched/sim.hpp"
#include "migsched/workload.hpp"
#include "migsched_b200.hpp"

namespace ref = migsched;
namespace gpu = migsched_b200;

static ref::SimResult to_ref(const gpu::SimResult& g) {
    ref::SimResult r;
    for (const gpu::SimEvent& e : g.events) {
        ref::SimEvent o;
        o.time_s = e.time_s;
        o.kind = static_cast<ref::EventKind>(e.kind);
        o.job = e.job;
        o.gpu = e.gpu;
        o.profile = e.profile;
        o.start = e.start;
        o.size = e.size;
        o.reused = e.reused;
        o.scheduled_s = e.scheduled_s;
        o.action = e.action;
        o.from_gpu = e.from_gpu;
        o.from_start = e.from_start;
        o.to_gpu = e.to_gpu;
        o.to_start = e.to_start;
        o.move_kind = e.move_kind;
        o.overlap_s = e.overlap_s;
        o.from_cost_before = e.from_cost_before;
        o.from_cost_after = e.from_cost_after;
        o.to_cost_before = e.to_cost_before;
        o.to_cost_after = e.to_cost_after;
        r.events.push_back(o);
    }
    const gpu::SimReport& s = g.report;
    for (const gpu::JobMetrics& m : s.per_job)
        r.report.per_job.push_back({m.id, m.profile, m.arrival_s, m.scheduled_s, m.completed_s, m.wait_s,
                                    m.execution_s, m.turnaround_s, m.gpu, m.migrations});
    r.report.mean_wait_s = s.mean_wait_s;
    r.report.mean_execution_s = s.mean_execution_s;
    r.report.mean_turnaround_s = s.mean_turnaround_s;
    r.report.workload_makespan_s = s.workload_makespan_s;
    r.report.migration_count = s.migration_count;
    r.report.reconfig_op_count = s.reconfig_op_count;
    r.report.gpu_count = s.gpu_count;
    r.report.complexity = {s.complexity.max_arrival_frag_evals, s.complexity.max_intra_iter_frag_evals,
                           s.complexity.max_inter_iter_frag_evals};
    r.report.frag_timeline = s.frag_timeline;
    return r;
}

int main() {
    gpu::Engine engine(0);
    int bad = 0, runs = 0;
    const char* presets[] = {"normal25", "long25", "normal50", "long50"};
    for (int pi = 0; pi < 4; ++pi)
        for (int G : {4, 8}) {
            for (std::uint64_t seed = 0; seed < 4; ++seed) {
                auto spec = *ref::preset(presets[pi]);
                spec.seed = seed;
                const auto trace = ref::generate(spec);
                ref::SimConfig rc;
                rc.gpu_count = G;
                rc.migration_overlap_s = seed % 2 ? 0.5 : 0.0;
                rc.reconfig_latency_s = seed == 3 ? 0.1 : 0.0;
                gpu::SimConfig gc;
                gc.gpu_count = G;
                gc.migration_overlap_s = rc.migration_overlap_s;
                gc.reconfig_latency_s = rc.reconfig_latency_s;
                std::vector<gpu::Job> gt;
                for (const auto& j : trace) gt.push_back({j.id, j.arrival_s, static_cast<gpu::ProfileId>(j.profile), j.service_s});
                const ref::SimResult want = ref::run(trace, rc);
                const ref::SimResult got = to_ref(gpu::run(gt, gc));
                ++runs;
                const bool same = ref::events_to_jsonl(want.events) == ref::events_to_jsonl(got.events) &&
                                  ref::report_to_json(want.report, rc) == ref::report_to_json(got.report, rc) &&
                                  ref::report_to_csv(want.report) == ref::report_to_csv(got.report) &&
                                  ref::frag_timeline_to_csv(want.report) == ref::frag_timeline_to_csv(got.report);
                if (!same) {
                    ++bad;
                    std::printf("MISMATCH %s G=%d seed=%llu\n", presets[pi], G, (unsigned long long)seed);
                }
            }
        }
    std::printf("cpp drop-in: %d/%d runs byte-identical (events.jsonl, report.json, report.csv, timeline.csv)\n",
                runs - bad, runs);
    return bad ? 1 : 0;
}
