// report_io.cpp — report emission: the reference CLI's output files
// (reports.cpp:14-116: events.jsonl, report.json, report.csv,
// fragcost_timeline.csv) byte for byte, formatted in parallel.
//
// At C2/C4 scale the event log runs to millions of lines and host formatting
// dominates end-to-end time: every line here is formatted
// independently on the host pool (chunks concatenated in order).  Doubles in
// JSON use the reference's own JSON library formatting — nlohmann/json
// 3.11.3's detail::to_chars (Grisu2, %g-like layout), non-finite as null —
// and CSV doubles are %.17g, what the reference's ostream at precision 17
// writes.  The JSON layout (member order, optional members per event, the
// dump(2) indentation of report.json) is produced directly, without
// building a JSON document.
#include <nlohmann/json.hpp>

// The byte format of every double written here is nlohmann 3.11.3's
// to_chars, the version the reference was built and its goldens made with.
static_assert(NLOHMANN_JSON_VERSION_MAJOR == 3 && NLOHMANN_JSON_VERSION_MINOR == 11 &&
                  NLOHMANN_JSON_VERSION_PATCH == 3,
              "report_io.cpp needs nlohmann/json 3.11.3 (third_party/nlohmann)");

#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "runtime.h"

using namespace msgk;

namespace {

const char* const kProfileNames[6] = {"7g.40gb", "4g.20gb", "3g.20gb", "2g.10gb", "1g.10gb", "1g.5gb"};
const char* const kKindNames[7] = {"arrival", "completion", "migration_start", "migration_end",
                                   "reconfig",  "enqueue",    "dequeue"};  // event_kind_name (sim.cpp:13-24)

const char* profile_name(int p) { return (p >= 0 && p < 6) ? kProfileNames[p] : ""; }

void put_double(std::string& o, double x) {  // serializer::dump_float
    if (!std::isfinite(x)) {
        o += "null";
        return;
    }
    char buf[64];
    char* end = nlohmann::detail::to_chars(buf, buf + sizeof(buf), x);
    o.append(buf, (size_t)(end - buf));
}
void put_int(std::string& o, long long v) {
    char buf[32];
    const int n = std::snprintf(buf, sizeof buf, "%lld", v);
    o.append(buf, (size_t)n);
}
void put_uint(std::string& o, unsigned long long v) {
    char buf[32];
    const int n = std::snprintf(buf, sizeof buf, "%llu", v);
    o.append(buf, (size_t)n);
}
void put_g17(std::string& o, double x) {
    char buf[64];
    const int n = std::snprintf(buf, sizeof buf, "%.17g", x);
    o.append(buf, (size_t)n);
}

// event_to_json_line (reports.cpp:14-37): members in this order, each only
// when the event carries it.
void event_line(std::string& o, const msg_event& e) {
    const uint32_t p = e.present;
    o += "{\"t\":";
    put_double(o, e.time_s);
    o += ",\"kind\":\"";
    o += (e.kind >= 0 && e.kind < 7) ? kKindNames[e.kind] : "unknown";
    o += '"';
    auto i = [&](uint32_t bit, const char* key, long long v) {
        if (!(p & bit)) return;
        o += ",\"";
        o += key;
        o += "\":";
        put_int(o, v);
    };
    auto d = [&](uint32_t bit, const char* key, double v) {
        if (!(p & bit)) return;
        o += ",\"";
        o += key;
        o += "\":";
        put_double(o, v);
    };
    auto s = [&](uint32_t bit, const char* key, const char* v) {
        if (!(p & bit)) return;
        o += ",\"";
        o += key;
        o += "\":\"";
        o += v;
        o += '"';
    };
    i(MSG_HAS_JOB, "job", e.job);
    i(MSG_HAS_GPU, "gpu", e.gpu);
    s(MSG_HAS_PROFILE, "profile", profile_name(e.profile));
    i(MSG_HAS_START, "start", e.start);
    i(MSG_HAS_SIZE, "size", e.size);
    if (p & MSG_HAS_REUSED) {
        o += ",\"reused\":";
        o += e.reused ? "true" : "false";
    }
    d(MSG_HAS_SCHEDULED, "scheduled_s", e.scheduled_s);
    s(MSG_HAS_ACTION, "action", e.action ? "destroy" : "create");
    i(MSG_HAS_FROM_GPU, "from_gpu", e.from_gpu);
    i(MSG_HAS_FROM_START, "from_start", e.from_start);
    i(MSG_HAS_TO_GPU, "to_gpu", e.to_gpu);
    i(MSG_HAS_TO_START, "to_start", e.to_start);
    s(MSG_HAS_MOVE_KIND, "move_kind", e.move_kind ? "inter" : "intra");
    d(MSG_HAS_OVERLAP, "overlap_s", e.overlap_s);
    d(MSG_HAS_COSTS, "from_cost_before", e.from_cost_before);
    d(MSG_HAS_COSTS, "from_cost_after", e.from_cost_after);
    d(MSG_HAS_COSTS, "to_cost_before", e.to_cost_before);
    d(MSG_HAS_COSTS, "to_cost_after", e.to_cost_after);
    o += "}\n";
}

// One per_job object of report.json at dump(2) indentation (level 2).
void job_object(std::string& o, const msg_job_row& m, bool last) {
    o += "    {\n      \"job_id\": ";
    put_int(o, m.id);
    o += ",\n      \"profile\": \"";
    o += profile_name(m.profile);
    o += "\",\n      \"arrival_s\": ";
    put_double(o, m.arrival_s);
    o += ",\n      \"scheduled_s\": ";
    put_double(o, m.scheduled_s);
    o += ",\n      \"completed_s\": ";
    put_double(o, m.completed_s);
    o += ",\n      \"wait_s\": ";
    put_double(o, m.wait_s);
    o += ",\n      \"execution_s\": ";
    put_double(o, m.execution_s);
    o += ",\n      \"turnaround_s\": ";
    put_double(o, m.turnaround_s);
    o += ",\n      \"gpu\": ";
    put_int(o, m.gpu);
    o += ",\n      \"migrations\": ";
    put_int(o, m.migrations);
    o += last ? "\n    }\n" : "\n    },\n";
}

void job_csv(std::string& o, const msg_job_row& m) {  // report_to_csv (reports.cpp:96-106)
    put_int(o, m.id);
    o += ',';
    o += profile_name(m.profile);
    o += ',';
    put_g17(o, m.arrival_s);
    o += ',';
    put_g17(o, m.scheduled_s);
    o += ',';
    put_g17(o, m.completed_s);
    o += ',';
    put_g17(o, m.wait_s);
    o += ',';
    put_g17(o, m.execution_s);
    o += ',';
    put_g17(o, m.turnaround_s);
    o += ',';
    put_int(o, m.gpu);
    o += ',';
    put_int(o, m.migrations);
    o += '\n';
}

// Formats items [0, n) with `one` in parallel chunks and appends them in order.
template <class F>
void parallel_append(std::string& out, uint64_t n, F&& one) {
    constexpr uint64_t kChunk = 4096;
    const uint64_t chunks = (n + kChunk - 1) / kChunk;
    std::vector<std::string> parts(chunks);
    parallel_for((uint32_t)chunks, 1, [&](uint32_t c) {
        std::string& s = parts[c];
        s.reserve(kChunk * 160);
        const uint64_t e = std::min<uint64_t>(n, (c + 1) * kChunk);
        for (uint64_t k = c * kChunk; k < e; ++k) one(s, k);
    });
    size_t total = out.size();
    for (auto& s : parts) total += s.size();
    out.reserve(total);
    for (auto& s : parts) out += s;
}

// report_to_json (reports.cpp:51-91) at dump(2).
void report_json(std::string& o, const msg_trace_summary& sm, const msg_config& cfg, const msg_job_row* jobs,
                 uint64_t n) {
    auto b = [](bool v) { return v ? "true" : "false"; };
    o += "{\n  \"schema\": 1,\n  \"config\": {\n    \"threshold\": ";
    put_double(o, cfg.threshold);
    o += ",\n    \"features\": {\n      \"load_balancing\": ";
    o += b(cfg.load_balancing);
    o += ",\n      \"dynamic_partitioning\": ";
    o += b(cfg.dynamic_partitioning);
    o += ",\n      \"migration\": ";
    o += b(cfg.migration);
    o += "\n    },\n    \"contention_alpha\": ";
    put_double(o, cfg.contention_alpha);
    o += ",\n    \"migration_overlap_s\": ";
    put_double(o, cfg.migration_overlap_s);
    o += ",\n    \"reconfig_latency_s\": ";
    put_double(o, cfg.reconfig_latency_s);
    o += ",\n    \"gpus\": ";
    put_int(o, cfg.gpu_count);
    o += ",\n    \"seed\": ";
    put_uint(o, cfg.seed);
    o += "\n  },\n  \"summary\": {\n    \"jobs\": ";
    put_uint(o, n);
    o += ",\n    \"mean_wait_s\": ";
    put_double(o, sm.mean_wait_s);
    o += ",\n    \"mean_execution_s\": ";
    put_double(o, sm.mean_execution_s);
    o += ",\n    \"mean_turnaround_s\": ";
    put_double(o, sm.mean_turnaround_s);
    o += ",\n    \"workload_makespan_s\": ";
    put_double(o, sm.workload_makespan_s);
    o += ",\n    \"migration_count\": ";
    put_int(o, sm.migration_count);
    o += ",\n    \"reconfig_op_count\": ";
    put_int(o, sm.reconfig_op_count);
    o += "\n  },\n  \"complexity\": {\n    \"max_arrival_frag_evals\": ";
    put_int(o, sm.max_arrival_frag_evals);
    o += ",\n    \"max_intra_iter_frag_evals\": ";
    put_int(o, sm.max_intra_iter_frag_evals);
    o += ",\n    \"max_inter_iter_frag_evals\": ";
    put_int(o, sm.max_inter_iter_frag_evals);
    if (n == 0) {
        o += "\n  },\n  \"per_job\": []\n}\n";
        return;
    }
    o += "\n  },\n  \"per_job\": [\n";
    parallel_append(o, n, [&](std::string& s, uint64_t k) { job_object(s, jobs[k], k + 1 == n); });
    o += "  ]\n}\n";
}

}  // namespace

extern "C" {

msg_status msg_format_text(int32_t kind, const msg_trace_summary* summary, const msg_config* cfg,
                           const msg_event* events, uint64_t n_events, const msg_job_row* jobs, uint64_t n_jobs,
                           const msg_timeline_point* timeline, uint64_t n_timeline, char** text, size_t* len) {
    if (!text || !len) return MSG_ERR_INVALID_ARGUMENT;
    *text = nullptr;
    *len = 0;
    std::string o;
    switch (kind) {
        case MSG_TEXT_EVENTS_JSONL:
            if (n_events && !events) return MSG_ERR_INVALID_ARGUMENT;
            o = "{\"schema\":1,\"kind\":\"migsched-events\"}\n";  // events_to_jsonl (reports.cpp:39-44)
            parallel_append(o, n_events, [&](std::string& s, uint64_t k) { event_line(s, events[k]); });
            break;
        case MSG_TEXT_REPORT_JSON:
            if (!summary || !cfg || (n_jobs && !jobs)) return MSG_ERR_INVALID_ARGUMENT;
            report_json(o, *summary, *cfg, jobs, n_jobs);
            break;
        case MSG_TEXT_REPORT_CSV:
            if (n_jobs && !jobs) return MSG_ERR_INVALID_ARGUMENT;
            o = "job_id,profile,arrival_s,scheduled_s,completed_s,wait_s,execution_s,turnaround_s,gpu,migrations\n";
            parallel_append(o, n_jobs, [&](std::string& s, uint64_t k) { job_csv(s, jobs[k]); });
            break;
        case MSG_TEXT_TIMELINE_CSV:  // frag_timeline_to_csv (reports.cpp:108-116)
            if (n_timeline && !timeline) return MSG_ERR_INVALID_ARGUMENT;
            o = "time_s,mean_frag_cost\n";
            parallel_append(o, n_timeline, [&](std::string& s, uint64_t k) {
                put_g17(s, timeline[k].time_s);
                s += ',';
                put_g17(s, timeline[k].mean_frag_cost);
                s += '\n';
            });
            break;
        default:
            return MSG_ERR_INVALID_ARGUMENT;
    }
    char* buf = static_cast<char*>(std::malloc(o.size() + 1));
    if (!buf) return MSG_ERR_INVALID_ARGUMENT;
    std::memcpy(buf, o.data(), o.size());
    buf[o.size()] = '\0';
    *text = buf;
    *len = o.size();
    return MSG_OK;
}

void msg_text_free(char* text) { std::free(text); }

}  // extern "C"
