// migsched_b200 — command-line front end of the B200 engine (SURVEY §8f
// row 3): the reference CLI's `simulate` and `ablate` (proj/tools/
// migsched.cpp:64-99,156-177) on the GPU, with the same output files and
// stdout, plus `sweep`, the C3 ablation grid (technique combinations x seeds
// x arrival loads) as one batch — one kernel launch.
//
//   migsched_b200 simulate [trace] [config] [--out DIR]
//   migsched_b200 ablate   [trace] [config] [--out DIR]
//   migsched_b200 sweep    --preset NAME --seeds N [--loads 10,15,25,35,50] [config] [--out DIR]
//   trace:  --trace FILE.jsonl | --preset NAME [--seed S] [--jobs N]
//   config: --gpus G --threshold T --alpha A --overlap S --latency S
//           --features lb,dyn,mig|none --static-layout static-a|b|c
//
// Options replace the reference's JSON config file (config.cpp, not part of
// this engine); defaults are SimConfig's (sim.hpp:88-95).  Errors print
// "error: <Code>: <message>" and exit 1, like the reference.
#include <nlohmann/json.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "migsched_b200.h"

namespace fs = std::filesystem;

namespace {

struct CliError {
    std::string code, message;
};

[[noreturn]] void fail(const std::string& code, const std::string& m) { throw CliError{code, m}; }

void check(msg_status st, msg_engine* eng = nullptr, const char* what = "") {
    if (st == MSG_OK) return;
    fail(msg_status_name(st), eng ? msg_engine_last_error(eng) : what);
}

// ---- options --------------------------------------------------------------
struct Options {
    std::string cmd, trace, preset = "normal25", out = "out", features, layout;
    uint64_t seed = 0;
    int jobs = 0, gpus = 4, seeds = 16;
    double threshold = 0.4, alpha = 0.15, overlap = 0.0, latency = 0.0;
    bool lb = true, dyn = true, mig = true;
    std::vector<double> loads{10, 15, 25, 35, 50};
};

Options parse(int argc, char** argv) {
    if (argc < 2) fail("BadConfig", "usage: migsched_b200 simulate|ablate|sweep [options]");
    Options o;
    o.cmd = argv[1];
    if (o.cmd != "simulate" && o.cmd != "ablate" && o.cmd != "sweep") fail("BadConfig", "unknown command " + o.cmd);
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) fail("BadConfig", "missing value for " + k);
            return argv[++i];
        };
        if (k == "--trace") o.trace = val();
        else if (k == "--preset") o.preset = val();
        else if (k == "--out") o.out = val();
        else if (k == "--seed") o.seed = std::stoull(val());
        else if (k == "--jobs") o.jobs = std::stoi(val());
        else if (k == "--gpus") o.gpus = std::stoi(val());
        else if (k == "--seeds") o.seeds = std::stoi(val());
        else if (k == "--threshold") o.threshold = std::stod(val());
        else if (k == "--alpha") o.alpha = std::stod(val());
        else if (k == "--overlap") o.overlap = std::stod(val());
        else if (k == "--latency") o.latency = std::stod(val());
        else if (k == "--static-layout") o.layout = val();
        else if (k == "--features") {
            const std::string f = val();
            o.lb = f.find("lb") != std::string::npos;
            o.dyn = f.find("dyn") != std::string::npos;
            o.mig = f.find("mig") != std::string::npos;
        } else if (k == "--loads") {
            o.loads.clear();
            std::stringstream ss(val());
            std::string x;
            while (std::getline(ss, x, ',')) o.loads.push_back(std::stod(x));
        } else {
            fail("BadConfig", "unknown option " + k);
        }
    }
    return o;
}

// static_layout_preset (scheduler.cpp:123-155), as (profile, start) per GPU
std::vector<std::vector<std::pair<int, int>>> layout_preset(const std::string& name) {
    if (name == "static-a") return {{{1, 0}, {2, 4}}, {{1, 0}, {2, 4}}, {{3, 0}, {3, 2}, {3, 4}, {5, 6}},
                                    {{5, 0}, {5, 1}, {5, 2}, {5, 3}, {3, 4}, {5, 6}}};
    if (name == "static-b") return {{{1, 0}, {3, 4}, {5, 6}}, {{1, 0}, {3, 4}, {5, 6}}, {{2, 0}, {2, 4}},
                                    {{2, 0}, {3, 4}, {5, 6}}};
    if (name == "static-c") return {{{1, 0}, {2, 4}}, {{2, 0}, {2, 4}}, {{3, 0}, {3, 2}, {3, 4}, {5, 6}},
                                    {{3, 0}, {3, 2}, {5, 4}, {5, 5}, {5, 6}}};
    fail("BadConfig", "unknown static layout \"" + name + "\"");
}

struct Config {  // msg_config + the storage its layout pointers refer to
    msg_config c{};
    std::vector<int32_t> off{0}, prof, start;
    Config(const Options& o, bool lb, bool dyn, bool mig, const std::string& layout) {
        c.threshold = o.threshold;
        c.contention_alpha = o.alpha;
        c.migration_overlap_s = o.overlap;
        c.reconfig_latency_s = o.latency;
        c.seed = o.seed;
        c.gpu_count = o.gpus;
        c.load_balancing = lb;
        c.dynamic_partitioning = dyn;
        c.migration = mig;
        if (!layout.empty()) {
            for (const auto& g : layout_preset(layout)) {
                for (const auto& [p, s] : g) {
                    prof.push_back(p);
                    start.push_back(s);
                }
                off.push_back((int32_t)prof.size());
            }
            c.has_static_layout = 1;
            c.layout_gpus = (int32_t)off.size() - 1;
            c.layout_offsets = off.data();
            c.layout_profile = prof.data();
            c.layout_start = start.data();
        }
    }
};

// ---- traces -----------------------------------------------------------------
struct Traces {  // msg_trace_batch storage
    std::vector<uint64_t> off{0};
    std::vector<int64_t> id;
    std::vector<double> arr, svc;
    std::vector<int32_t> prof;
    std::vector<uint32_t> cfg;
    void add(const int64_t* i, const double* a, const int32_t* p, const double* s, uint64_t n, uint32_t ci) {
        id.insert(id.end(), i, i + n);
        arr.insert(arr.end(), a, a + n);
        prof.insert(prof.end(), p, p + n);
        svc.insert(svc.end(), s, s + n);
        off.push_back(id.size());
        cfg.push_back(ci);
    }
    msg_trace_batch batch() const {
        msg_trace_batch b{};
        b.n_traces = (uint32_t)cfg.size();
        b.offsets = off.data();
        b.job_id = id.data();
        b.arrival_s = arr.data();
        b.profile = prof.data();
        b.service_s = svc.data();
        b.config_index = cfg.data();
        return b;
    }
};

void add_generated(Traces& t, msg_workload_spec spec, uint32_t ci) {
    const size_t n = (size_t)std::max(spec.job_count, 0);
    std::vector<int64_t> id(n + 1);
    std::vector<double> a(n + 1), s(n + 1);
    std::vector<int32_t> p(n + 1);
    check(msg_generate(&spec, id.data(), a.data(), p.data(), s.data()), nullptr, "generate");
    t.add(id.data(), a.data(), p.data(), s.data(), n, ci);
}

msg_workload_spec preset_spec(const Options& o) {  // resolve_trace (migsched.cpp:33-47)
    msg_workload_spec spec{};
    if (msg_workload_preset(o.preset.c_str(), &spec) != MSG_OK)
        fail("BadConfig", "unknown preset \"" + o.preset + "\" (expected one of normal25, long25, normal50, long50)");
    spec.seed = o.seed;
    if (o.jobs > 0) spec.job_count = o.jobs;
    return spec;
}

void add_trace(Traces& t, const Options& o, uint32_t ci) {
    if (o.trace.empty()) return add_generated(t, preset_spec(o), ci);
    msg_trace_file* f = nullptr;
    char msg[512];
    const msg_status st = msg_trace_load(o.trace.c_str(), &f, msg, sizeof msg);
    if (st != MSG_OK) {
        const std::string m(msg), code = msg_status_name(st);
        fail(code, m.size() > code.size() + 2 ? m.substr(code.size() + 2) : m);
    }
    t.add(msg_trace_file_ids(f), msg_trace_file_arrival(f), msg_trace_file_profile(f), msg_trace_file_service(f),
          msg_trace_file_jobs(f), ci);
    msg_trace_file_free(f);
}

// ---- outputs ------------------------------------------------------------------
void write_file(const std::string& path, const char* data, size_t n) {
    std::ofstream out(path, std::ios::binary);
    if (!out) fail("BadConfig", "cannot write file " + path);
    out.write(data, (std::streamsize)n);
}

std::string num(double x) {  // the reference's JSON number formatting
    if (!std::isfinite(x)) return "null";
    char buf[64];
    char* e = nlohmann::detail::to_chars(buf, buf + sizeof buf, x);
    return std::string(buf, (size_t)(e - buf));
}

const msg_trace_summary& ok_summary(const msg_batch_result* r, uint32_t t) {
    const msg_trace_summary* s = msg_result_summary(r, t);
    if (s->status != MSG_OK) {
        const std::string m = msg_result_message(r, t), code = msg_status_name(s->status);
        fail(code, m.rfind(code + ": ", 0) == 0 ? m.substr(code.size() + 2) : m);
    }
    return *s;
}

int simulate(msg_engine* eng, const Options& o) {
    Config cfg(o, o.lb, o.dyn, o.mig, o.layout);
    Traces t;
    add_trace(t, o, 0);
    const msg_trace_batch b = t.batch();
    msg_batch_result* r = nullptr;
    check(msg_run_batch(eng, &b, &cfg.c, 1, MSG_OUT_JOBS | MSG_OUT_EVENTS | MSG_OUT_TIMELINE, &r), eng);
    const msg_trace_summary& s = ok_summary(r, 0);
    uint64_t ne = 0, nj = 0, nt = 0;
    const msg_event* ev = msg_result_events(r, 0, &ne);
    const msg_job_row* jb = msg_result_jobs(r, 0, &nj);
    const msg_timeline_point* tl = msg_result_timeline(r, 0, &nt);
    fs::create_directories(o.out);
    const struct {
        int kind;
        const char* file;
    } files[] = {{MSG_TEXT_REPORT_JSON, "report.json"},
                 {MSG_TEXT_REPORT_CSV, "report.csv"},
                 {MSG_TEXT_EVENTS_JSONL, "events.jsonl"},
                 {MSG_TEXT_TIMELINE_CSV, "fragcost_timeline.csv"}};
    for (const auto& f : files) {
        char* text = nullptr;
        size_t len = 0;
        check(msg_format_text(f.kind, &s, &cfg.c, ev, ne, jb, nj, tl, nt, &text, &len), nullptr, "format");
        write_file(o.out + "/" + f.file, text, len);
        msg_text_free(text);
    }
    std::printf(  // print_summary (migsched.cpp:57-62)
        "jobs=%zu mean_wait=%.3fs mean_execution=%.3fs mean_turnaround=%.3fs makespan=%.3fs migrations=%ld "
        "reconfig_ops=%ld\n",
        (size_t)nj, s.mean_wait_s, s.mean_execution_s, s.mean_turnaround_s, s.workload_makespan_s,
        (long)s.migration_count, (long)s.reconfig_op_count);
    msg_result_free(r);
    return 0;
}

struct Step {
    const char* name;
    bool lb, dyn, mig;
};
const Step kSteps[4] = {{"baseline", false, false, false},
                        {"lb", true, false, false},
                        {"lb+dyn", true, true, false},
                        {"lb+dyn+migr", true, true, true}};

// run_ablation (migsched.cpp:64-99): the four combinations on one trace,
// one batch; static-a stands in for a missing layout when dyn is off.
int ablate(msg_engine* eng, const Options& o) {
    std::vector<Config> cfgs;
    cfgs.reserve(4);
    for (const Step& st : kSteps)
        cfgs.emplace_back(o, st.lb, st.dyn, st.mig, (!st.dyn && o.layout.empty()) ? "static-a" : o.layout);
    Traces one, t;
    add_trace(one, o, 0);
    for (uint32_t k = 0; k < 4; ++k) t.add(one.id.data(), one.arr.data(), one.prof.data(), one.svc.data(), one.off[1], k);
    std::vector<msg_config> cs;
    for (auto& c : cfgs) cs.push_back(c.c);
    const msg_trace_batch b = t.batch();
    msg_batch_result* r = nullptr;
    check(msg_run_batch(eng, &b, cs.data(), 4, 0, &r), eng);
    std::string js = "{\n  \"schema\": 1,\n  \"rows\": [\n", table = "configuration        mean_turnaround_s   normalized\n";
    double base = 0.0;
    for (uint32_t k = 0; k < 4; ++k) {  // ablation_to_json / ablation_to_table (reports.cpp:137-168)
        const msg_trace_summary& s = ok_summary(r, k);
        if (k == 0) base = s.mean_turnaround_s;
        const double norm = base > 0.0 ? s.mean_turnaround_s / base : 1.0;
        auto b2 = [](bool v) { return v ? "true" : "false"; };
        js += std::string("    {\n      \"name\": \"") + kSteps[k].name + "\",\n      \"features\": {\n" +
              "        \"load_balancing\": " + b2(kSteps[k].lb) + ",\n        \"dynamic_partitioning\": " +
              b2(kSteps[k].dyn) + ",\n        \"migration\": " + b2(kSteps[k].mig) + "\n      },\n" +
              "      \"mean_turnaround_s\": " + num(s.mean_turnaround_s) + ",\n      \"normalized_turnaround\": " +
              num(norm) + ",\n      \"mean_wait_s\": " + num(s.mean_wait_s) + ",\n      \"mean_execution_s\": " +
              num(s.mean_execution_s) + ",\n      \"workload_makespan_s\": " + num(s.workload_makespan_s) +
              (k == 3 ? "\n    }\n" : "\n    },\n");
        table += kSteps[k].name;
        for (size_t i = std::strlen(kSteps[k].name); i < 21; ++i) table += ' ';
        char buf[64];
        std::snprintf(buf, sizeof buf, "%-20.3f%.4f\n", s.mean_turnaround_s, norm);
        table += buf;
    }
    js += "  ]\n}\n";
    fs::create_directories(o.out);
    write_file(o.out + "/ablation.json", js.data(), js.size());
    std::printf("%s", table.c_str());
    msg_result_free(r);
    return 0;
}

// C3: combinations x seeds x loads in one batch; per (combination, load)
// the seed-mean of the per-trace means (sums in seed order).
int sweep(msg_engine* eng, const Options& o) {
    std::vector<Config> cfgs;
    cfgs.reserve(4);
    for (const Step& st : kSteps)
        cfgs.emplace_back(o, st.lb, st.dyn, st.mig, (!st.dyn && o.layout.empty()) ? "static-a" : o.layout);
    std::vector<msg_config> cs;
    for (auto& c : cfgs) cs.push_back(c.c);
    Traces t;
    for (double load : o.loads)
        for (uint32_t k = 0; k < 4; ++k)
            for (int sd = 0; sd < o.seeds; ++sd) {
                msg_workload_spec spec = preset_spec(o);
                spec.mean_interarrival_s = load;
                spec.seed = o.seed + (uint64_t)sd;
                add_generated(t, spec, k);
            }
    const msg_trace_batch b = t.batch();
    msg_batch_result* r = nullptr;
    check(msg_run_batch(eng, &b, cs.data(), 4, 0, &r), eng);
    std::string js = "{\n  \"schema\": 1,\n  \"preset\": \"" + o.preset + "\",\n  \"gpus\": " + std::to_string(o.gpus) +
                     ",\n  \"seeds\": " + std::to_string(o.seeds) + ",\n  \"rows\": [\n";
    uint32_t tr = 0;
    uint64_t events = 0;
    for (size_t li = 0; li < o.loads.size(); ++li)
        for (uint32_t k = 0; k < 4; ++k) {
            double turn = 0.0, wait = 0.0, make = 0.0;
            for (int sd = 0; sd < o.seeds; ++sd, ++tr) {
                const msg_trace_summary& s = ok_summary(r, tr);
                turn += s.mean_turnaround_s;
                wait += s.mean_wait_s;
                make += s.workload_makespan_s;
                events += s.handler_events;
            }
            const double n = (double)o.seeds;
            js += std::string("    {\n      \"name\": \"") + kSteps[k].name + "\",\n      \"mean_interarrival_s\": " +
                  num(o.loads[li]) + ",\n      \"mean_turnaround_s\": " + num(turn / n) + ",\n      \"mean_wait_s\": " +
                  num(wait / n) + ",\n      \"workload_makespan_s\": " + num(make / n) +
                  ((li + 1 == o.loads.size() && k == 3) ? "\n    }\n" : "\n    },\n");
        }
    js += "  ]\n}\n";
    fs::create_directories(o.out);
    write_file(o.out + "/sweep.json", js.data(), js.size());
    std::printf("sweep: %u traces, %llu decisions\n", b.n_traces, (unsigned long long)events);
    msg_result_free(r);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    msg_engine* eng = nullptr;
    try {
        const Options o = parse(argc, argv);
        check(msg_engine_create(0, &eng), nullptr, "no usable CUDA device");
        const int rc = o.cmd == "simulate" ? simulate(eng, o) : o.cmd == "ablate" ? ablate(eng, o) : sweep(eng, o);
        msg_engine_destroy(eng);
        return rc;
    } catch (const CliError& e) {
        std::fprintf(stderr, "error: %s: %s\n", e.code.c_str(), e.message.c_str());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
    }
    if (eng) msg_engine_destroy(eng);
    return 1;
}
