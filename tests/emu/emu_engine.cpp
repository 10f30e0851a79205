// TEST INFRASTRUCTURE ONLY — runs the unchanged device code
// (paper_2512_16099_b200/csrc/engine_core.cuh) on 32 host threads per trace,
// with the product's own staging/decoding (staging.h), and returns results
// in the ABI record formats so tests can diff them against the reference.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "cluster_core.cuh"
#include "engine_core.cuh"
#include "staging.h"

using namespace msgk;

namespace {

struct EmuResult {
    int status = 0;
    std::string message;
    msg_trace_summary summary{};
    std::vector<msg_event> events;
    std::vector<msg_job_row> jobs;
    std::vector<msg_timeline_point> timeline;
};

template <int SPL, bool ND = false>
void run_warp_t(const SimArgs& a, const DevTables* tb) {
    auto ws = std::make_unique<WarpSmem<SPL>>();
    std::memset(ws.get(), 0xA5, sizeof(WarpSmem<SPL>));  // garbage, like real smem
    wp::EmuWarp warp;
    std::vector<std::thread> lanes;
    for (unsigned l = 0; l < 32; ++l) {
        lanes.emplace_back([&, l]() {
            wp::g_warp = &warp;
            wp::g_lane = l;
            wp::g_phase = 0;
            simulate_trace<SPL, true, false, ND>(a, tb, ws.get(), 0);
        });
    }
    for (auto& t : lanes) t.join();
}
// MSG_EMU_ND=1: the no-delay instantiation, as the library picks it (reconfig
// latency +0 and no migration overlap)
template <int SPL>
void run_warp(const SimArgs& a, const DevTables* tb) {
    if (a.no_delay) run_warp_t<SPL, true>(a, tb);
    else run_warp_t<SPL, false>(a, tb);
}

// The pipelined msg_run_batch's IO instantiation (zero-copy inputs,
// progressive SoA rows in "host" memory, completion flag).
template <int SPL>
void run_warp_io(const SimArgs& a, const DevTables* tb) {
    auto ws = std::make_unique<WarpSmem<SPL>>();
    std::memset(ws.get(), 0xA5, sizeof(WarpSmem<SPL>));
    wp::EmuWarp warp;
    std::vector<std::thread> lanes;
    for (unsigned l = 0; l < 32; ++l) {
        lanes.emplace_back([&, l]() {
            wp::g_warp = &warp;
            wp::g_lane = l;
            wp::g_phase = 0;
            simulate_trace<SPL, false, true>(a, tb, ws.get(), 0);
        });
    }
    for (auto& t : lanes) t.join();
}

// Block engine (G > 32) on D device groups (MSG_EMU_GROUPS) of S emulated
// blocks each (one cluster per group) of `nt` threads (nt/32 warps + a block
// barrier; a cluster barrier across a group's blocks).  Each group gets its
// own SimArgs like a separate GPU would: its own FCFS queue copy, the shared
// job rows / summary / timeline of group 0, and the host-memory inboxes of
// every group.
void run_block(const SimArgs& a0, const DevTables* tb, unsigned nt, unsigned S, unsigned D, bool gpu_smem,
               bool slots, int G) {
    const unsigned NB = S * D;
    std::vector<std::unique_ptr<BlockScratch>> sc;
    std::vector<std::unique_ptr<wp::EmuBlock>> blocks;
    std::vector<std::vector<unsigned char>> smem;
    std::vector<std::unique_ptr<wp::EmuCluster>> clusters;
    std::vector<std::unique_ptr<wp::EmuWarp>> warps;
    std::vector<XInbox> inbox(D);
    std::memset(inbox.data(), 0, sizeof(XInbox) * D);
    std::vector<std::vector<int32_t>> queues(D, std::vector<int32_t>(std::max<uint32_t>(a0.traces[0].n_jobs, 1)));
    std::vector<SimArgs> args(D, a0);
    for (unsigned d = 0; d < D; ++d) {
        args[d].n_dev = D;
        args[d].dev0 = d;
        args[d].vdev = 1;
        args[d].queue = d ? queues[d].data() : a0.queue;
        for (unsigned k = 0; k < D; ++k) args[d].inbox[k] = &inbox[k];
        clusters.emplace_back(new wp::EmuCluster());
        clusters.back()->S = S;
        clusters.back()->n = S * nt;
    }
    for (unsigned b = 0; b < NB; ++b) {
        sc.emplace_back(new BlockScratch());
        std::memset(sc.back().get(), 0xA5, sizeof(BlockScratch));
        clusters[b / S]->base[b % S] = reinterpret_cast<char*>(sc.back().get());
        blocks.emplace_back(new wp::EmuBlock());
        blocks.back()->n = nt;
        smem.emplace_back(105 * (size_t)((G + NB - 1) / NB) + 16, 0xA5);  // stands in for dynamic smem
        for (unsigned i = 0; i < nt / 32; ++i) warps.emplace_back(new wp::EmuWarp());
    }
    std::vector<std::thread> th;
    for (unsigned b = 0; b < NB; ++b)
        for (unsigned t = 0; t < nt; ++t)
            th.emplace_back([&, b, t]() {
                wp::g_block = blocks[b].get();
                wp::g_warp = warps[b * (nt / 32) + t / 32].get();
                wp::g_lane = t % 32;
                wp::g_tid = t;
                wp::g_phase = 0;
                wp::g_cluster = S > 1 ? clusters[b / S].get() : nullptr;
                wp::g_crank = b % S;
                simulate_large_trace<true>(args[b / S], tb, sc[b].get(), gpu_smem ? smem[b].data() : nullptr,
                                           gpu_smem && slots, 0);
            });
    for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

void* emu_run(const msg_trace_batch* b, uint32_t t, const msg_config* c) {
    auto* r = new EmuResult();
    CfgState cs = validate_config(*c);
    r->summary.gpu_count = c->gpu_count;
    if (cs.status != MSG_OK) {
        r->status = r->summary.status = cs.status;
        r->message = cs.message;
        return r;
    }
    TraceCheck tc = check_trace(b, t);
    if (tc.status != MSG_OK) {
        r->status = r->summary.status = tc.status;
        r->message = tc.message;
        return r;
    }
    DevTrace tr{};
    tr.n_jobs = (uint32_t)(b->offsets[t + 1] - b->offsets[t]);
    tr.has_perm = tc.identity ? 0 : 1;
    tr.ev_cap = 64 * tr.n_jobs + 256;
    tr.tl_cap = 32 * tr.n_jobs + 64;
    const size_t N = std::max<uint32_t>(tr.n_jobs, 1);
    std::vector<double> ha(N), hs(N);
    std::vector<uint8_t> hp(N);
    std::vector<int64_t> hid(N);
    std::vector<uint32_t> hperm(N);
    stage_trace_arrays(b, t, tr, ha.data(), hs.data(), hp.data(), hid.data(), hperm.data());
    cs.dev.init_off = 0;
    DevTables tables;
    build_tables(&tables);
    static std::vector<uint16_t> stab = [&] {
        std::vector<uint16_t> v(kScoreTab);
        build_score_table(tables, v.data());
        return v;
    }();
    std::vector<int32_t> queue(N);
    std::vector<JobOut> jobs(N);
    std::vector<EventRec> evs(tr.ev_cap);
    std::vector<double> tl(2 * (size_t)tr.tl_cap);
    DevSummary sum{};
    SimArgs a{};
    a.traces = &tr;
    a.configs = &cs.dev;
    a.init_slots = cs.init.empty() ? nullptr : cs.init.data();
    a.tables = &tables;
    a.score_tab = stab.data();
    a.arrival = ha.data();
    a.service = hs.data();
    a.profile = hp.data();
    a.perm = hperm.data();
    a.queue = queue.data();
    a.jobs = jobs.data();
    a.events = evs.data();
    a.timeline = tl.data();
    a.summary = &sum;
    a.n_traces = 1;
    a.out_flags = OF_JOBS | OF_EVENTS | OF_TIMELINE;
    a.no_delay = std::getenv("MSG_EMU_ND") && cs.dev.latency == 0.0 && !std::signbit(cs.dev.latency) &&
                 cs.dev.overlap <= 0.0;
    const int G = c->gpu_count;
    // block-engine arena (used when G > 32, or when MSG_EMU_FORCE_BLOCK is set)
    const size_t ns = 8 * (size_t)G;
    std::vector<uint8_t> c_st(ns), c_prof(ns), c_gcid(G);
    std::vector<uint16_t> c_mig(ns);
    std::vector<uint32_t> c_cseq(ns), c_amseq(ns), c_gw(G), c_gx(G);
    std::vector<int32_t> c_aslot(ns), c_apos(ns), c_ajob(ns);
    std::vector<uint8_t> c_ast(ns);
    std::vector<double> c_arem(ns), c_atkey(ns);
    uint32_t large_idx = 0;
    const bool block = G > 32 || std::getenv("MSG_EMU_FORCE_BLOCK") != nullptr;
    if (block) {
        tr.large = 1;
        tr.cl_goff = 0;
        a.large_idx = &large_idx;
        a.n_large = 1;
        a.c_st = c_st.data();
        a.c_prof = c_prof.data();
        a.c_mig = c_mig.data();
        a.c_cseq = c_cseq.data();
        a.c_apos = c_apos.data();
        a.c_aslot = c_aslot.data();
        a.c_ast = c_ast.data();
        a.c_ajob = c_ajob.data();
        a.c_amseq = c_amseq.data();
        a.c_arem = c_arem.data();
        a.c_atkey = c_atkey.data();
        a.c_gw = c_gw.data();
        a.c_gx = c_gx.data();
        a.c_gcid = c_gcid.data();
        const char* nt = std::getenv("MSG_EMU_BLOCK_THREADS");
        const char* gs = std::getenv("MSG_EMU_GPU_SMEM");  // "0": per-GPU words in global memory
        const char* sh = std::getenv("MSG_EMU_SHARDS");    // thread-block cluster size (shards)
        const bool smem = !(gs && gs[0] == '0');
        const unsigned S = sh ? (unsigned)std::atoi(sh) : 1u;
        const char* gr = std::getenv("MSG_EMU_GROUPS");  // device groups
        const unsigned D = gr ? (unsigned)std::atoi(gr) : 1u;
        if (S > 1 || D > 1) a.out_flags &= ~OF_EVENTS;  // the sharded engine runs without the event log
        a.max_gpus = (uint32_t)G;
        a.smem_gpus = smem ? (uint32_t)G : 0u;
        if (std::getenv("MSG_EMU_DEBUG")) std::fprintf(stderr, "emu block engine: S=%u G=%d\n", S, G);
        const char* ss = std::getenv("MSG_EMU_SLOT_SMEM");  // "0": slots in global memory
        run_block(a, &tables, nt ? (unsigned)std::atoi(nt) : 64u, S < 1 ? 1u : S, D < 1 ? 1u : D, smem,
                  !(ss && ss[0] == '0'), G);
    } else if (std::getenv("MSG_EMU_IO") && tc.identity) {
        // IO kernel: inputs read from the batch itself (zero copy) into
        // zeroed device arrays, SoA job rows + prefix word + flag in "host"
        // memory; checked against the device records afterwards
        std::fill(ha.begin(), ha.end(), 0.0);
        std::fill(hs.begin(), hs.end(), 0.0);
        std::fill(hp.begin(), hp.end(), 0);
        const uint64_t o = b->offsets[t];
        a.zc_arrival = b->arrival_s + o;
        a.zc_service = b->service_s + o;
        a.zc_profile = b->profile + o;
        a.perm = nullptr;
        a.out_flags = OF_JOBS;
        std::vector<double> soa(3 * N, -7.0);
        uint64_t prog = 0;
        uint32_t done = 0;
        DevSummary hsum{};
        a.jobs_host = reinterpret_cast<JobOut*>(soa.data());
        a.rows_soa = N;
        a.prog_host = &prog;
        a.prog_mask = 31;
        a.done_host = &done;
        a.done_epoch = 5;
        a.summary_host = &hsum;
        if (G <= 4) run_warp_io<1>(a, &tables);
        else if (G <= 8) run_warp_io<2>(a, &tables);
        else if (G <= 16) run_warp_io<4>(a, &tables);
        else run_warp_io<8>(a, &tables);
        bool ok = done == 5 && std::memcmp(&hsum, &sum, sizeof(sum)) == 0;
        if (sum.status == MSG_OK) {
            const uint64_t* gm = reinterpret_cast<const uint64_t*>(soa.data() + 2 * N);
            for (uint32_t k = 0; k < tr.n_jobs && ok; ++k)
                ok = std::memcmp(&soa[k], &jobs[k].sched, 8) == 0 && std::memcmp(&soa[N + k], &jobs[k].done, 8) == 0 &&
                     gm[k] == ((uint64_t)(uint32_t)jobs[k].gpu | ((uint64_t)(uint32_t)jobs[k].mig << 32)) &&
                     ha[k] == b->arrival_s[o + k] && hs[k] == b->service_s[o + k] && hp[k] == b->profile[o + k];
            ok = ok && (prog == 0 || ((prog >> 32) == 5 && (uint32_t)prog <= tr.n_jobs));
        }
        if (!ok) {
            r->status = r->summary.status = -99;
            r->message = "emulated IO kernel: host records differ from the device records";
            return r;
        }
    } else if (G <= 4) run_warp<1>(a, &tables);
    else if (G <= 8) run_warp<2>(a, &tables);
    else if (G <= 16) run_warp<4>(a, &tables);
    else run_warp<8>(a, &tables);

    msg_trace_summary& o = r->summary;
    o.status = sum.status;
    o.n_jobs = tr.n_jobs;
    o.handler_events = sum.handler_events;
    o.n_events = sum.n_events;
    o.timeline_samples = sum.timeline_samples;
    o.migration_count = sum.migrations;
    o.reconfig_op_count = sum.reconfig_ops;
    o.enqueue_count = sum.enqueues;
    o.dequeue_count = sum.dequeues;
    o.max_arrival_frag_evals = sum.max_arr;
    o.max_intra_iter_frag_evals = sum.max_intra;
    o.max_inter_iter_frag_evals = sum.max_inter;
    o.mean_wait_s = sum.mean_wait;
    o.mean_execution_s = sum.mean_exec;
    o.mean_turnaround_s = sum.mean_turn;
    o.workload_makespan_s = sum.makespan;
    o.timeline_sum = sum.tl_sum;
    r->status = sum.status;
    if (sum.status != MSG_OK) {
        r->message = "JobsPending: job " + std::to_string(sum.pending_rank >= 0 ? hid[sum.pending_rank] : -1) +
                     " did not complete";
        return r;
    }
    for (uint32_t k = 0; k < tr.n_jobs; ++k) {
        msg_job_row row;
        std::memset(&row, 0, sizeof(row));
        row.id = hid[k];
        row.arrival_s = ha[k];
        row.scheduled_s = jobs[k].sched;
        row.completed_s = jobs[k].done;
        row.wait_s = row.scheduled_s - row.arrival_s;
        row.execution_s = row.completed_s - row.scheduled_s;
        row.turnaround_s = row.wait_s + row.execution_s;
        row.profile = hp[k];
        row.gpu = jobs[k].gpu;
        row.migrations = jobs[k].mig;
        r->jobs.push_back(row);
    }
    const uint64_t ne = std::min<uint64_t>(sum.n_events, tr.ev_cap);
    r->events.resize(ne);
    for (uint64_t i = 0; i < ne; ++i) decode_event(evs[i], hid.data(), c->migration_overlap_s, &r->events[i]);
    const uint64_t nt = std::min<uint64_t>(sum.timeline_samples, tr.tl_cap);
    for (uint64_t i = 0; i < nt; ++i) r->timeline.push_back({tl[2 * i], tl[2 * i + 1]});
    return r;
}

int emu_result_status(void* h) { return static_cast<EmuResult*>(h)->status; }
const char* emu_result_message(void* h) { return static_cast<EmuResult*>(h)->message.c_str(); }
const msg_trace_summary* emu_result_summary(void* h) { return &static_cast<EmuResult*>(h)->summary; }
const msg_event* emu_result_events(void* h, uint64_t* n) {
    auto* r = static_cast<EmuResult*>(h);
    *n = r->events.size();
    return r->events.data();
}
const msg_job_row* emu_result_jobs(void* h, uint64_t* n) {
    auto* r = static_cast<EmuResult*>(h);
    *n = r->jobs.size();
    return r->jobs.data();
}
const msg_timeline_point* emu_result_timeline(void* h, uint64_t* n) {
    auto* r = static_cast<EmuResult*>(h);
    *n = r->timeline.size();
    return r->timeline.data();
}
void emu_result_free(void* h) { delete static_cast<EmuResult*>(h); }

}  // extern "C"

namespace {
template <int SPL>
void run_snap_warp(const SnapArgs& a, const DevTables* tb, uint32_t i) {
    auto ws = std::make_unique<WarpSmem<SPL>>();
    std::memset(ws.get(), 0xA5, sizeof(WarpSmem<SPL>));
    wp::EmuWarp warp;
    std::vector<std::thread> lanes;
    for (unsigned l = 0; l < 32; ++l)
        lanes.emplace_back([&, l]() {
            wp::g_warp = &warp;
            wp::g_lane = l;
            wp::g_phase = 0;
            snapshot_op<SPL>(a, tb, ws.get(), i);
        });
    for (auto& t : lanes) t.join();
}
}  // namespace

extern "C" {
// Decision-level snapshot op (decide.cu body) on the host emulation:
// op = SOP_*, slots updated in place (plans), out = n x 8 ints, events =
// n x ev_cap records.  Returns 0 or a staging status.
int emu_snapshot(int32_t op, uint32_t n, int32_t G, msg_instance* slots, const int32_t* arg, double threshold,
                 int32_t lb, int32_t dyn, int32_t enabled, double overlap, int32_t* out, EventRec* events,
                 uint32_t ev_cap) {
    Staged st;
    std::string err;
    msg_status e = stage_snapshots(n, G, slots, nullptr, nullptr, &st, &err);
    if (e != MSG_OK) return e;
    DevTables tables;
    build_tables(&tables);
    std::vector<uint32_t> wout(st.words.size());
    std::vector<int32_t> jout(st.jobs.size());
    SnapArgs a{};
    a.tables = &tables;
    a.slot_in = st.words.data();
    a.job_in = st.jobs.data();
    a.slot_out = wout.data();
    a.job_out = jout.data();
    a.arg = arg;
    a.out = out;
    a.events = events;
    a.ev_cap = ev_cap;
    a.n = n;
    a.G = G;
    a.op = op;
    a.cflags = (lb ? CF_LB : 0u) | (dyn ? CF_DYN : 0u);
    a.lazymask = lazymask_of(threshold);
    a.overlap = overlap;
    a.enabled = enabled;
    for (uint32_t i = 0; i < n; ++i) {
        if (G <= 4) run_snap_warp<1>(a, &tables, i);
        else if (G <= 8) run_snap_warp<2>(a, &tables, i);
        else if (G <= 16) run_snap_warp<4>(a, &tables, i);
        else run_snap_warp<8>(a, &tables, i);
    }
    if (op > SOP_DISPATCH) unstage_snapshots(n, G, wout, jout, st, slots);
    return 0;
}
}
