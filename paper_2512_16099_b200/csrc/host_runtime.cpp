// host_runtime.cpp — the C ABI of include/migsched_b200.h.
//
// Host responsibilities only: validation with the reference's error order
// (Engine::Engine, sim.cpp:73-116), staging traces into HBM in job-id (rank)
// order, launching the sm_100a kernels, and decoding the kernels' compact
// records into the ABI structs.  Every scheduling decision, planner step and
// event-loop step runs on the GPU (engine_core.cuh); there is no CPU path.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <immintrin.h>
#include <sys/mman.h>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include <chrono>
#include <cstdlib>

#include "dev_types.h"
#include "host_tables.h"
#include "staging.h"
#include "runtime.h"
#include "kernels.h"
#include "migsched_b200.h"

using namespace msgk;

struct msg_staged {
    msg_engine* eng = nullptr;
    uint32_t n_in = 0;
    uint32_t out_flags = 0;
    int spl = 1;
    std::vector<int32_t> status;      // per input trace (validation)
    std::vector<std::string> message;
    std::vector<int32_t> dev_index;   // input trace -> device trace or -1
    std::vector<uint32_t> src_of;     // device trace -> input trace
    std::vector<int32_t> gpu_count;   // per input trace
    std::vector<double> overlap;      // per device trace
    std::vector<DevTrace> traces;
    std::vector<DevConfig> configs;
    std::vector<uint32_t> init;
    uint64_t n_jobs = 0, ev_total = 0, tl_total = 0;
    bool any_perm = false;
    uint32_t ev_per_job = 16, tl_per_job = 8;
    uint64_t handler_events = 0;
    // block engine (G > 32): large traces and their cluster arena
    std::vector<uint32_t> large_idx;
    uint64_t large_gpus = 0;
    bool any_small = false;
    DevBuf d_large_idx, c_st, c_prof, c_mig, c_cseq, c_apos, c_aslot, c_ast, c_ajob, c_amseq, c_arem,
        c_atkey, c_gw, c_gx, c_gcid;
    uint32_t large_max_g = 0;
    uint32_t large_min_g = 0;
    const PeerBinding* peer = nullptr;  // set by msg_run_peer for one launch
    bool no_rerun = false;              // multi-GPU run: an output overflow cannot be re-run alone
    bool htr_ready = false;             // h_traces already holds the layout (stage_impl's fast path)
    // pinned host mirrors (rank order)
    HostBuf h_arrival, h_service, h_profile, h_perm, h_ids;
    HostBuf h_jobs, h_events, h_timeline, h_summary;
    HostBuf h_done;           // run_pipelined: per-trace completion flags (mapped, written by the kernel)
    HostBuf h_prog;           // run_pipelined: per-trace published row prefixes (epoch << 32 | jobs)
    HostBuf h_traces;         // run_pipelined: pinned copy of the trace descriptors (async H2D)
    uint32_t done_epoch = 0;  // the flag value of the current run
    // device
    DevBuf d_arrival, d_service, d_profile, d_perm, d_traces, d_configs, d_init, d_tables_unused;
    DevBuf d_prof32;  // run_pipelined, direct inputs: the caller's int32 profiles (narrowed in-kernel)
    DevBuf d_queue, d_jobs, d_events, d_timeline, d_summary;
    DevBuf d_inbox;  // device-group exchange inboxes (MSG_VDEV > 1)
};

namespace {
// MSG_PROFILE=1: per-phase host timings of msg_run_batch on stderr.
struct PhaseTimer {
    bool on = std::getenv("MSG_PROFILE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[msg] %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};
}  // namespace

namespace {
// Recycled per-job row buffers: a batch result's rows (72 B per job) go back
// here when the result is freed, so repeated batches of similar size write
// into already-faulted pages instead of fresh allocations.
struct FreeRows {
    void operator()(msg_job_row* p) const { std::free(p); }
};
struct RowBuf {
    std::unique_ptr<msg_job_row[], FreeRows> p;
    uint64_t cap = 0;
};
std::mutex g_rows_m;
std::vector<RowBuf> g_rows;

RowBuf take_rows(uint64_t n) {
    {
        std::lock_guard<std::mutex> lk(g_rows_m);
        for (size_t i = 0; i < g_rows.size(); ++i) {
            if (g_rows[i].cap >= n && g_rows[i].cap <= 2 * n + 1024) {
                RowBuf b = std::move(g_rows[i]);
                g_rows.erase(g_rows.begin() + (long)i);
                return b;
            }
        }
    }
    RowBuf b;
    b.cap = std::max<uint64_t>(n, 1);
    // 2 MiB-aligned and backed by transparent huge pages where the kernel
    // offers them (madvise mode): ~36x fewer first-touch faults for a C2
    // result (59 MB of rows).
    constexpr size_t kHuge = 2u << 20;
    const size_t bytes = (b.cap * sizeof(msg_job_row) + kHuge - 1) & ~(kHuge - 1);
    void* m = std::aligned_alloc(kHuge, bytes);
    if (!m) throw std::bad_alloc();
    madvise(m, bytes, MADV_HUGEPAGE);
    b.p.reset(static_cast<msg_job_row*>(m));
    return b;
}

void give_rows(RowBuf&& b) {
    if (!b.p) return;
    std::lock_guard<std::mutex> lk(g_rows_m);
    if (g_rows.size() < 2) g_rows.push_back(std::move(b));
}
}  // namespace

struct msg_batch_result {
    std::vector<msg_trace_summary> summaries;
    std::vector<std::string> messages;
    bool has_jobs = false;
    RowBuf jobs;  // all traces, trace-major (filled in parallel, no zero-init pass)
    uint64_t n_jobs_all = 0;
    std::vector<uint64_t> job_off;        // n_traces + 1
    std::vector<std::vector<msg_event>> events;
    std::vector<std::vector<msg_timeline_point>> timeline;
    ~msg_batch_result() { give_rows(std::move(jobs)); }
};

namespace {

// defer_arrays: validate, lay out and allocate, copy the per-trace metadata,
// but leave the job arrays (pinned staging + H2D) to the caller
// (run_pipelined, chunk by chunk).
// One per-job row (sim.cpp:467-500 JobRecord fields).
inline void put_row(msg_job_row* dst, int64_t id, double arrival, const JobOut& j, int32_t profile) {
    msg_job_row& row = *dst;
    row.id = id;
    row.arrival_s = arrival;
    row.scheduled_s = j.sched;
    row.completed_s = j.done;
    row.wait_s = row.scheduled_s - row.arrival_s;  // sim.cpp:473-475
    row.execution_s = row.completed_s - row.scheduled_s;
    row.turnaround_s = row.wait_s + row.execution_s;
    row.profile = profile;
    row.gpu = j.gpu;
    row.migrations = j.mig;
    row.reserved0 = 0;
}

// A trace's rows, written with non-temporal 16-byte stores in pairs (144 B
// = 9 aligned vectors): the row buffer is far larger than the caches and is
// not read back here, so the stores skip the read-for-ownership.
// nt false (MSG_ROWS_NT=0): plain stores.
// Job records as the kernels leave them on the host: AoS JobOut (event-loop
// kernel) or SoA columns sched / done / gpu | migrations << 32 (the
// pipelined IO kernel: every warp store then fills whole 128-byte lines).
struct JobsAoS {
    const JobOut* p;
    JobOut operator[](uint64_t i) const { return p[i]; }
    JobsAoS operator+(uint64_t i) const { return {p + i}; }
};
struct JobsSoA {
    const double* sched;
    const double* done;
    const uint64_t* gm;
    JobOut operator[](uint64_t i) const {
        const uint64_t x = gm[i];
        return JobOut{sched[i], done[i], (int32_t)(uint32_t)x, (int32_t)(uint32_t)(x >> 32)};
    }
    JobsSoA operator+(uint64_t i) const { return {sched + i, done + i, gm + i}; }
};

template <class P, class J>
inline void put_rows(msg_job_row* rows, uint32_t n, const int64_t* ids, const double* ha, const J hj,
                     const P* hp, bool nt) {
    uint32_t r = 0;
    if (nt) {
        if (n && (reinterpret_cast<uintptr_t>(rows) & 15)) {
            put_row(rows, ids[0], ha[0], hj[0], hp[0]);
            r = 1;
        }
        for (; r + 2 <= n; r += 2) {
            alignas(16) msg_job_row tmp[2];
            put_row(tmp, ids[r], ha[r], hj[r], hp[r]);
            put_row(tmp + 1, ids[r + 1], ha[r + 1], hj[r + 1], hp[r + 1]);
            const __m128i* src = reinterpret_cast<const __m128i*>(tmp);
            __m128i* dst = reinterpret_cast<__m128i*>(rows + r);
            for (int k = 0; k < 9; ++k) _mm_stream_si128(dst + k, _mm_load_si128(src + k));
        }
    }
    for (; r < n; ++r) put_row(rows + r, ids[r], ha[r], hj[r], hp[r]);
    if (nt) _mm_sfence();
}

// True when [p, p + bytes) is page-locked host memory this process has
// registered with CUDA (cudaHostAlloc / msg_host_alloc / cudaHostRegister):
// the copy engines can read it directly.
// *dev (optional): the device view of p (mapped page-locked memory: with
// unified addressing the address itself), null if not mapped.
bool host_pinned(const void* p, size_t bytes, const void** dev = nullptr) {
    if (dev) *dev = nullptr;
    if (!p || !bytes) return false;
    bool first = true;
    for (const void* q : {p, static_cast<const void*>(static_cast<const char*>(p) + bytes - 1)}) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, q) != cudaSuccess) {
            cudaGetLastError();  // clear the sticky "not a CUDA pointer" on old drivers
            return false;
        }
        if (at.type != cudaMemoryTypeHost) return false;
        if (first && dev) *dev = at.devicePointer;
        first = false;
    }
    return true;
}


// stage_impl's second half: pinned staging (unless deferred), device
// buffers, the H2D copies of configs / init / traces, and the ordering event.
msg_status stage_buffers(msg_engine* eng, msg_staged* s, const msg_trace_batch* b, bool defer_arrays) {
    PhaseTimer pt;
    const uint64_t njobs = s->n_jobs;
    // Host staging into pinned buffers, rank (job-id) order.
    const size_t N = std::max<uint64_t>(njobs, 1);
    CK(s->h_arrival.ensure(N * sizeof(double)));
    CK(s->h_service.ensure(N * sizeof(double)));
    CK(s->h_profile.ensure(N));
    CK(s->h_ids.ensure(N * sizeof(int64_t)));
    bool any_perm = defer_arrays;  // deferred checks: identity order is not known yet
    for (auto& tr : s->traces) any_perm |= tr.has_perm != 0;
    s->any_perm = any_perm;
    if (any_perm) CK(s->h_perm.ensure(N * sizeof(uint32_t)));
    double* ha = s->h_arrival.as<double>();
    double* hs = s->h_service.as<double>();
    uint8_t* hp = s->h_profile.as<uint8_t>();
    int64_t* hid = s->h_ids.as<int64_t>();
    uint32_t* hperm = any_perm ? s->h_perm.as<uint32_t>() : nullptr;
    if (!defer_arrays)
        parallel_for((uint32_t)s->traces.size(), 32, [&](uint32_t d) {
            stage_trace_arrays(b, s->src_of[d], s->traces[d], ha, hs, hp, hid, hperm);
        });
    pt.mark("  stage arrays");
    // Device buffers + H2D.
    cudaStream_t st = eng->stream;
    CK(s->d_arrival.ensure(N * sizeof(double)));
    CK(s->d_service.ensure(N * sizeof(double)));
    CK(s->d_profile.ensure(N));
    CK(s->d_queue.ensure(N * sizeof(int32_t)));
    CK(s->d_jobs.ensure(N * sizeof(JobOut)));
    CK(s->d_traces.ensure(std::max<size_t>(s->traces.size(), 1) * sizeof(DevTrace)));
    CK(s->d_configs.ensure(std::max<size_t>(s->configs.size(), 1) * sizeof(DevConfig)));
    CK(s->d_init.ensure(std::max<size_t>(s->init.size(), 1) * sizeof(uint32_t)));
    CK(s->d_summary.ensure(std::max<size_t>(s->traces.size(), 1) * sizeof(DevSummary)));
    if (any_perm) CK(s->d_perm.ensure(N * sizeof(uint32_t)));
    if (s->ev_total) CK(s->d_events.ensure(s->ev_total * sizeof(EventRec)));
    if (s->tl_total) CK(s->d_timeline.ensure(s->tl_total * 2 * sizeof(double)));
    if (!s->large_idx.empty()) {
        const size_t ng = s->large_gpus, ns = 8 * ng;
        CK(s->d_large_idx.ensure(s->large_idx.size() * 4));
        CK(s->c_st.ensure(ns));
        CK(s->c_prof.ensure(ns));
        CK(s->c_mig.ensure(ns * 2));
        CK(s->c_cseq.ensure(ns * 4));
        CK(s->c_apos.ensure(ns * 4));
        CK(s->c_aslot.ensure(ns * 4));
        CK(s->c_ast.ensure(ns));
        CK(s->c_ajob.ensure(ns * 4));
        CK(s->c_amseq.ensure(ns * 4));
        CK(s->c_arem.ensure(ns * 8));
        CK(s->c_atkey.ensure(ns * 8));
        CK(s->c_gw.ensure(ng * 4));
        CK(s->c_gx.ensure(ng * 4));
        CK(s->c_gcid.ensure(ng));
        CK(cudaMemcpyAsync(s->d_large_idx.p, s->large_idx.data(), s->large_idx.size() * 4, cudaMemcpyHostToDevice,
                           st));
    }
    if (njobs && !defer_arrays) {
        CK(cudaMemcpyAsync(s->d_arrival.p, ha, njobs * sizeof(double), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(s->d_service.p, hs, njobs * sizeof(double), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(s->d_profile.p, hp, njobs, cudaMemcpyHostToDevice, st));
        if (any_perm) CK(cudaMemcpyAsync(s->d_perm.p, hperm, njobs * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    }
    if (!s->traces.empty() && !defer_arrays)
        CK(cudaMemcpyAsync(s->d_traces.p, s->traces.data(), s->traces.size() * sizeof(DevTrace),
                           cudaMemcpyHostToDevice, st));
    if (!s->configs.empty())
        CK(cudaMemcpyAsync(s->d_configs.p, s->configs.data(), s->configs.size() * sizeof(DevConfig),
                           cudaMemcpyHostToDevice, st));
    if (!s->init.empty())
        CK(cudaMemcpyAsync(s->d_init.p, s->init.data(), s->init.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                           st));
    // Pageable sources: cudaMemcpyAsync returns once they are staged.  The
    // pipelined path orders its streams after these copies with an event
    // (no host wait); the plain path launches on this stream anyway, but its
    // callers read the staged object right away, so it waits.
    if (defer_arrays) {
        CK(cudaEventRecord(eng->staged, st));
    } else {
        CK(cudaStreamSynchronize(st));
    }
    return MSG_OK;
}

msg_status stage_impl(msg_engine* eng, const msg_trace_batch* b, const msg_config* cfgs, uint32_t n_cfgs,
                      uint32_t flags, msg_staged* s, bool defer_arrays = false) {
    if (!b || (b->n_traces && (!b->offsets || !b->job_id || !b->arrival_s || !b->profile || !b->service_s)) ||
        (n_cfgs == 0 && b->n_traces)) {
        eng->last_error = "InvalidArgument: null batch arrays or no configs";
        return MSG_ERR_INVALID_ARGUMENT;
    }
    s->eng = eng;
    // messages: clear only the previous call's (failing traces), keep the
    // vector (no per-call construction of n empty strings)
    for (size_t t = 0; t < s->status.size() && t < s->message.size(); ++t)
        if (s->status[t] != MSG_OK) s->message[t].clear();
    s->n_in = b->n_traces;
    s->out_flags = flags;
    s->status.assign(s->n_in, MSG_OK);
    s->message.resize(s->n_in);
    s->dev_index.assign(s->n_in, -1);
    s->gpu_count.assign(s->n_in, 0);
    s->configs.clear();
    s->init.clear();
    s->htr_ready = false;
    s->handler_events = 0;

    // Configs referenced by the batch.
    std::vector<CfgState> cs(n_cfgs);
    for (uint32_t i = 0; i < n_cfgs; ++i) cs[i] = validate_config(cfgs[i]);
    for (uint32_t i = 0; i < n_cfgs; ++i) {
        cs[i].dev.init_off = (uint32_t)s->init.size();
        s->init.insert(s->init.end(), cs[i].init.begin(), cs[i].init.end());
        s->configs.push_back(cs[i].dev);
    }

    PhaseTimer pt;
    // Fast layout for the pipelined path (checks deferred) with one valid
    // small-cluster config and no event log / timeline: every trace on the
    // device in input order, so the layout is the batch's own offsets and is
    // filled in parallel.
    bool one_cfg = n_cfgs == 1;
    if (one_cfg && b->config_index)
        for (uint32_t t = 0; t < s->n_in && one_cfg; ++t) one_cfg = b->config_index[t] == 0;
    if (defer_arrays && one_cfg && cs[0].status == MSG_OK && cfgs[0].gpu_count <= (int)kMaxGpusEnsemble &&
        !(flags & (MSG_OUT_EVENTS | MSG_OUT_TIMELINE))) {
        const uint32_t n = s->n_in;
        const uint64_t j0 = n ? b->offsets[0] : 0;
        s->traces.resize(n);  // every entry is rewritten below (no clear: no zero-fill pass)
        s->src_of.resize(n);
        s->overlap.assign(n, cfgs[0].migration_overlap_s);
        std::fill(s->gpu_count.begin(), s->gpu_count.end(), cfgs[0].gpu_count);
        CK(s->h_traces.ensure(std::max<uint32_t>(n, 1) * sizeof(DevTrace)));
        DevTrace* htr = s->h_traces.as<DevTrace>();  // the pinned copy for the H2D, written alongside
        parallel_for(n, 512, [&](uint32_t t) {
            DevTrace tr{};
            tr.job_off = b->offsets[t] - j0;
            tr.n_jobs = (uint32_t)(b->offsets[t + 1] - b->offsets[t]);
            s->traces[t] = tr;  // cfg 0, identity order until the checks say otherwise
            htr[t] = tr;
            s->src_of[t] = t;
            s->dev_index[t] = (int32_t)t;
        });
        s->htr_ready = true;
        s->large_idx.clear();
        s->large_gpus = 0;
        s->large_max_g = s->large_min_g = 0;
        s->any_small = n > 0;
        s->n_jobs = n ? b->offsets[n] - j0 : 0;
        const int maxG = cfgs[0].gpu_count;
        s->spl = maxG <= 4 ? 1 : maxG <= 8 ? 2 : maxG <= 16 ? 4 : 8;
        s->ev_total = s->tl_total = 0;
        s->any_perm = true;  // deferred checks: identity order is not known yet
        pt.mark("  layout (parallel)");
        return stage_buffers(eng, s, b, true);
    }
    s->src_of.clear();
    s->traces.clear();
    s->overlap.clear();
    // Per-trace validation (parallel), in input order.
    std::vector<TraceCheck> checks(s->n_in);
    for (uint32_t t = 0; t < s->n_in; ++t) {
        const uint32_t ci = b->config_index ? b->config_index[t] : 0;
        if (ci >= n_cfgs) {
            eng->last_error = "InvalidArgument: config_index out of range";
            return MSG_ERR_INVALID_ARGUMENT;
        }
    }
    // defer_arrays (the pipelined path): only config errors here; each
    // trace is checked by run_pipelined just before its chunk is staged,
    // and a failing one keeps its (unused) slot in the layout.
    parallel_for(s->n_in, defer_arrays ? 4096 : 64, [&](uint32_t t) {
        const uint32_t ci = b->config_index ? b->config_index[t] : 0;
        if (cs[ci].status != MSG_OK) {
            checks[t].status = cs[ci].status;
            checks[t].message = cs[ci].message;
            return;
        }
        if (!defer_arrays) checks[t] = check_trace(b, t);
    });

    pt.mark("  validate");
    uint64_t njobs = 0;
    int maxG = 1;
    s->large_idx.clear();
    s->large_gpus = 0;
    s->large_max_g = 0;
    s->large_min_g = 0;
    s->any_small = false;
    for (uint32_t t = 0; t < s->n_in; ++t) {
        const uint32_t ci = b->config_index ? b->config_index[t] : 0;
        s->gpu_count[t] = cfgs[ci].gpu_count;
        s->status[t] = checks[t].status;
        s->message[t] = checks[t].message;
        if (checks[t].status != MSG_OK) continue;
        DevTrace tr{};
        tr.job_off = njobs;
        tr.n_jobs = (uint32_t)(b->offsets[t + 1] - b->offsets[t]);
        tr.cfg = ci;
        tr.has_perm = checks[t].identity ? 0 : 1;
        tr.large = cfgs[ci].gpu_count > (int)kMaxGpusEnsemble ? 1u : 0u;
        if (tr.large) {
            tr.cl_goff = s->large_gpus;
            s->large_gpus += (uint64_t)cfgs[ci].gpu_count;
            s->large_max_g = std::max(s->large_max_g, (uint32_t)cfgs[ci].gpu_count);
            s->large_min_g = s->large_min_g ? std::min(s->large_min_g, (uint32_t)cfgs[ci].gpu_count)
                                            : (uint32_t)cfgs[ci].gpu_count;
            s->large_idx.push_back((uint32_t)s->traces.size());
        } else {
            s->any_small = true;
            maxG = std::max(maxG, cfgs[ci].gpu_count);
        }
        s->dev_index[t] = (int32_t)s->traces.size();
        s->src_of.push_back(t);
        s->traces.push_back(tr);
        s->overlap.push_back(cfgs[ci].migration_overlap_s);
        njobs += tr.n_jobs;
    }
    s->n_jobs = njobs;
    s->spl = maxG <= 4 ? 1 : maxG <= 8 ? 2 : maxG <= 16 ? 4 : 8;
    // Output capacities.
    uint64_t ev = 0, tl = 0;
    for (auto& tr : s->traces) {
        tr.ev_off = ev;
        tr.tl_off = tl;
        tr.ev_cap = (flags & MSG_OUT_EVENTS) ? s->ev_per_job * tr.n_jobs + 256 : 0;
        tr.tl_cap = (flags & MSG_OUT_TIMELINE) ? s->tl_per_job * tr.n_jobs + 64 : 0;
        ev += tr.ev_cap;
        tl += tr.tl_cap;
    }
    s->ev_total = ev;
    s->tl_total = tl;
    return stage_buffers(eng, s, b, defer_arrays);
}

// CTAs per large trace (cluster_core.cuh): >= 1024 GPUs per shard, up to
// kMaxShards; 1 when any large trace is within the exact-timeline size or
// the event log is requested.  MSG_SHARDS overrides the count (tuning).
bool shardable(uint32_t min_g, uint32_t out_flags) {
    return min_g > (uint32_t)kExactTimelineGpus && !(out_flags & OF_EVENTS);
}

// Device groups per large trace on this GPU (MSG_VDEV; default 1): the
// multi-GPU exchange protocol exercised with all groups on one device.
uint32_t choose_vdev(uint32_t min_g, uint32_t out_flags, uint32_t shards) {
    const char* e = std::getenv("MSG_VDEV");
    if (!e || !shardable(min_g, out_flags)) return 1;
    const int v = std::atoi(e);
    uint32_t D = v < 1 ? 1u : std::min<uint32_t>((uint32_t)v, (uint32_t)kMaxDev);
    while (D > 1 && min_g < D * shards) --D;
    return D;
}

uint32_t choose_shards(uint32_t min_g, uint32_t out_flags) {
    if (!shardable(min_g, out_flags)) return 1;
    uint32_t S = 1;
    if (const char* e = std::getenv("MSG_SHARDS")) {
        const int v = std::atoi(e);
        S = v < 1 ? 1u : std::min<uint32_t>((uint32_t)v, (uint32_t)kMaxShards);
    } else {
        while (S < (uint32_t)kMaxShards && min_g / (2 * S) >= 1024) S *= 2;
    }
    return std::min(S, min_g);
}

SimArgs make_args(msg_engine* eng, msg_staged* s) {
    SimArgs a{};
    a.traces = s->d_traces.as<DevTrace>();
    a.configs = s->d_configs.as<DevConfig>();
    a.init_slots = s->d_init.as<uint32_t>();
    a.tables = eng->tables.as<DevTables>();
    a.score_tab = eng->score_tab.as<uint16_t>();
    a.arrival = s->d_arrival.as<double>();
    a.service = s->d_service.as<double>();
    a.profile = s->d_profile.as<uint8_t>();
    a.perm = s->any_perm ? s->d_perm.as<uint32_t>() : nullptr;
    a.queue = s->d_queue.as<int32_t>();
    a.jobs = s->d_jobs.as<JobOut>();
    a.events = s->ev_total ? s->d_events.as<EventRec>() : nullptr;
    a.timeline = s->tl_total ? s->d_timeline.as<double>() : nullptr;
    a.summary = s->d_summary.as<DevSummary>();
    a.n_traces = (uint32_t)s->traces.size();
    a.out_flags = s->out_flags;
    // the no-delay kernels (engine_core.cuh, ND): reconfiguration latency
    // exactly +0 and no migration overlap in every config of the batch
    a.no_delay = 1;
    for (const DevConfig& c : s->configs)
        if (!(c.latency == 0.0 && !std::signbit(c.latency) && c.overlap <= 0.0)) a.no_delay = 0;
    a.n_large = (uint32_t)s->large_idx.size();
    if (a.n_large) {
        a.large_idx = s->d_large_idx.as<uint32_t>();
        a.c_st = s->c_st.as<uint8_t>();
        a.c_prof = s->c_prof.as<uint8_t>();
        a.c_mig = s->c_mig.as<uint16_t>();
        a.c_cseq = s->c_cseq.as<uint32_t>();
        a.c_apos = s->c_apos.as<int32_t>();
        a.c_aslot = s->c_aslot.as<int32_t>();
        a.c_ast = s->c_ast.as<uint8_t>();
        a.c_ajob = s->c_ajob.as<int32_t>();
        a.c_amseq = s->c_amseq.as<uint32_t>();
        a.c_arem = s->c_arem.as<double>();
        a.c_atkey = s->c_atkey.as<double>();
        a.max_gpus = s->large_max_g;
        a.shards = choose_shards(s->large_min_g, s->out_flags);
        a.n_dev = a.vdev = choose_vdev(s->large_min_g, s->out_flags, a.shards);
        a.dev0 = 0;  // inboxes are bound at launch (launch_impl)
        a.c_gw = s->c_gw.as<uint32_t>();
        a.c_gx = s->c_gx.as<uint32_t>();
        a.c_gcid = s->c_gcid.as<uint8_t>();
    }
    return a;
}

msg_status launch_impl(msg_engine* eng, msg_staged* s) {
    if (s->traces.empty()) return MSG_OK;
    SimArgs a = make_args(eng, s);
    if (s->peer) {  // one group of a multi-GPU run: this GPU's part of the trace
        const PeerBinding& pb = *s->peer;
        a.n_dev = pb.world;
        a.dev0 = pb.rank;
        a.vdev = 1;
        for (uint32_t k = 0; k < pb.world; ++k) a.inbox[k] = pb.inbox[k];
        a.epoch = pb.epoch;
        a.jobs = static_cast<JobOut*>(pb.jobs);
        a.summary = static_cast<DevSummary*>(pb.summary);
        a.timeline = static_cast<double*>(pb.timeline);
        cudaError_t e = launch_cluster(a, eng->stream);
        if (e != cudaSuccess) return cuda_fail(eng, e, "launch_cluster (peer)");
        ++eng->launches;
        return MSG_OK;
    }
    if (s->any_small) {
        cudaError_t e = launch_sim(s->spl, a, eng->stream);
        if (e != cudaSuccess) return cuda_fail(eng, e, "launch_sim");
        ++eng->launches;
    }
    if (a.n_large) {
        if (a.n_dev > 1) {
            const size_t bytes = (size_t)a.n_dev * a.n_large * sizeof(XInbox);
            CK(s->d_inbox.ensure(bytes));
            SimArgs b = a;  // one XInbox per (group, large trace); stamps zeroed per launch
            for (uint32_t k = 0; k < a.n_dev; ++k)
                b.inbox[k] = static_cast<char*>(s->d_inbox.p) + k * (size_t)a.n_large * sizeof(XInbox);
            CK(cudaMemsetAsync(s->d_inbox.p, 0, bytes, eng->stream));
            cudaError_t e = launch_cluster(b, eng->stream);
            if (e == cudaErrorCooperativeLaunchTooLarge)
            {
                eng->last_error = "Unsupported: device groups do not fit co-resident on this GPU";
                return MSG_ERR_UNSUPPORTED;
            }
            if (e != cudaSuccess) return cuda_fail(eng, e, "launch_cluster");
            ++eng->launches;
            return MSG_OK;
        }
        cudaError_t e = launch_cluster(a, eng->stream);
        if (e != cudaSuccess) return cuda_fail(eng, e, "launch_cluster");
        ++eng->launches;
    }
    return MSG_OK;
}

msg_status collect_impl(msg_engine* eng, msg_staged* s, msg_batch_result** out) {
    cudaStream_t st = eng->stream;
    const size_t T = s->traces.size();
    for (int attempt = 0;; ++attempt) {
        CK(s->h_summary.ensure(std::max<size_t>(T, 1) * sizeof(DevSummary)));
        if (T) CK(cudaMemcpyAsync(s->h_summary.p, s->d_summary.p, T * sizeof(DevSummary), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        // Output-capacity overflow: grow and re-run (deterministic, same result).
        const DevSummary* ds = s->h_summary.as<DevSummary>();
        bool overflow = false;
        for (size_t d = 0; d < T; ++d)
            overflow |= (s->traces[d].ev_cap && ds[d].n_events > s->traces[d].ev_cap) ||
                        (s->traces[d].tl_cap && ds[d].timeline_samples > s->traces[d].tl_cap);
        if (!overflow) break;
        if (attempt > 6 || s->no_rerun) {
            eng->last_error = "Unsupported: event log exceeds the output capacity";
            return MSG_ERR_UNSUPPORTED;
        }
        s->ev_per_job *= 4;
        s->tl_per_job *= 4;
        uint64_t ev = 0, tl = 0;
        for (auto& tr : s->traces) {
            tr.ev_off = ev;
            tr.tl_off = tl;
            tr.ev_cap = (s->out_flags & MSG_OUT_EVENTS) ? s->ev_per_job * tr.n_jobs + 256 : 0;
            tr.tl_cap = (s->out_flags & MSG_OUT_TIMELINE) ? s->tl_per_job * tr.n_jobs + 64 : 0;
            ev += tr.ev_cap;
            tl += tr.tl_cap;
        }
        s->ev_total = ev;
        s->tl_total = tl;
        if (ev) CK(s->d_events.ensure(ev * sizeof(EventRec)));
        if (tl) CK(s->d_timeline.ensure(tl * 2 * sizeof(double)));
        CK(cudaMemcpy(s->d_traces.p, s->traces.data(), T * sizeof(DevTrace), cudaMemcpyHostToDevice));
        msg_status ls = launch_impl(eng, s);
        if (ls != MSG_OK) return ls;
    }
    const bool want_jobs = (s->out_flags & MSG_OUT_JOBS) != 0;
    const bool want_ev = (s->out_flags & MSG_OUT_EVENTS) != 0;
    const bool want_tl = (s->out_flags & MSG_OUT_TIMELINE) != 0;
    if (want_jobs && s->n_jobs) {
        CK(s->h_jobs.ensure(s->n_jobs * sizeof(JobOut)));
        CK(cudaMemcpyAsync(s->h_jobs.p, s->d_jobs.p, s->n_jobs * sizeof(JobOut), cudaMemcpyDeviceToHost, st));
    }
    if (want_ev && s->ev_total) {
        CK(s->h_events.ensure(s->ev_total * sizeof(EventRec)));
        CK(cudaMemcpyAsync(s->h_events.p, s->d_events.p, s->ev_total * sizeof(EventRec), cudaMemcpyDeviceToHost, st));
    }
    if (want_tl && s->tl_total) {
        CK(s->h_timeline.ensure(s->tl_total * 2 * sizeof(double)));
        CK(cudaMemcpyAsync(s->h_timeline.p, s->d_timeline.p, s->tl_total * 2 * sizeof(double),
                           cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));

    auto res = std::make_unique<msg_batch_result>();
    res->summaries.resize(s->n_in);
    res->messages = s->message;
    if (want_jobs) {
        res->has_jobs = true;
        res->job_off.assign(s->n_in + 1, 0);
        for (uint32_t t = 0; t < s->n_in; ++t) {
            const int32_t d = s->dev_index[t];
            const bool rows = d >= 0 && s->h_summary.as<DevSummary>()[d].status == MSG_OK;
            res->job_off[t + 1] = res->job_off[t] + (rows ? s->traces[d].n_jobs : 0);
        }
        res->n_jobs_all = res->job_off[s->n_in];
        res->jobs = take_rows(res->n_jobs_all);
    }
    if (want_ev) res->events.resize(s->n_in);
    if (want_tl) res->timeline.resize(s->n_in);
    const DevSummary* ds = s->h_summary.as<DevSummary>();
    const JobOut* hj = s->h_jobs.as<JobOut>();
    const EventRec* he = s->h_events.as<EventRec>();
    const double* ht = s->h_timeline.as<double>();
    const double* ha = s->h_arrival.as<double>();
    const uint8_t* hp = s->h_profile.as<uint8_t>();
    const int64_t* hid = s->h_ids.as<int64_t>();
    std::atomic<uint64_t> handler{0};
    parallel_for(s->n_in, 64, [&](uint32_t t) {
        msg_trace_summary& o = res->summaries[t];
        std::memset(&o, 0, sizeof(o));
        o.status = s->status[t];
        o.gpu_count = s->gpu_count[t];
        const int32_t d = s->dev_index[t];
        if (d < 0) return;
        const DevTrace& tr = s->traces[d];
        const DevSummary& x = ds[d];
        o.status = x.status;
        o.n_jobs = tr.n_jobs;
        o.handler_events = x.handler_events;
        o.n_events = x.n_events;
        o.timeline_samples = x.timeline_samples;
        o.migration_count = x.migrations;
        o.reconfig_op_count = x.reconfig_ops;
        o.enqueue_count = x.enqueues;
        o.dequeue_count = x.dequeues;
        o.max_arrival_frag_evals = x.max_arr;
        o.max_intra_iter_frag_evals = x.max_intra;
        o.max_inter_iter_frag_evals = x.max_inter;
        o.mean_wait_s = x.mean_wait;
        o.mean_execution_s = x.mean_exec;
        o.mean_turnaround_s = x.mean_turn;
        o.workload_makespan_s = x.makespan;
        o.timeline_sum = x.tl_sum;
        handler += x.handler_events;
        const int64_t* ids = hid + tr.job_off;
        if (x.status == MSG_ERR_JOBS_PENDING) {
            const int64_t jid = x.pending_rank >= 0 ? ids[x.pending_rank] : -1;
            res->messages[t] = "JobsPending: job " + std::to_string(jid) + " did not complete";
            return;  // the reference throws: no report, no log
        }
        if (want_jobs) {
            msg_job_row* rows = res->jobs.p.get() + res->job_off[t];
            for (uint32_t r = 0; r < tr.n_jobs; ++r)
                put_row(rows + r, ids[r], ha[tr.job_off + r], hj[tr.job_off + r], hp[tr.job_off + r]);
        }
        if (want_ev) {
            auto& evs = res->events[t];
            const uint64_t n = std::min<uint64_t>(x.n_events, tr.ev_cap);
            evs.resize(n);
            for (uint64_t i = 0; i < n; ++i) decode_event(he[tr.ev_off + i], ids, s->overlap[d], &evs[i]);
        }
        if (want_tl) {
            auto& tlv = res->timeline[t];
            const uint64_t n = std::min<uint64_t>(x.timeline_samples, tr.tl_cap);
            tlv.resize(n);
            for (uint64_t i = 0; i < n; ++i)
                tlv[i] = msg_timeline_point{ht[2 * (tr.tl_off + i)], ht[2 * (tr.tl_off + i) + 1]};
        }
    });
    s->handler_events = handler.load();
    *out = res.release();
    return MSG_OK;
}


// ---- pipelined msg_run_batch for large ensembles ---------------------------
// Summary / job-row output over many small-cluster traces: the batch is cut
// into trace ranges (pipe_bounds), each on its own stream — host staging of
// chunk k+1 overlaps the H2D + kernel of chunk k, and the D2H + decode of
// the first chunks overlap the kernels of the last.  The chunk kernels run
// concurrently (one warp per trace, latency-bound), so the wall time is
// close to validation + one chunk's staging + the kernel + one chunk's
// readback.
constexpr int kMaxPipeChunks = 8;  // == size of msg_engine::pstream

// Chunk boundaries over the device traces: relative chunk weights from
// MSG_PIPE_W ("1,2,2,3"; tuning), else kDefaultPipe equal chunks.
constexpr int kDefaultPipe = 8;  // r01-v18 sweep (tools/pipe_tune.py): 8 equal chunks ~4% faster than 4 on the C2 e2e
int pipe_bounds(uint32_t T, uint32_t* d0s) {
    double w[kMaxPipeChunks];
    int n = 0;
    if (const char* e = std::getenv("MSG_PIPE_W")) {
        const char* c = e;
        while (*c && n < kMaxPipeChunks) {
            char* end = nullptr;
            const double v = std::strtod(c, &end);
            if (end == c) break;
            if (v > 0) w[n++] = v;
            c = *end == ',' ? end + 1 : end;
        }
    }
    if (n == 0)
        for (n = 0; n < kDefaultPipe; ++n) w[n] = 1.0;
    double tot = 0, acc = 0;
    for (int k = 0; k < n; ++k) tot += w[k];
    d0s[0] = 0;
    for (int k = 0; k < n; ++k) {
        acc += w[k];
        d0s[k + 1] = k + 1 == n ? T : (uint32_t)std::min<double>(T, std::floor(T * acc / tot));
    }
    return n;
}

void fill_summary(msg_trace_summary& o, const DevTrace& tr, const DevSummary& x) {
    o.status = x.status;
    o.n_jobs = tr.n_jobs;
    o.handler_events = x.handler_events;
    o.n_events = x.n_events;
    o.timeline_samples = x.timeline_samples;
    o.migration_count = x.migrations;
    o.reconfig_op_count = x.reconfig_ops;
    o.enqueue_count = x.enqueues;
    o.dequeue_count = x.dequeues;
    o.max_arrival_frag_evals = x.max_arr;
    o.max_intra_iter_frag_evals = x.max_intra;
    o.max_inter_iter_frag_evals = x.max_inter;
    o.mean_wait_s = x.mean_wait;
    o.mean_execution_s = x.mean_exec;
    o.mean_turnaround_s = x.mean_turn;
    o.workload_makespan_s = x.makespan;
    o.timeline_sum = x.tl_sum;
}

// Pauses between two idle polling sweeps over mapped host flags (tuning:
// MSG_POLL_BACKOFF).
int poll_backoff() {
    const char* e = std::getenv("MSG_POLL_BACKOFF");
    return e ? std::atoi(e) : 32;
}

msg_status run_pipelined(msg_engine* eng, const msg_trace_batch* b, msg_staged* s, msg_batch_result** out,
                         bool allow_zc = true) {
    const uint32_t T = (uint32_t)s->traces.size();
    const bool want_jobs = (s->out_flags & MSG_OUT_JOBS) != 0;
    PhaseTimer pt;
    uint32_t d0s[kMaxPipeChunks + 1];
    int n_chunks = pipe_bounds(T, d0s);
    // Job records reach the host through the kernel's own stores into mapped
    // pinned memory as each trace finishes (MSG_JOBS_D2H=1: one copy per chunk
    // after its kernel instead).
    auto env_off = [](const char* name) {
        const char* e = std::getenv(name);
        return e && e[0] == '0';
    };
    const bool jobs_d2h = std::getenv("MSG_JOBS_D2H") != nullptr;
    // Each trace also publishes its summary and a completion flag in mapped
    // host memory, so host threads decode traces as they finish, under the
    // kernels still running (MSG_PIPE_POLL=0: chunk by chunk after each
    // chunk's event).
    const bool poll = !jobs_d2h && !env_off("MSG_PIPE_POLL");
    const int kPollBackoff = poll_backoff();
    const bool rows_nt = !env_off("MSG_ROWS_NT");
    for (int k = 0; k < n_chunks; ++k) {
        if (!eng->pstream[k]) CK(cudaStreamCreateWithFlags(&eng->pstream[k], cudaStreamNonBlocking));
        if (!eng->pevent[k]) CK(cudaEventCreateWithFlags(&eng->pevent[k], cudaEventDisableTiming));
    }
    const size_t N = std::max<uint64_t>(s->n_jobs, 1);
    CK(s->h_summary.ensure(std::max<uint32_t>(T, 1) * sizeof(DevSummary)));
    if (want_jobs) CK(s->h_jobs.ensure(N * sizeof(JobOut)));
    if (poll) {
        const void* had = s->h_done.p;
        CK(s->h_done.ensure(std::max<uint32_t>(T, 1) * sizeof(uint32_t)));
        if (s->h_done.p != had) std::memset(s->h_done.p, 0, s->h_done.cap);
        if (++s->done_epoch == 0) s->done_epoch = 1;  // 0 is the zeroed buffer
    }
    volatile uint32_t* hdone = poll ? s->h_done.as<uint32_t>() : nullptr;
    double* ha = s->h_arrival.as<double>();
    double* hs = s->h_service.as<double>();
    uint8_t* hp = s->h_profile.as<uint8_t>();
    int64_t* hid = s->h_ids.as<int64_t>();
    uint32_t* hperm = s->any_perm ? s->h_perm.as<uint32_t>() : nullptr;
    SimArgs a = make_args(eng, s);
    auto joff = [&](uint32_t d) { return d < T ? s->traces[d].job_off : s->n_jobs; };
    // Direct inputs: when the caller's arrival / service / profile arrays are
    // page-locked (msg_host_alloc), the copy engines read them in place —
    // the host only validates (read-only) and there is no staging copy.
    // Requires the device layout to be the batch's own job order: every
    // input trace on the device, in order.  A chunk holding a trace whose
    // ids are not increasing (rank order differs from input order) is
    // staged as usual.  MSG_NO_DIRECT=1 disables it.
    const uint64_t jbase = T ? b->offsets[0] : 0, jall = T ? b->offsets[b->n_traces] - jbase : 0;
    const void *dv_a = nullptr, *dv_s = nullptr, *dv_p = nullptr;  // device views (zero copy)
    const bool direct = T && jall && s->traces.size() == s->n_in && std::getenv("MSG_NO_DIRECT") == nullptr &&
                        host_pinned(b->arrival_s + jbase, jall * sizeof(double), &dv_a) &&
                        host_pinned(b->service_s + jbase, jall * sizeof(double), &dv_s) &&
                        host_pinned(b->profile + jbase, jall * sizeof(int32_t), &dv_p);
    if (direct) CK(s->d_prof32.ensure(N * sizeof(int32_t)));
    CK(s->h_traces.ensure(std::max<uint32_t>(T, 1) * sizeof(DevTrace)));
    uint8_t chunk_direct[kMaxPipeChunks] = {};
    // Zero copy (direct inputs; MSG_NO_ZC=1 disables): the kernel reads the
    // caller's arrays in place over PCIe as each trace's arrivals reach them
    // (engine_core.cuh zc_fetch), so the whole batch launches at once, before
    // any host pass over the jobs, and the checks run on the host threads
    // under the kernel.  A trace failing its check is reported as such (its
    // device results are ignored); a valid trace whose ids are not increasing
    // needs the rank permutation, so then the batch re-runs staged.
    const bool zc = direct && allow_zc && !std::getenv("MSG_NO_ZC") && dv_a && dv_s && dv_p;
    const double* zc_a = zc ? static_cast<const double*>(dv_a) : nullptr;
    const double* zc_s = zc ? static_cast<const double*>(dv_s) : nullptr;
    const int32_t* zc_p = zc ? static_cast<const int32_t*>(dv_p) : nullptr;
    // Progressive rows (default with zero copy; MSG_PIPE_PROG=0 / 1 forces
    // off / on): each warp also publishes the completed prefix of its
    // trace's records as it goes, so the host decodes rows while the kernel
    // runs instead of after each trace ends (the decode is host-memory-bound:
    // ~95 MB of traffic for C2).  With staged chunks the finish times are
    // already spread by the chunks' staggered starts, and there the flushes
    // cost more than they save (profiles/r02, e2e_zc logs).
    const char* pe = std::getenv("MSG_PIPE_PROG");
    const bool prog = poll && want_jobs && !jobs_d2h && (pe ? pe[0] != '0' : zc_p != nullptr);
    if (prog) {
        const void* had = s->h_prog.p;
        CK(s->h_prog.ensure(std::max<uint32_t>(T, 1) * sizeof(uint64_t)));
        if (s->h_prog.p != had) std::memset(s->h_prog.p, 0, s->h_prog.cap);  // epoch 0 is never current
    }
    volatile uint64_t* hprog = prog ? s->h_prog.as<uint64_t>() : nullptr;
    // flush cadence in arrivals (MSG_PROG_EVERY, a power of two >= 32; tuning)
    uint32_t prog_mask = 63;  // r02 sweep (tools/zc_kernel_variants.py): 32 / 64 / 128 / 256 -> 1.71 / 1.60 / 1.71 / 1.69 ms
    if (const char* e = std::getenv("MSG_PROG_EVERY")) {
        const unsigned long v = std::strtoul(e, nullptr, 10);
        if (v >= 32 && (v & (v - 1)) == 0) prog_mask = (uint32_t)v - 1;
    }
    for (int k = 0; k < (zc_p ? 1 : n_chunks); ++k) CK(cudaStreamWaitEvent(eng->pstream[k], eng->staged, 0));
    if (zc_p) {
        cudaStream_t st = eng->pstream[0];
        n_chunks = 1;
        d0s[1] = T;
        DevTrace* htr = s->h_traces.as<DevTrace>();
        if (!s->htr_ready) std::memcpy(htr, s->traces.data(), T * sizeof(DevTrace));  // (the fast layout wrote it)
        CK(cudaMemcpyAsync(s->d_traces.as<DevTrace>(), htr, T * sizeof(DevTrace), cudaMemcpyHostToDevice, st));
        SimArgs c = a;
        c.perm = nullptr;
        c.zc_arrival = zc_a;
        c.zc_service = zc_s;
        c.zc_profile = zc_p;
        if (want_jobs && !jobs_d2h) c.jobs_host = s->h_jobs.as<JobOut>();
        if (poll) {
            c.summary_host = s->h_summary.as<DevSummary>();
            c.done_host = s->h_done.as<uint32_t>();
            c.done_epoch = s->done_epoch;
            if (prog) {
                c.prog_host = s->h_prog.as<uint64_t>();
                c.prog_mask = prog_mask;
            }
        }
        if (want_jobs && !jobs_d2h) c.rows_soa = s->n_jobs;
        if (pt.on) CK(cudaEventRecord(eng->ev0, st));
        cudaError_t e = launch_sim(s->spl, c, st);
        if (e != cudaSuccess) return cuda_fail(eng, e, "launch_sim (zero copy)");
        if (pt.on) CK(cudaEventRecord(eng->ev1, st));
        ++eng->launches;
        if (!poll)
            CK(cudaMemcpyAsync(s->h_summary.as<DevSummary>(), s->d_summary.as<DevSummary>(), T * sizeof(DevSummary),
                               cudaMemcpyDeviceToHost, st));
        if (want_jobs && jobs_d2h)
            CK(cudaMemcpyAsync(s->h_jobs.as<JobOut>(), s->d_jobs.as<JobOut>(), s->n_jobs * sizeof(JobOut),
                               cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(eng->pevent[0], st));
        pt.mark("  zero-copy launch");
        std::atomic<uint32_t> n_perm{0};
        parallel_for(T, 32, [&](uint32_t d) {
            const uint32_t t = s->src_of[d];
            TraceCheck ck = check_trace(b, t);
            if (ck.status != MSG_OK) {
                s->status[t] = ck.status;
                s->message[t] = std::move(ck.message);
            } else if (!ck.identity) {
                n_perm.fetch_add(1, std::memory_order_relaxed);
            }
        });
        pt.mark("  checks (under the kernel)");
        if (n_perm.load()) {
            CK(cudaEventSynchronize(eng->pevent[0]));
            return run_pipelined(eng, b, s, out, false);
        }
        chunk_direct[0] = 1;
    }
    for (int k = 0; k < n_chunks && !zc_p; ++k) {
        const uint32_t d0 = d0s[k], d1 = d0s[k + 1];
        if (d0 == d1) continue;
        cudaStream_t st = eng->pstream[k];
        // Check (sim.cpp:97-116) each trace of the chunk and, unless the
        // chunk goes direct, stage it while its inputs are hot; a failing
        // trace runs as an empty one and is reported from its check.
        std::atomic<uint32_t> n_perm{0};
        parallel_for(d1 - d0, 32, [&](uint32_t i) {
            const uint32_t d = d0 + i, t = s->src_of[d];
            DevTrace& tr = s->traces[d];
            TraceCheck c = check_trace(b, t);
            if (c.status != MSG_OK) {
                s->status[t] = c.status;
                s->message[t] = std::move(c.message);
                tr.n_jobs = 0;
                tr.has_perm = 0;
                return;
            }
            tr.has_perm = c.identity ? 0 : 1;
            if (tr.has_perm) n_perm.fetch_add(1, std::memory_order_relaxed);
            if (!direct) stage_trace_arrays(b, t, tr, ha, hs, hp, hid, hperm, false);  // ids stay in the batch
        });
        const bool cdirect = direct && n_perm.load() == 0;
        if (direct && !cdirect)
            parallel_for(d1 - d0, 32, [&](uint32_t i) {
                const uint32_t d = d0 + i, t = s->src_of[d];
                if (s->status[t] == MSG_OK) stage_trace_arrays(b, t, s->traces[d], ha, hs, hp, hid, hperm, false);
            });
        chunk_direct[k] = cdirect;
        DevTrace* htr = s->h_traces.as<DevTrace>();
        std::memcpy(htr + d0, s->traces.data() + d0, (d1 - d0) * sizeof(DevTrace));
        CK(cudaMemcpyAsync(s->d_traces.as<DevTrace>() + d0, htr + d0, (d1 - d0) * sizeof(DevTrace),
                           cudaMemcpyHostToDevice, st));
        const uint64_t j0 = joff(d0), j1 = joff(d1), nj = j1 - j0;
        if (nj && cdirect) {
            CK(cudaMemcpyAsync(s->d_arrival.as<double>() + j0, b->arrival_s + jbase + j0, nj * sizeof(double),
                               cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(s->d_service.as<double>() + j0, b->service_s + jbase + j0, nj * sizeof(double),
                               cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(s->d_prof32.as<int32_t>() + j0, b->profile + jbase + j0, nj * sizeof(int32_t),
                               cudaMemcpyHostToDevice, st));
        } else if (nj) {
            CK(cudaMemcpyAsync(s->d_arrival.as<double>() + j0, ha + j0, nj * sizeof(double), cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(s->d_service.as<double>() + j0, hs + j0, nj * sizeof(double), cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(s->d_profile.as<uint8_t>() + j0, hp + j0, nj, cudaMemcpyHostToDevice, st));
            if (n_perm.load())
                CK(cudaMemcpyAsync(s->d_perm.as<uint32_t>() + j0, hperm + j0, nj * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, st));
        }
        SimArgs c = a;
        c.profile32 = cdirect ? s->d_prof32.as<int32_t>() : nullptr;
        c.traces = s->d_traces.as<DevTrace>() + d0;
        c.summary = s->d_summary.as<DevSummary>() + d0;
        c.n_traces = d1 - d0;
        if (want_jobs && !jobs_d2h) c.jobs_host = s->h_jobs.as<JobOut>();  // finished traces store their rows
        if (poll) {
            c.summary_host = s->h_summary.as<DevSummary>() + d0;
            c.done_host = s->h_done.as<uint32_t>() + d0;
            c.done_epoch = s->done_epoch;
            if (prog) {
                c.prog_host = s->h_prog.as<uint64_t>() + d0;
                c.prog_mask = prog_mask;
                if (want_jobs) c.rows_soa = s->n_jobs;  // the IO kernel
            }
        }
        cudaError_t e = launch_sim(s->spl, c, st);
        if (e != cudaSuccess) return cuda_fail(eng, e, "launch_sim (pipelined)");
        ++eng->launches;
        if (!poll)
            CK(cudaMemcpyAsync(s->h_summary.as<DevSummary>() + d0, s->d_summary.as<DevSummary>() + d0,
                               (d1 - d0) * sizeof(DevSummary), cudaMemcpyDeviceToHost, st));
        if (want_jobs && nj && jobs_d2h)
            CK(cudaMemcpyAsync(s->h_jobs.as<JobOut>() + j0, s->d_jobs.as<JobOut>() + j0, nj * sizeof(JobOut),
                               cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(eng->pevent[k], st));
        pt.mark("  chunk staged+enqueued");
    }
    // Result layout: rows for every valid trace (JobsPending traces are
    // squeezed out at the end, a rare path).
    auto res = std::make_unique<msg_batch_result>();
    res->summaries.resize(s->n_in);
    res->messages = s->message;
    std::memset(res->summaries.data(), 0, s->n_in * sizeof(msg_trace_summary));
    for (uint32_t t = 0; t < s->n_in; ++t) {
        res->summaries[t].status = s->status[t];
        res->summaries[t].gpu_count = s->gpu_count[t];
    }
    if (want_jobs) {
        res->has_jobs = true;
        res->job_off.assign(s->n_in + 1, 0);
        for (uint32_t t = 0; t < s->n_in; ++t) {
            const int32_t d = s->dev_index[t];
            res->job_off[t + 1] = res->job_off[t] + (d >= 0 ? s->traces[d].n_jobs : 0);
        }
        res->n_jobs_all = res->job_off[s->n_in];
        res->jobs = take_rows(res->n_jobs_all);
    }
    const DevSummary* ds = s->h_summary.as<DevSummary>();
    const JobOut* hj = s->h_jobs.as<JobOut>();
    std::atomic<uint64_t> handler{0};
    std::atomic<bool> pending{false}, lost{false};
    // Waits for trace d's completion flag; false if its chunk ended (or
    // failed) without it — then the chunk's event reports the error below.
    auto wait_done = [&](uint32_t d) {
        int k = 0;
        while (k + 1 < n_chunks && d >= d0s[k + 1]) ++k;
        for (uint32_t spins = 1;; ++spins) {
            if (hdone[d] == s->done_epoch) break;
            for (int i = 1; i < kPollBackoff / 8; ++i) _mm_pause();
            if ((spins & 4095u) == 0) {
                const cudaError_t q = cudaEventQuery(eng->pevent[k]);
                if (q != cudaErrorNotReady && hdone[d] != s->done_epoch) {
                    lost = true;
                    return false;
                }
            }
            _mm_pause();
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        return true;
    };
    auto chunk_of = [&](uint32_t d) {
        int kc = 0;
        while (kc + 1 < n_chunks && d >= d0s[kc + 1]) ++kc;
        return kc;
    };
    // Rows [from, to) of device trace d into the result.
    // the IO kernel (zero copy or progressive rows) leaves SoA columns
    const bool io_soa = want_jobs && !jobs_d2h && (zc_p || prog);
    const double* hjd = s->h_jobs.as<double>();
    auto rows_range = [&](uint32_t d, uint32_t from, uint32_t to) {
        const uint32_t t = s->src_of[d];
        const DevTrace& tr = s->traces[d];
        const int64_t* ids = (tr.has_perm ? hid + tr.job_off : b->job_id + b->offsets[t]) + from;
        msg_job_row* dst = res->jobs.p.get() + res->job_off[t] + from;
        auto put = [&](auto jo) {
            if (chunk_direct[chunk_of(d)])  // arrival and profile straight from the caller's batch
                put_rows(dst, to - from, ids, b->arrival_s + b->offsets[t] + from, jo,
                         b->profile + b->offsets[t] + from, rows_nt);
            else
                put_rows(dst, to - from, ids, ha + tr.job_off + from, jo, hp + tr.job_off + from, rows_nt);
        };
        if (io_soa)
            put(JobsSoA{hjd, hjd + s->n_jobs, reinterpret_cast<const uint64_t*>(hjd + 2 * s->n_jobs)} +
                (tr.job_off + from));
        else
            put(JobsAoS{hj + tr.job_off + from});
    };
    // Device trace d has finished (summary and records visible): its summary
    // and its rows from `from` on.
    auto finish_trace = [&](uint32_t d, uint32_t from) {
        const uint32_t t = s->src_of[d];
        const DevTrace& tr = s->traces[d];
        const DevSummary& x = ds[d];
        fill_summary(res->summaries[t], tr, x);
        handler += x.handler_events;
        if (x.status == MSG_ERR_JOBS_PENDING) {
            const int64_t* ids = tr.has_perm ? hid + tr.job_off : b->job_id + b->offsets[t];
            const int64_t jid = x.pending_rank >= 0 ? ids[x.pending_rank] : -1;
            res->messages[t] = "JobsPending: job " + std::to_string(jid) + " did not complete";
            pending = true;
            return;
        }
        if (want_jobs && from < tr.n_jobs) rows_range(d, from, tr.n_jobs);
    };
    if (prog) {
        // Each host thread polls its share of the traces: new published
        // prefixes are decoded as they appear, a finished trace gets its tail
        // and summary.
        HostPool& pool = HostPool::get();
        const unsigned nth = std::min(pool.size(), std::max(1u, T / 32));
        std::atomic<unsigned> next_id{0};
        pool.run(nth, [&] {
            // blocks of 16 traces dealt round-robin: every thread gets traces
            // of every pipeline chunk (the chunks start at different times)
            const unsigned i = next_id.fetch_add(1);
            std::vector<uint32_t> open, dec;
            for (uint32_t b0 = 16 * i; b0 < T; b0 += 16 * nth)
                for (uint32_t d = b0; d < std::min(T, b0 + 16); ++d)
                    if (s->status[s->src_of[d]] == MSG_OK) open.push_back(d);
            dec.assign(open.size(), 0);
            for (uint32_t idle = 1; !open.empty();) {
                bool moved = false;
                for (size_t k = 0; k < open.size();) {
                    const uint32_t d = open[k];
                    if (hdone[d] == s->done_epoch) {
                        std::atomic_thread_fence(std::memory_order_acquire);
                        finish_trace(d, dec[k]);
                        open[k] = open.back();
                        dec[k] = dec.back();
                        open.pop_back();
                        dec.pop_back();
                        moved = true;
                        continue;
                    }
                    const uint64_t pw = hprog[d];
                    if ((uint32_t)(pw >> 32) == s->done_epoch && (uint32_t)pw > dec[k]) {
                        std::atomic_thread_fence(std::memory_order_acquire);
                        rows_range(d, dec[k], (uint32_t)pw);
                        dec[k] = (uint32_t)pw;
                        moved = true;
                    }
                    ++k;
                }
                if (moved) {
                    idle = 1;
                    continue;
                }
                // back off (~2 us) after a sweep without news: the flags and
                // prefixes share cache lines with the kernel's ongoing
                // PCIe writes, and tight polling slows those writes down
                for (int i = 0; i < kPollBackoff; ++i) _mm_pause();
                if ((++idle & 4095u) == 0) {  // every kernel ended and a trace never published: failure
                    bool all = true;
                    for (int c = 0; c < n_chunks && all; ++c)
                        all = d0s[c] == d0s[c + 1] || cudaEventQuery(eng->pevent[c]) != cudaErrorNotReady;
                    if (all && hdone[open[0]] != s->done_epoch) {
                        lost = true;
                        return;
                    }
                }
            }
        });
        pt.mark("  progressive decode");
    }
    for (int k = 0; k < (poll ? 1 : n_chunks) && !prog; ++k) {
        const uint32_t d0 = poll ? 0 : d0s[k], d1 = poll ? T : d0s[k + 1];
        if (d0 == d1) continue;
        if (!poll) CK(cudaEventSynchronize(eng->pevent[k]));
        pt.mark("  chunk kernel+D2H done");
        parallel_for(d1 - d0, 64, [&](uint32_t i) {
            const uint32_t d = d0 + i, t = s->src_of[d];
            if (s->status[t] != MSG_OK) return;  // failed its check: reported as such, no rows
            if (poll && !wait_done(d)) return;
            finish_trace(d, 0);
        });
        pt.mark("  chunk decoded");
    }
    if (poll) {
        for (int k = 0; k < n_chunks; ++k)
            if (d0s[k] != d0s[k + 1]) CK(cudaEventSynchronize(eng->pevent[k]));
        if (lost) {
            eng->last_error = "CudaError: a pipelined chunk completed without publishing a trace";
            return MSG_ERR_CUDA;
        }
    }
    if (pt.on && zc_p) {
        float ms = 0.f;
        CK(cudaEventSynchronize(eng->ev1));
        CK(cudaEventElapsedTime(&ms, eng->ev0, eng->ev1));
        std::fprintf(stderr, "[msg]   zero-copy kernel       %8.3f ms (device)\n", ms);
    }
    if (pending && want_jobs) {  // the reference throws for these traces: drop their rows
        uint64_t w = 0;
        std::vector<uint64_t> off(s->n_in + 1, 0);
        for (uint32_t t = 0; t < s->n_in; ++t) {
            const uint64_t b0 = res->job_off[t], n = res->job_off[t + 1] - b0;
            const bool keep = res->summaries[t].status == MSG_OK;
            if (keep && w != b0) std::memmove(res->jobs.p.get() + w, res->jobs.p.get() + b0, n * sizeof(msg_job_row));
            w += keep ? n : 0;
            off[t + 1] = w;
        }
        res->job_off = std::move(off);
        res->n_jobs_all = w;
    }
    s->handler_events = handler.load();
    *out = res.release();
    return MSG_OK;
}

uint64_t env_u64(const char* name, uint64_t dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::strtoull(e, nullptr, 10) : dflt;
}

// Warm start (msg_engine_create): the pipeline's streams, every event-loop
// kernel loaded, the host thread pool started, and a workspace for
// MSG_RESERVE_JOBS jobs (default 2^20; 0: none) in MSG_RESERVE_TRACES traces
// (default 8192) — pinned and device buffers plus a pre-faulted row buffer —
// so that the first msg_run_batch of up to that size pays no lazy kernel
// load, stream creation, allocation or first-touch page fault.
msg_status reserve_workspace(msg_engine* eng, msg_staged* s, uint64_t J, uint64_t T);

msg_status warm_engine(msg_engine* eng) {
    PhaseTimer pt;
    for (int k = 0; k < kMaxPipeChunks; ++k) {
        CK(cudaStreamCreateWithFlags(&eng->pstream[k], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&eng->pevent[k], cudaEventDisableTiming));
    }
    pt.mark("warm: streams");
    CK(preload_engine_kernels());
    pt.mark("warm: kernels loaded");
    parallel_for(1u << 12, 1, [](uint32_t) {});
    pt.mark("warm: host pool");
    const uint64_t J = env_u64("MSG_RESERVE_JOBS", 1ull << 20);
    const uint64_t T = std::max<uint64_t>(env_u64("MSG_RESERVE_TRACES", 8192), 1);
    if (!J) return MSG_OK;
    eng->cached = new msg_staged();
    // Best effort: a reservation that does not fit (pinned or device memory)
    // only costs the first call its allocations.
    const msg_status rs = reserve_workspace(eng, eng->cached, J, T);
    if (rs != MSG_OK) {
        cudaGetLastError();
        eng->last_error.clear();
    }
    pt.mark("warm: workspace");
    return MSG_OK;
}

msg_status reserve_workspace(msg_engine* eng, msg_staged* s, uint64_t J, uint64_t T) {
    PhaseTimer pt;
    // the sizes stage_impl / run_pipelined ask for at J jobs and T traces
    CK(s->h_arrival.ensure(J * sizeof(double)));
    CK(s->h_service.ensure(J * sizeof(double)));
    CK(s->h_profile.ensure(J));
    CK(s->h_ids.ensure(J * sizeof(int64_t)));
    CK(s->h_perm.ensure(J * sizeof(uint32_t)));
    CK(s->h_jobs.ensure(J * sizeof(JobOut)));
    CK(s->h_summary.ensure(T * sizeof(DevSummary)));
    CK(s->h_traces.ensure(T * sizeof(DevTrace)));
    CK(s->h_done.ensure(T * sizeof(uint32_t)));
    std::memset(s->h_done.p, 0, s->h_done.cap);
    CK(s->h_prog.ensure(T * sizeof(uint64_t)));
    std::memset(s->h_prog.p, 0, s->h_prog.cap);
    pt.mark("warm: pinned buffers");
    CK(s->d_arrival.ensure(J * sizeof(double)));
    CK(s->d_service.ensure(J * sizeof(double)));
    CK(s->d_profile.ensure(J));
    CK(s->d_prof32.ensure(J * sizeof(int32_t)));
    CK(s->d_perm.ensure(J * sizeof(uint32_t)));
    CK(s->d_queue.ensure(J * sizeof(int32_t)));
    CK(s->d_jobs.ensure(J * sizeof(JobOut)));
    CK(s->d_traces.ensure(T * sizeof(DevTrace)));
    CK(s->d_summary.ensure(T * sizeof(DevSummary)));
    pt.mark("warm: device buffers");
    // two row buffers: a caller that keeps the previous result while it
    // makes the next call needs both in rotation
    RowBuf rows[2] = {take_rows(J), take_rows(J)};
    for (RowBuf& rb : rows) {
        msg_job_row* r = rb.p.get();
        const uint64_t per_page = 4096 / sizeof(msg_job_row);  // a row in every 4 KiB page
        parallel_for((uint32_t)((J + 8191) / 8192), 1, [&](uint32_t i) {  // first touch, in parallel
            const uint64_t hi = std::min<uint64_t>(J, (uint64_t)(i + 1) * 8192);
            for (uint64_t j = (uint64_t)i * 8192; j < hi; j += per_page) r[j].id = 0;
        });
    }
    for (RowBuf& rb : rows) give_rows(std::move(rb));
    pt.mark("warm: row buffer");
    return MSG_OK;
}

}  // namespace

extern "C" {

const char* msg_status_name(int status) {
    if (status >= 0 && status <= 13) return kStatusNames[status];
    if (status == MSG_ERR_CUDA) return "CudaError";
    if (status == MSG_ERR_UNSUPPORTED) return "Unsupported";
    if (status == MSG_ERR_INVALID_ARGUMENT) return "InvalidArgument";
    return "Unknown";
}

msg_status msg_engine_create(int device, msg_engine** out) {
    if (!out) return MSG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    auto e = std::make_unique<msg_engine>();
    msg_engine* eng = e.get();
    e->device = device;
    int n = 0;
    cudaError_t err = cudaGetDeviceCount(&n);
    if (err != cudaSuccess || device < 0 || device >= n) {
        return MSG_ERR_CUDA;  // no usable device: there is no CPU fallback
    }
    PhaseTimer pt;
    CK(cudaSetDevice(device));
    pt.mark("create: context");
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    e->sm_count = prop.multiProcessorCount;
    std::snprintf(e->name, sizeof(e->name), "%s", prop.name);
    if (prop.major < 10) {
        return MSG_ERR_CUDA;  // kernels are built for sm_100a only
    }
    CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&e->ev0));
    CK(cudaEventCreate(&e->ev1));
    CK(cudaEventCreateWithFlags(&e->staged, cudaEventDisableTiming));
    DevTables t;
    if (build_tables(&t) != 31) return MSG_ERR_INVALID_ARGUMENT;
    CK(e->tables.ensure(sizeof(DevTables)));
    CK(cudaMemcpy(e->tables.p, &t, sizeof(DevTables), cudaMemcpyHostToDevice));
    std::vector<uint16_t> stab(kScoreTab);
    build_score_table(t, stab.data());
    CK(e->score_tab.ensure(sizeof(uint16_t) * kScoreTab));
    CK(cudaMemcpy(e->score_tab.p, stab.data(), sizeof(uint16_t) * kScoreTab, cudaMemcpyHostToDevice));
    const msg_status ws = warm_engine(eng);
    if (ws != MSG_OK) return ws;
    *out = e.release();
    return MSG_OK;
}

void msg_engine_destroy(msg_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    if (e->cached) msg_staged_free(e->cached);
    if (e->stream) cudaStreamSynchronize(e->stream);
    if (e->ev0) cudaEventDestroy(e->ev0);
    if (e->ev1) cudaEventDestroy(e->ev1);
    if (e->staged) cudaEventDestroy(e->staged);
    for (int k = 0; k < 8; ++k) {
        if (e->pstream[k]) {
            cudaStreamSynchronize(e->pstream[k]);
            cudaStreamDestroy(e->pstream[k]);
        }
        if (e->pevent[k]) cudaEventDestroy(e->pevent[k]);
    }
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

const char* msg_engine_last_error(const msg_engine* e) { return e ? e->last_error.c_str() : "no engine"; }

uint64_t msg_engine_launch_count(const msg_engine* e) { return e ? e->launches : 0; }

msg_status msg_engine_device_info(const msg_engine* e, char* name, size_t name_len, int32_t* sm_count) {
    if (!e) return MSG_ERR_INVALID_ARGUMENT;
    if (name && name_len) std::snprintf(name, name_len, "%s", e->name);
    if (sm_count) *sm_count = e->sm_count;
    return MSG_OK;
}

msg_status msg_stage(msg_engine* eng, const msg_trace_batch* batch, const msg_config* cfgs, uint32_t n_cfgs,
                     uint32_t out_flags, msg_staged** out) {
    if (!eng || !out) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    auto s = std::make_unique<msg_staged>();
    msg_status st = stage_impl(eng, batch, cfgs, n_cfgs, out_flags, s.get());
    if (st != MSG_OK) return st;
    *out = s.release();
    return MSG_OK;
}

msg_status msg_launch(msg_engine* eng, msg_staged* s) {
    if (!eng || !s) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    return launch_impl(eng, s);
}

msg_status msg_collect(msg_engine* eng, msg_staged* s, msg_batch_result** out) {
    if (!eng || !s || !out) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    return collect_impl(eng, s, out);
}

void msg_staged_free(msg_staged* s) { delete s; }

uint64_t msg_staged_handler_events(const msg_staged* s) { return s ? s->handler_events : 0; }

msg_status msg_run_batch(msg_engine* eng, const msg_trace_batch* batch, const msg_config* cfgs, uint32_t n_cfgs,
                         uint32_t out_flags, msg_batch_result** out) {
    if (!eng || !out) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    if (!eng->cached) eng->cached = new msg_staged();  // grow-only workspace reused across calls
    msg_staged* s = eng->cached;
    s->ev_per_job = 16;
    s->tl_per_job = 8;
    PhaseTimer pt;
    // Large ensembles of small clusters with summary / job-row output run
    // pipelined (run_pipelined); anything else through stage / launch / collect.
    const bool pipe = batch && batch->n_traces >= 512 && (out_flags & ~(uint32_t)MSG_OUT_JOBS) == 0 &&
                      std::getenv("MSG_NO_PIPELINE") == nullptr;
    msg_status st = stage_impl(eng, batch, cfgs, n_cfgs, out_flags, s, pipe);
    if (st != MSG_OK) return st;
    if (pipe) {
        if (s->large_idx.empty()) {
            st = run_pipelined(eng, batch, s, out);
            pt.mark("pipelined run");
            return st;
        }
        st = stage_impl(eng, batch, cfgs, n_cfgs, out_flags, s, false);  // large clusters: the plain path
        if (st != MSG_OK) return st;
    }
    pt.mark("stage (validate+H2D)");
    st = launch_impl(eng, s);
    if (st != MSG_OK) return st;
    if (pt.on) {
        cudaStreamSynchronize(eng->stream);
        pt.mark("kernel");
    }
    st = collect_impl(eng, s, out);
    pt.mark("collect (D2H+decode)");
    return st;
}

msg_status msg_host_alloc(size_t bytes, void** out) {
    if (!out) return MSG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (cudaHostAlloc(out, std::max<size_t>(bytes, 64), cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
        *out = nullptr;
        cudaGetLastError();
        return MSG_ERR_CUDA;
    }
    return MSG_OK;
}

void msg_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

msg_status msg_engine_sync(msg_engine* eng) {
    if (!eng) return MSG_ERR_INVALID_ARGUMENT;
    CK(cudaStreamSynchronize(eng->stream));
    return MSG_OK;
}

msg_status msg_time_launch(msg_engine* eng, msg_staged* s, float* ms) {
    if (!eng || !s || !ms) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    CK(cudaEventRecord(eng->ev0, eng->stream));
    msg_status st = launch_impl(eng, s);
    if (st != MSG_OK) return st;
    CK(cudaEventRecord(eng->ev1, eng->stream));
    CK(cudaEventSynchronize(eng->ev1));
    CK(cudaEventElapsedTime(ms, eng->ev0, eng->ev1));
    return MSG_OK;
}

msg_status msg_engine_flush_l2(msg_engine* eng) {
    msg_status st = msg_engine_flush_l2_async(eng);
    if (st != MSG_OK) return st;
    CK(cudaStreamSynchronize(eng->stream));
    return MSG_OK;
}

msg_status msg_engine_flush_l2_async(msg_engine* eng) {
    if (!eng) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    const size_t bytes = 256ull << 20;
    CK(eng->flush.ensure(bytes));
    CK(cudaMemsetAsync(eng->flush.p, eng->launches & 0xFF, bytes, eng->stream));
    return MSG_OK;
}

uint32_t msg_result_n_traces(const msg_batch_result* r) { return r ? (uint32_t)r->summaries.size() : 0; }

const msg_trace_summary* msg_result_summary(const msg_batch_result* r, uint32_t t) {
    return (r && t < r->summaries.size()) ? &r->summaries[t] : nullptr;
}

const msg_job_row* msg_result_jobs(const msg_batch_result* r, uint32_t t, uint64_t* n) {
    if (n) *n = 0;
    if (!r || !r->has_jobs || t + 1 >= r->job_off.size()) return nullptr;
    if (n) *n = r->job_off[t + 1] - r->job_off[t];
    return r->jobs.p.get() + r->job_off[t];
}

const msg_trace_summary* msg_result_summaries(const msg_batch_result* r) {
    return (r && !r->summaries.empty()) ? r->summaries.data() : nullptr;
}

const msg_job_row* msg_result_all_jobs(const msg_batch_result* r, const uint64_t** offsets, uint64_t* n) {
    if (n) *n = 0;
    if (offsets) *offsets = nullptr;
    if (!r || !r->has_jobs) return nullptr;
    if (offsets) *offsets = r->job_off.data();
    if (n) *n = r->n_jobs_all;
    return r->jobs.p.get();
}

const msg_event* msg_result_events(const msg_batch_result* r, uint32_t t, uint64_t* n) {
    if (n) *n = 0;
    if (!r || t >= r->events.size()) return nullptr;
    if (n) *n = r->events[t].size();
    return r->events[t].data();
}

const msg_timeline_point* msg_result_timeline(const msg_batch_result* r, uint32_t t, uint64_t* n) {
    if (n) *n = 0;
    if (!r || t >= r->timeline.size()) return nullptr;
    if (n) *n = r->timeline[t].size();
    return r->timeline[t].data();
}

const char* msg_result_message(const msg_batch_result* r, uint32_t t) {
    return (r && t < r->messages.size()) ? r->messages[t].c_str() : "";
}

void msg_result_free(msg_batch_result* r) { delete r; }

}  // extern "C"

// ---- multi-GPU device groups (one process per GPU) --------------------------
struct msg_peer {
    int device = 0;
    uint32_t world = 1, rank = 0;
    uint64_t max_jobs = 0, max_samples = 0;
    uint32_t epoch = 0;
    msgk::DevBuf inbox, jobs, summary, timeline;  // jobs / summary / timeline: rank 0 only
    void* p_inbox[kMaxDev] = {};
    void* p_jobs = nullptr;
    void* p_summary = nullptr;
    void* p_timeline = nullptr;
    std::vector<void*> opened;  // IPC mappings to close
    bool connected = false;
};

extern "C" {

size_t msg_peer_handle_size(void) { return 4 * sizeof(cudaIpcMemHandle_t); }

msg_status msg_peer_open(msg_engine* eng, int32_t world, int32_t rank, uint64_t max_jobs, msg_peer** out) {
    if (!eng || !out || world < 1 || world > kMaxDev || rank < 0 || rank >= world) return MSG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    cudaSetDevice(eng->device);
    auto p = std::make_unique<msg_peer>();
    p->device = eng->device;
    p->world = (uint32_t)world;
    p->rank = (uint32_t)rank;
    p->max_jobs = std::max<uint64_t>(max_jobs, 1);
    p->max_samples = 8 * p->max_jobs + 64;  // collect's timeline capacity (tl_per_job = 8)
    CK(p->inbox.ensure(sizeof(XInbox)));
    CK(cudaMemset(p->inbox.p, 0, p->inbox.cap));
    if (rank == 0) {
        CK(p->jobs.ensure(p->max_jobs * sizeof(JobOut)));
        CK(p->summary.ensure(sizeof(DevSummary)));
        CK(p->timeline.ensure(p->max_samples * 2 * sizeof(double)));
        p->p_jobs = p->jobs.p;
        p->p_summary = p->summary.p;
        p->p_timeline = p->timeline.p;
    }
    p->p_inbox[rank] = p->inbox.p;
    *out = p.release();
    return MSG_OK;
}

msg_status msg_peer_export(msg_peer* p, void* blob) {
    if (!p || !blob) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(p->device);
    cudaIpcMemHandle_t h[4];
    std::memset(h, 0, sizeof(h));
    msg_engine* eng = nullptr;  // CK needs the name; errors carry no engine message here
    CK(cudaIpcGetMemHandle(&h[0], p->inbox.p));
    if (p->rank == 0) {
        CK(cudaIpcGetMemHandle(&h[1], p->jobs.p));
        CK(cudaIpcGetMemHandle(&h[2], p->summary.p));
        CK(cudaIpcGetMemHandle(&h[3], p->timeline.p));
    }
    std::memcpy(blob, h, sizeof(h));
    return MSG_OK;
}

msg_status msg_peer_connect(msg_peer* p, const void* blobs) {
    if (!p || !blobs) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(p->device);
    msg_engine* eng = nullptr;
    const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(blobs);
    auto open = [&](const cudaIpcMemHandle_t& hd, void** ptr) -> cudaError_t {
        cudaError_t e = cudaIpcOpenMemHandle(ptr, hd, cudaIpcMemLazyEnablePeerAccess);
        if (e == cudaSuccess) p->opened.push_back(*ptr);
        return e;
    };
    for (uint32_t k = 0; k < p->world; ++k)
        if (k != p->rank) CK(open(h[4 * k], &p->p_inbox[k]));
    if (p->rank != 0) {
        CK(open(h[1], &p->p_jobs));
        CK(open(h[2], &p->p_summary));
        CK(open(h[3], &p->p_timeline));
    }
    p->connected = true;
    return MSG_OK;
}

void msg_peer_close(msg_peer* p) {
    if (!p) return;
    cudaSetDevice(p->device);
    for (void* q : p->opened) cudaIpcCloseMemHandle(q);
    delete p;
}

msg_status msg_run_peer(msg_engine* eng, msg_peer* p, const msg_trace_batch* batch, const msg_config* cfg,
                        uint32_t out_flags, msg_batch_result** out) {
    if (!eng || !p || !batch || !cfg || !p->connected) return MSG_ERR_INVALID_ARGUMENT;
    if (out) *out = nullptr;
    if (batch->n_traces != 1) {
        eng->last_error = "InvalidArgument: msg_run_peer takes one trace";
        return MSG_ERR_INVALID_ARGUMENT;
    }
    cudaSetDevice(eng->device);
    if (!eng->cached) eng->cached = new msg_staged();
    msg_staged* s = eng->cached;
    s->ev_per_job = 16;
    s->tl_per_job = 8;
    msg_status st = stage_impl(eng, batch, cfg, 1, out_flags & ~(uint32_t)MSG_OUT_EVENTS, s);
    if (st != MSG_OK) return st;
    if (!s->traces.empty()) {  // (validation is deterministic: every rank agrees)
        if (s->large_idx.size() != 1 || !shardable(s->large_min_g, s->out_flags)) {
            eng->last_error = "Unsupported: multi-GPU runs need more than 512 GPUs per cluster";
            return MSG_ERR_UNSUPPORTED;
        }
        if (s->n_jobs > p->max_jobs || s->tl_total > p->max_samples) {
            eng->last_error = "Unsupported: trace larger than the peer group's capacity";
            return MSG_ERR_UNSUPPORTED;
        }
        PeerBinding pb;
        pb.world = p->world;
        pb.rank = p->rank;
        pb.epoch = ++p->epoch;
        for (uint32_t k = 0; k < p->world; ++k) pb.inbox[k] = p->p_inbox[k];
        pb.jobs = p->p_jobs;
        pb.summary = p->p_summary;
        pb.timeline = p->p_timeline;
        s->peer = &pb;
        st = launch_impl(eng, s);
        s->peer = nullptr;
        if (st != MSG_OK) return st;
        CK(cudaStreamSynchronize(eng->stream));
        if (p->rank != 0) return MSG_OK;  // results live on rank 0
        CK(cudaMemcpyAsync(s->d_summary.p, p->p_summary, sizeof(DevSummary), cudaMemcpyDeviceToDevice, eng->stream));
        if (s->n_jobs)
            CK(cudaMemcpyAsync(s->d_jobs.p, p->p_jobs, s->n_jobs * sizeof(JobOut), cudaMemcpyDeviceToDevice,
                               eng->stream));
        if (s->tl_total)
            CK(cudaMemcpyAsync(s->d_timeline.p, p->p_timeline, s->tl_total * 2 * sizeof(double),
                               cudaMemcpyDeviceToDevice, eng->stream));
    } else if (p->rank != 0) {
        return MSG_OK;
    }
    s->no_rerun = true;
    st = out ? collect_impl(eng, s, out) : MSG_OK;
    s->no_rerun = false;
    return st;
}

}  // extern "C"
