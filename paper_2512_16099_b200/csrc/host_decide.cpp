// host_decide.cpp — decision-level entries of the C ABI: the reference's
// per-callback policy functions (scheduler.hpp:59-83, migration.hpp:46-63)
// on batches of cluster snapshots.  Host side: validation, job-id ranking,
// staging; all decisions run in decide.cu / score.cu kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "decide.h"
#include "dev_types.h"
#include "host_tables.h"
#include "migsched_b200.h"
#include "runtime.h"
#include "staging.h"

using namespace msgk;

namespace {

constexpr uint32_t kPlanEvCap = 4096;  // event records per snapshot (moves + reconfig ops)

struct SnapRun {
    std::vector<uint32_t> words_out;
    std::vector<int32_t> jobs_out;
    std::vector<int32_t> out;
    std::vector<EventRec> events;
};

msg_status run_snapshot_kernel(msg_engine* eng, SnapArgs a, const Staged& st, const std::vector<int32_t>& arg,
                               const std::vector<int32_t>* queue, const std::vector<uint32_t>* qlen,
                               const std::vector<uint8_t>* rprof, SnapRun* r) {
    const size_t slots = st.words.size();
    const size_t n = a.n;
    CK(eng->dscr[0].ensure(std::max<size_t>(slots, 1) * 4));
    CK(eng->dscr[1].ensure(std::max<size_t>(slots, 1) * 4));
    CK(eng->dscr[2].ensure(std::max<size_t>(slots, 1) * 4));
    CK(eng->dscr[3].ensure(std::max<size_t>(slots, 1) * 4));
    CK(eng->dscr[4].ensure(std::max<size_t>(n, 1) * 4));
    CK(eng->dscr[5].ensure(std::max<size_t>(n, 1) * 32));
    CK(eng->dscr[6].ensure(std::max<size_t>(n * a.ev_cap, 1) * sizeof(EventRec)));
    cudaStream_t s = eng->stream;
    CK(cudaMemcpyAsync(eng->dscr[0].p, st.words.data(), slots * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(eng->dscr[1].p, st.jobs.data(), slots * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(eng->dscr[4].p, arg.data(), n * 4, cudaMemcpyHostToDevice, s));
    a.tables = eng->tables.as<DevTables>();
    a.slot_in = eng->dscr[0].as<uint32_t>();
    a.job_in = eng->dscr[1].as<int32_t>();
    a.slot_out = eng->dscr[2].as<uint32_t>();
    a.job_out = eng->dscr[3].as<int32_t>();
    a.arg = eng->dscr[4].as<int32_t>();
    a.out = eng->dscr[5].as<int32_t>();
    a.events = eng->dscr[6].as<EventRec>();
    if (queue) {
        CK(eng->dscr[7].ensure(std::max<size_t>(queue->size(), 1) * 4));
        CK(eng->dscr[8].ensure(std::max<size_t>(qlen->size(), 1) * 4));
        CK(eng->dscr[9].ensure(std::max<size_t>(n * a.rank_cap, 1) * sizeof(JobOut)));
        CK(eng->dscr[10].ensure(std::max<size_t>(rprof->size(), 1)));
        CK(cudaMemcpyAsync(eng->dscr[7].p, queue->data(), queue->size() * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(eng->dscr[8].p, qlen->data(), qlen->size() * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(eng->dscr[10].p, rprof->data(), rprof->size(), cudaMemcpyHostToDevice, s));
        a.queue = eng->dscr[7].as<int32_t>();
        a.q_len = eng->dscr[8].as<uint32_t>();
        a.scratch = eng->dscr[9].as<JobOut>();
        a.rank_profile = eng->dscr[10].as<uint8_t>();
    }
    cudaError_t e = launch_snapshot(a, s);
    if (e != cudaSuccess) return cuda_fail(eng, e, "launch_snapshot");
    ++eng->launches;
    r->words_out.resize(slots);
    r->jobs_out.resize(slots);
    r->out.resize(n * 8);
    r->events.resize(n * a.ev_cap);
    CK(cudaMemcpyAsync(r->out.data(), a.out, n * 32, cudaMemcpyDeviceToHost, s));
    if (a.op > SOP_DISPATCH) {
        CK(cudaMemcpyAsync(r->words_out.data(), a.slot_out, slots * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(r->jobs_out.data(), a.job_out, slots * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(r->events.data(), a.events, n * a.ev_cap * sizeof(EventRec), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    return MSG_OK;
}

msg_status fail(msg_engine* eng, msg_status st, const std::string& m) {
    eng->last_error = m;
    return st;
}

}  // namespace

extern "C" {

uint64_t msg_pack_gpu_word(const msg_instance* s8) {
    uint64_t bc = 0, bm = 0, km = 0, ex = 0;
    for (int s = 0; s < 8; ++s) {
        const msg_instance& x = s8[s];
        if (x.state == MSG_SLOT_EMPTY || x.profile < 0 || x.profile >= MSG_PROFILE_COUNT) continue;
        if (!((host_startmask(x.profile) >> s) & 1u)) continue;
        const unsigned m = host_fpm(x.profile, s);
        if (x.state == MSG_SLOT_BUSY) {
            bc |= host_fpc(x.profile, s);
            bm |= m;
            km |= m;
        } else if (x.state == MSG_SLOT_DRAINING) {
            km |= m;
        } else {
            ex |= 1ull << placement_index(x.profile, s);
        }
    }
    return bc | (bm << 8) | (km << 16) | (ex << 24);
}

msg_status msg_score_device(msg_engine* eng, uint32_t n, int64_t G, const uint64_t* d_words, const uint8_t* d_profile,
                            const msg_sched_config* cfg, uint64_t* d_out) {
    if (!eng || !cfg || G < 0) return MSG_ERR_INVALID_ARGUMENT;
    if (G >= (1ll << 32)) return fail(eng, MSG_ERR_UNSUPPORTED, "Unsupported: gpu_count >= 2^32");
    cudaSetDevice(eng->device);
    ScoreArgs a{};
    a.tables = eng->tables.as<DevTables>();
    a.stab = eng->score_tab.as<uint16_t>();
    a.words = d_words;
    a.profile = d_profile;
    a.out = d_out;
    a.G = (uint64_t)G;
    a.n = n;
    a.lb = cfg->load_balancing ? 1u : 0u;
    a.dyn = cfg->dynamic_partitioning ? 1u : 0u;
    a.lazymask = lazymask_of(cfg->threshold);
    CK(eng->dscr[7].ensure((2 * (size_t)n + 1) * sizeof(uint32_t)));
    a.scratch = eng->dscr[7].as<uint32_t>();
    CK(eng->dscr[8].ensure(std::max<size_t>(score_items_bytes(n, (uint64_t)G), 16)));
    a.items = eng->dscr[8].as<uint64_t>();
    cudaError_t e = launch_score(a, eng->stream);
    if (e != cudaSuccess) return cuda_fail(eng, e, "launch_score");
    ++eng->launches;
    return MSG_OK;
}

// frag_cost(gpu) (frag.cpp:60-65) for n GPU snapshots of 8 slots each.
msg_status msg_frag_cost_batch(msg_engine* eng, uint32_t n, const msg_instance* slots, int32_t* numer,
                               double* cost) {
    if (!eng || (n && !slots)) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    if (!n) return MSG_OK;
    std::string err;
    std::vector<uint64_t> words(n);
    for (uint32_t i = 0; i < n; ++i) {
        msg_status e = check_gpu(slots + (size_t)i * 8, &err);
        if (e != MSG_OK) return fail(eng, e, err);
        words[i] = msg_pack_gpu_word(slots + (size_t)i * 8);
    }
    CK(eng->dscr[9].ensure((size_t)n * 8));
    CK(eng->dscr[10].ensure((size_t)n * 4));
    CK(eng->dscr[11].ensure((size_t)n * 8));
    CK(cudaMemcpyAsync(eng->dscr[9].p, words.data(), (size_t)n * 8, cudaMemcpyHostToDevice, eng->stream));
    cudaError_t e = launch_frag_cost(eng->tables.as<DevTables>(), eng->dscr[9].as<uint64_t>(), n,
                                     eng->dscr[10].as<int32_t>(), eng->dscr[11].as<double>(), eng->stream);
    if (e != cudaSuccess) return cuda_fail(eng, e, "launch_frag_cost");
    ++eng->launches;
    if (numer) CK(cudaMemcpyAsync(numer, eng->dscr[10].p, (size_t)n * 4, cudaMemcpyDeviceToHost, eng->stream));
    if (cost) CK(cudaMemcpyAsync(cost, eng->dscr[11].p, (size_t)n * 8, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaStreamSynchronize(eng->stream));
    return MSG_OK;
}

msg_status msg_time_score_device(msg_engine* eng, uint32_t n, int64_t G, const uint64_t* d_words,
                                 const uint8_t* d_profile, const msg_sched_config* cfg, uint64_t* d_out, float* ms) {
    if (!eng || !ms) return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    CK(cudaEventRecord(eng->ev0, eng->stream));
    msg_status st = msg_score_device(eng, n, G, d_words, d_profile, cfg, d_out);
    if (st != MSG_OK) return st;
    CK(cudaEventRecord(eng->ev1, eng->stream));
    CK(cudaEventSynchronize(eng->ev1));
    CK(cudaEventElapsedTime(ms, eng->ev0, eng->ev1));
    return MSG_OK;
}

// schedule / first_fit_schedule / dispatch_schedule (scheduler.cpp:47-104).
msg_status msg_schedule_batch(msg_engine* eng, int32_t op, uint32_t n, int32_t G, const msg_instance* slots,
                              const int32_t* profile, const msg_sched_config* cfg, msg_decision* out) {
    if (!eng || !slots || !profile || !cfg || !out || G < 0 || op < MSG_OP_SCHEDULE || op > MSG_OP_DISPATCH)
        return MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    std::memset(out, 0, sizeof(msg_decision) * n);
    for (uint32_t i = 0; i < n; ++i)
        if (profile[i] < 0 || profile[i] >= MSG_PROFILE_COUNT)  // require_known_profile (scheduler.cpp:11-15)
            return fail(eng, MSG_ERR_UNKNOWN_PROFILE, "UnknownProfile: job requests an unknown profile");
    const bool lb = op == MSG_OP_SCHEDULE || (op == MSG_OP_DISPATCH && cfg->load_balancing);
    if (lb && G > 0 && (cfg->threshold < 0.0 || cfg->threshold > 1.0))  // classify (gpu.cpp:172-177)
        return fail(eng, MSG_ERR_BAD_THRESHOLD, "BadThreshold: load-balancing threshold must be in [0,1]");
    std::string err;
    if (G <= 32) {
        Staged st;
        msg_status e = stage_snapshots(n, G, slots, nullptr, nullptr, &st, &err);
        if (e != MSG_OK) return fail(eng, e, err);
        if (G == 0 || n == 0) return MSG_OK;
        SnapArgs a{};
        a.n = n;
        a.G = G;
        a.op = op;
        a.cflags = (lb ? CF_LB : 0u) | (cfg->dynamic_partitioning ? CF_DYN : 0u);
        a.lazymask = lazymask_of(cfg->threshold);
        a.ev_cap = 1;
        std::vector<int32_t> arg(profile, profile + n);
        SnapRun r;
        e = run_snapshot_kernel(eng, a, st, arg, nullptr, nullptr, nullptr, &r);
        if (e != MSG_OK) return e;
        for (uint32_t i = 0; i < n; ++i) {
            const int32_t* o = &r.out[i * 8];
            out[i] = msg_decision{o[0], o[1], o[2], o[3], o[4], o[5]};
        }
        return MSG_OK;
    }
    // Large clusters: packed words streamed through the HBM scorer.
    for (uint32_t i = 0; i < n; ++i)
        for (int g = 0; g < G; ++g) {
            msg_status e = check_gpu(slots + ((size_t)i * G + g) * 8, &err);
            if (e != MSG_OK) return fail(eng, e, err);
        }
    std::vector<uint64_t> words((size_t)n * G);
    for (size_t k = 0; k < words.size(); ++k) words[k] = msg_pack_gpu_word(slots + k * 8);
    std::vector<uint8_t> prof(profile, profile + n);
    CK(eng->dscr[0].ensure(std::max<size_t>(words.size(), 1) * 8));
    CK(eng->dscr[1].ensure(std::max<size_t>(n, 1)));
    CK(eng->dscr[2].ensure(std::max<size_t>(n, 1) * 16));
    CK(cudaMemcpyAsync(eng->dscr[0].p, words.data(), words.size() * 8, cudaMemcpyHostToDevice, eng->stream));
    CK(cudaMemcpyAsync(eng->dscr[1].p, prof.data(), n, cudaMemcpyHostToDevice, eng->stream));
    msg_sched_config c2 = *cfg;
    c2.load_balancing = lb ? 1 : 0;
    msg_status e = msg_score_device(eng, n, G, eng->dscr[0].as<uint64_t>(), eng->dscr[1].as<uint8_t>(), &c2,
                                    eng->dscr[2].as<uint64_t>());
    if (e != MSG_OK) return e;
    std::vector<uint64_t> res((size_t)n * 2);
    CK(cudaMemcpyAsync(res.data(), eng->dscr[2].p, n * 16, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaStreamSynchronize(eng->stream));
    for (uint32_t i = 0; i < n; ++i) {
        const uint64_t k = res[2 * i];
        const uint32_t nl = (uint32_t)(res[2 * i + 1] >> 32), nb = (uint32_t)res[2 * i + 1];
        msg_decision d{};
        d.evaluated_candidates = lb ? (int32_t)(nl + (nl == 0 ? nb : 0)) : 0;
        if (k != ~0ull) {
            d.placed = 1;
            d.gpu = (int32_t)((k >> 3) & 0xFFFFFFFFull);
            d.start = (int32_t)(k & 7);
            d.size = host_ms(profile[i]);
            if (lb) {
                d.reused = ((k >> 35) & 1) == 0;
            } else {
                const msg_instance& x = slots[((size_t)i * G + d.gpu) * 8 + d.start];
                d.reused = x.state == MSG_SLOT_IDLE && x.profile == profile[i];
            }
        }
        out[i] = d;
    }
    return MSG_OK;
}

// on_departure / plan_intra / plan_inter (migration.cpp:71-220).
msg_status msg_plan_batch(msg_engine* eng, int32_t op, uint32_t n, int32_t G, msg_instance* slots, const int32_t* gpu,
                          double threshold, int32_t enabled, double overlap_s, uint32_t max_moves, msg_move* moves,
                          msg_plan_summary* sums) {
    if (!eng || !slots || !gpu || !sums || G < 1 || G > 32 || op < MSG_PLAN_ON_DEPARTURE || op > MSG_PLAN_INTER)
        return eng ? fail(eng, G > 32 ? MSG_ERR_UNSUPPORTED : MSG_ERR_INVALID_ARGUMENT,
                          "InvalidArgument: plan batch arguments (G in 1..32)")
                   : MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    std::memset(sums, 0, sizeof(msg_plan_summary) * n);
    std::string err;
    Staged st;
    msg_status e = stage_snapshots(n, G, slots, nullptr, nullptr, &st, &err);
    if (e != MSG_OK) return fail(eng, e, err);
    // Per-snapshot argument checks in the reference's order.
    std::vector<uint32_t> run;
    std::vector<int32_t> arg(n, 0);
    const bool classifies = op == MSG_PLAN_INTER || (op == MSG_PLAN_ON_DEPARTURE && enabled);
    for (uint32_t i = 0; i < n; ++i) {
        sums[i].kind = -1;
        if (gpu[i] < 0 || gpu[i] >= G) {
            sums[i].status = MSG_ERR_UNKNOWN_GPU;  // gpu_at (migration.cpp:12-17)
            continue;
        }
        if (classifies && (threshold < 0.0 || threshold > 1.0)) {
            sums[i].status = MSG_ERR_BAD_THRESHOLD;
            continue;
        }
        arg[i] = gpu[i];
    }
    SnapArgs a{};
    a.n = n;
    a.G = G;
    a.op = op == MSG_PLAN_ON_DEPARTURE ? SOP_ON_DEPARTURE : op == MSG_PLAN_INTRA ? SOP_PLAN_INTRA : SOP_PLAN_INTER;
    a.cflags = 0;
    a.lazymask = lazymask_of(threshold);
    a.overlap = overlap_s;
    a.enabled = enabled;
    a.ev_cap = kPlanEvCap;
    SnapRun r;
    e = run_snapshot_kernel(eng, a, st, arg, nullptr, nullptr, nullptr, &r);
    if (e != MSG_OK) return e;
    std::vector<msg_instance> before(slots, slots + (size_t)n * G * 8);
    unstage_snapshots(n, G, r.words_out, r.jobs_out, st, slots);
    for (uint32_t i = 0; i < n; ++i) {
        const size_t b = (size_t)i * G * 8;
        if (sums[i].status != MSG_OK) {  // rejected before planning: state untouched
            std::copy(before.begin() + b, before.begin() + b + (size_t)G * 8, slots + b);
            continue;
        }
        const int32_t* o = &r.out[i * 8];
        sums[i].status = o[0];
        sums[i].kind = o[1];
        sums[i].n_moves = o[2];
        sums[i].n_iterations = o[3];
        sums[i].max_evals = o[4];
        if (o[0] != MSG_OK) {
            std::copy(before.begin() + b, before.begin() + b + (size_t)G * 8, slots + b);
            continue;
        }
        if ((uint32_t)o[5] > a.ev_cap) sums[i].status = MSG_ERR_UNSUPPORTED;  // plan longer than the record buffer
        // Decode moves from the MigrationStart / Reconfig records.
        const EventRec* ev = &r.events[(size_t)i * a.ev_cap];
        const uint32_t ne = std::min<uint32_t>((uint32_t)o[5], a.ev_cap);
        uint32_t m = 0;
        for (uint32_t k = 0; k < ne; ++k) {
            if (ev[k].kind != 2) continue;
            if (m < max_moves && moves) {
                msg_event me;
                decode_event(ev[k], st.ids[i].data(), overlap_s, &me);
                msg_move& mv = moves[(size_t)i * max_moves + m];
                std::memset(&mv, 0, sizeof(mv));
                mv.job = me.job;
                mv.profile = me.profile;
                mv.from_gpu = me.from_gpu;
                mv.from_start = me.from_start;
                mv.to_gpu = me.to_gpu;
                mv.to_start = me.to_start;
                mv.move_kind = me.move_kind;
                mv.from_cost_before = me.from_cost_before;
                mv.from_cost_after = me.from_cost_after;
                mv.to_cost_before = me.to_cost_before;
                mv.to_cost_after = me.to_cost_after;
                int destroyed = 0, created = 0;
                for (uint32_t q = k + 1; q < ne && ev[q].kind == 4; ++q) {
                    if (ev[q].flags & EF_DESTROY) ++destroyed;
                    else ++created;
                }
                mv.n_destroyed = destroyed;
                mv.reused = created == 0;
            }
            ++m;
        }
    }
    return MSG_OK;
}

// try_dequeue (scheduler.cpp:106-121).
msg_status msg_try_dequeue_batch(msg_engine* eng, uint32_t n, int32_t G, msg_instance* slots, const uint64_t* qoff,
                                 const int64_t* qjob, const int32_t* qprof, const msg_sched_config* cfg,
                                 msg_dequeue_item* placed, uint32_t* n_placed) {
    if (!eng || !slots || !qoff || !cfg || !n_placed || G < 0 || G > 32)
        return eng ? fail(eng, G > 32 ? MSG_ERR_UNSUPPORTED : MSG_ERR_INVALID_ARGUMENT,
                          "InvalidArgument: try_dequeue batch arguments (G <= 32)")
                   : MSG_ERR_INVALID_ARGUMENT;
    cudaSetDevice(eng->device);
    std::string err;
    for (uint32_t i = 0; i < n; ++i) {
        n_placed[i] = 0;
        for (uint64_t k = qoff[i]; k < qoff[i + 1]; ++k)
            if (qprof[k] < 0 || qprof[k] >= MSG_PROFILE_COUNT)
                return fail(eng, MSG_ERR_UNKNOWN_PROFILE, "UnknownProfile: queued job with an unknown profile");
    }
    if (cfg->load_balancing && G > 0 && (cfg->threshold < 0.0 || cfg->threshold > 1.0))
        return fail(eng, MSG_ERR_BAD_THRESHOLD, "BadThreshold: load-balancing threshold must be in [0,1]");
    Staged st;
    msg_status e = stage_snapshots(n, G, slots, qoff, qjob, &st, &err);
    if (e != MSG_OK) return fail(eng, e, err);
    if (G == 0 || n == 0) return MSG_OK;
    uint32_t qcap = 1, rcap = 1;
    for (uint32_t i = 0; i < n; ++i) {
        qcap = std::max<uint32_t>(qcap, (uint32_t)(qoff[i + 1] - qoff[i]));
        rcap = std::max<uint32_t>(rcap, (uint32_t)st.ids[i].size());
    }
    std::vector<int32_t> queue((size_t)n * qcap, 0);
    std::vector<uint32_t> qlen(n);
    std::vector<uint8_t> rprof((size_t)n * rcap, 0);
    for (uint32_t i = 0; i < n; ++i) {
        qlen[i] = (uint32_t)(qoff[i + 1] - qoff[i]);
        const auto& ids = st.ids[i];
        for (uint64_t k = qoff[i]; k < qoff[i + 1]; ++k) {
            const int32_t r = (int32_t)(std::lower_bound(ids.begin(), ids.end(), qjob[k]) - ids.begin());
            queue[(size_t)i * qcap + (k - qoff[i])] = r;
            rprof[(size_t)i * rcap + r] = (uint8_t)qprof[k];
        }
    }
    SnapArgs a{};
    a.n = n;
    a.G = G;
    a.op = SOP_TRY_DEQUEUE;
    a.cflags = (cfg->load_balancing ? CF_LB : 0u) | (cfg->dynamic_partitioning ? CF_DYN : 0u);
    a.lazymask = lazymask_of(cfg->threshold);
    a.q_cap = qcap;
    a.rank_cap = rcap;
    a.ev_cap = qcap * 10 + 16;
    SnapRun r;
    std::vector<int32_t> arg(n, 0);
    e = run_snapshot_kernel(eng, a, st, arg, &queue, &qlen, &rprof, &r);
    if (e != MSG_OK) return e;
    unstage_snapshots(n, G, r.words_out, r.jobs_out, st, slots);
    for (uint32_t i = 0; i < n; ++i) {
        const int32_t* o = &r.out[i * 8];
        n_placed[i] = (uint32_t)o[0];
        const EventRec* ev = &r.events[(size_t)i * a.ev_cap];
        const uint32_t ne = std::min<uint32_t>((uint32_t)o[1], a.ev_cap);
        uint32_t m = 0;
        for (uint32_t k = 0; k < ne; ++k) {
            if (ev[k].kind != 6) continue;
            msg_dequeue_item& it = placed[qoff[i] + m++];
            it.job = st.ids[i][ev[k].job];
            it.gpu = ev[k].gpu;
            it.start = ev[k].start;
            it.size = host_ms(ev[k].profile);
            it.reused = (ev[k].flags & EF_REUSED) ? 1 : 0;
            it.evaluated_candidates = (int32_t)ev[k].aux;
            int destroyed = 0;
            for (uint32_t q = k + 1; q < ne && ev[q].kind == 4; ++q) destroyed += (ev[q].flags & EF_DESTROY) ? 1 : 0;
            it.n_destroyed = destroyed;
        }
    }
    return MSG_OK;
}

}  // extern "C"
