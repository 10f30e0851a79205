// engine_core.cuh — one warp replays one trace of the reference's
// discrete-event MIG scheduler (proj/src/sim.cpp:71-410) bit-exactly.
//
// Layout (per warp, in shared memory, WarpSmem<SPL>): one slot per
// (GPU g, start s) — slot = 8g + s — holding the instance that starts at s
// (profile, state, creation sequence) and, when a job is bound, that job's
// runtime state (remaining work, last update, timer time, migrations).
// Lane L owns slots L, L+32, ... (SPL = slots per lane), so the 8 slots of
// one GPU sit in 8 consecutive lanes.  A per-GPU word caches the busy
// compute / busy memory / blocked memory masks and the running-job count.
//
// Every timer of the reference's heap (sim.cpp:37-56) lives in a slot:
//   ST_RUN   -> Completion   (kind 0) at the latest prediction
//   ST_DRAIN -> MigrationEnd (kind 1) of the draining source replica
//   ST_WAIT  -> ServiceStart (kind 2)
// plus the next Arrival (kind 3) prefetched from HBM.  The next event is a
// warp-wide lexicographic argmin over (time, kind, job id, push seq) done
// with three REDUX.MIN steps — the same order TimerLater imposes, minus the
// stale completions the reference pops and ignores (sim.cpp:271-273).
//
// All placement / planner scoring is integer: the fragmentation cost of a
// post-placement mask pair is a rank (0..30) looked up in a 2 KiB table
// computed from the exact rational metric (frag.cpp:44-58); ranks are
// order-isomorphic to Frac comparisons, so packed u32 keys
// [pass|cost|!reused|gpu|start] reduce with a single REDUX.MIN.
//
// FP64 arithmetic uses the _rn intrinsics only (no contraction), replaying
// the reference's exact operation sequence.
#pragma once
#include "dev_types.h"
#include "warp_prims.cuh"

namespace msgk {

#ifdef MSG_SIM_PHASES
// Development build only: SM cycles of the event loop per phase, summed over
// warps — 0 timer scan + advance, 1 arrival, 2 service start, 3 departure
// (incl. planners and the dequeue pass), 4 timeline sample.
__device__ unsigned long long g_simph[8];
#endif

constexpr unsigned NONE = 0xFFFFFFFFu;
constexpr int MAX_JOB_BITS = 22;  // job ranks < 2^22 (inter key layout)

// EventKind (sim.hpp:20-28)
enum : uint8_t {
    EV_ARRIVAL = 0,
    EV_COMPLETION = 1,
    EV_MIGRATION_START = 2,
    EV_MIGRATION_END = 3,
    EV_RECONFIG = 4,
    EV_ENQUEUE = 5,
    EV_DEQUEUE = 6
};
enum : int32_t { STATUS_OK = 0, STATUS_JOBS_PENDING = 12 };

// ---- MIG geometry (profiles.cpp:8-15, 43-57) ------------------------------
MSG_DI unsigned cs_of(int p) { return (kCsPack >> (4 * p)) & 0xFu; }
MSG_DI unsigned ms_of(int p) { return (kMsPack >> (4 * p)) & 0xFu; }
MSG_DI unsigned startmask_of(int p) { return (unsigned)(kStartMask >> (8 * p)) & 0xFFu; }
MSG_DI unsigned stride_of(int p) { return (kStridePack >> (4 * p)) & 0xFu; }
MSG_DI unsigned count_of(int p) { return (kCountPack >> (4 * p)) & 0xFu; }
// slice_footprint: compute bits [s, s+cs), memory bits [s, s+ms).
MSG_DI unsigned fpc(int p, int s) { return ((1u << cs_of(p)) - 1u) << s; }
MSG_DI unsigned fpm(int p, int s) { return ((1u << ms_of(p)) - 1u) << s; }

// ---- per-GPU word: busy_c | busy_m<<8 | blocked_m<<16 | running<<24 --------
MSG_DI unsigned w_bc(unsigned w) { return w & 0x7Fu; }
MSG_DI unsigned w_bm(unsigned w) { return (w >> 8) & 0xFFu; }
MSG_DI unsigned w_km(unsigned w) { return (w >> 16) & 0xFFu; }
MSG_DI unsigned w_k(unsigned w) { return (w >> 24) & 0xFu; }

// Order-preserving u64 image of a double (-0 canonicalised to +0, which the
// reference's `a.time != b.time` also treats as equal).
MSG_DI uint64_t time_key(double t) {
    const uint64_t b = wp::dbits(wp::dadd(t, 0.0));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <int SPL>
struct alignas(16) WarpSmem {
    static constexpr int NS = 32 * SPL;  // slots
    static constexpr int NG = 4 * SPL;   // GPUs
    struct alignas(16) RT {
        double rem;    // RunJob::remaining_work (WAIT: service demand)
        double tkey;   // timer time of the slot
    };
    RT rt[NS];         // side by side: the timer scan reads both with one 16-byte load
    double gcost[NG];  // frag_cost(gpu) for the timeline (4-mask form)
    double tlp[NG + 2];  // timeline prefix sums: tlp[g] = ((c0 + c1) + ...) + c(g-1), reference order
    struct alignas(8) JM {
        int32_t job;    // bound job rank (RUN/WAIT) or migrating job (DRAIN)
        uint32_t mseq;  // MigrationEnd push sequence
    };
    JM jm[NS];
    uint32_t cseq[NS]; // instance creation order (vector order, gpu.cpp:88-111)
    uint32_t gw[NG];   // per-GPU mask word
    uint16_t mig[NS];  // migrations of the bound job
    uint8_t act[NS];   // the armed slots as a list: act[0 .. n_act) (SPL >= 2)
    uint8_t apos[NS];  // slot -> its index in act[] while armed
    uint8_t prof[NS];  // instance profile
    uint8_t st[NS];    // ST_*
    // zero-copy inputs (SimArgs::zc_*): this trace's caller arrays
    const double* zc_a;
    const double* zc_s;
    const int32_t* zc_p;
    // IO kernel: this trace's SoA host columns (SimArgs::rows_soa)
    double* rows_s;
    double* rows_d;
    uint64_t* rows_gm;
    // progressive row flushes (SimArgs::prog_host): rows published so far
    uint64_t* prog_h;
    uint32_t prog;
    uint32_t prog_epoch;
};


struct CreateRes {
    bool reused;
    unsigned dmask;  // destroyed slots (bit = start) on the GPU
    unsigned dprof;  // lane-local (lanes 0..7): profile of the slot before
    unsigned dseq;   // lane-local: creation sequence of the slot before
};

struct Decision {
    bool placed;
    bool reused;
    int g;
    int s;
    unsigned evals;
};

// Zero-copy inputs (SimArgs::zc_*), IO kernel only: jobs j0 .. j0+31 read
// from the caller's page-locked arrays when the trace's arrivals reach the
// block (three independent loads per lane: one PCIe round trip per 32
// arrivals) and published into the trace's device arrays, which every
// later read (arrival prefetch, queue heads, metrics) uses.  Out-of-range
// profiles and non-positive services are clamped only to keep the kernel
// in bounds: the host check (staging.h check_trace), run concurrently,
// rejects such a trace and its results are discarded.  (Staging the next
// block asynchronously with cp.async into shared memory was slower on the
// B200: profiles/r02, e2e_zc_r02p.log.)
// Blocks [0, kZcFirst), [kZcFirst, 32), then 32 jobs each: every trace asks
// for its first block at the same instant, so a small first block shortens
// that burst (4096 traces x 8 jobs x 20 B) and with it the traces' start.
#ifndef MSG_ZC_FIRST
#define MSG_ZC_FIRST 8
#endif
constexpr uint32_t kZcFirst = MSG_ZC_FIRST;
template <class WS>
MSG_DI void zc_fetch_block(WS* sm, double* arr, double* svc, uint8_t* prf, uint32_t j0, uint32_t N) {
    const unsigned L = wp::lane();
    const uint32_t j = j0 + L;
    const uint32_t len = j0 == 0 ? kZcFirst : (j0 == kZcFirst ? 32u - kZcFirst : 32u);
    if (j < N && L < len) {
        const double t = sm->zc_a[j];
        double v = sm->zc_s[j];
        int p = sm->zc_p[j];
        if ((unsigned)p >= (unsigned)kProfileCount) p = 0;
        if (!(v > 0.0)) v = 1.0;
        arr[j] = t;
        svc[j] = v;
        prf[j] = (uint8_t)p;
    }
    wp::sync();
}

// One job's record into the IO kernel's SoA host columns.
template <class WS>
MSG_DI void store_row_host(WS* sm, uint32_t j, const JobOut& jo) {
    sm->rows_s[j] = jo.sched;
    sm->rows_d[j] = jo.done;
    sm->rows_gm[j] = (uint64_t)(uint32_t)jo.gpu | ((uint64_t)(uint32_t)jo.mig << 32);
}

// Progressive rows (SimArgs::prog_host): extend the completed prefix (jobs
// whose record has its gpu set at completion) and, when it grew by a block
// or more, copy those records to the host, fence, then publish the count.
template <class WS>
MSG_DI void rows_flush_block(WS* sm, const JobOut* jobs, uint32_t N) {
    const unsigned L = wp::lane();
    wp::sync();
    const uint32_t p = sm->prog;
    uint32_t q = p;
    for (;;) {
        const uint32_t j = q + L;
        const unsigned nf = ~wp::ballot(j < N && jobs[j].gpu >= 0);
        const uint32_t adv = nf ? (uint32_t)(wp::ffs(nf) - 1) : 32u;
        q += adv;
        if (adv < 32u) break;
    }
    if (q - p < 32u) return;  // amortise the system-scope fence
    for (uint32_t j = p + L; j < q; j += 32) store_row_host(sm, j, jobs[j]);
    // The system-scope fence is this path's cost (~0.1 ms of the C2 IO
    // kernel; a lane-0 release store compiles to the same MEMBAR): hence a
    // flush every 64 arrivals (SimArgs::prog_mask), not every block.
    wp::gfence_sys();
    wp::sync();
    if (L == 0) {
        sm->prog = q;
        *(volatile uint64_t*)sm->prog_h = ((uint64_t)sm->prog_epoch << 32) | q;
    }
    wp::sync();
}

// IO: the pipelined msg_run_batch's host-I/O instantiation (summary / job
// rows only): zero-copy inputs and progressive row flushes (SimArgs::zc_*,
// prog_host).
// ND ("no delays"): every config of the launch has reconfiguration latency
// 0 and migration overlap 0 (SimArgs::no_delay; the reference defaults), so
// no slot is ever WaitingStart or Draining: every armed timer is a
// completion, and the latency / overlap branches fold away (C2 kernel
// 1.139 -> 1.017 ms, same results).

// SPL: slots per lane (ceil(8G/32)).  DETAIL: the kernel writes the event
// log / timeline records when requested; the summary-only instantiation has
// no emission code at all (smaller hot loop, fewer I-cache misses).
template <int SPL, bool DETAIL = true, bool IO = false, bool ND = false>
struct TraceSim {
    using WS = WarpSmem<SPL>;
    WS* sm;
    const DevTables* tb;
    const double* arr;
    const double* svc;
    const uint8_t* prf;
    const uint32_t* perm;
    int32_t* queue;
    JobOut* jobs;
    JobOut* jobs_h;  // SimArgs::jobs_host of this trace, or null
    EventRec* evs;
    double* tl;
    uint32_t N, ev_cap, tl_cap, oflags;
    uint32_t prog_mask;  // IO: progressive row flush cadence (SimArgs::prog_mask)
    // SimConfig
    int G;
    uint32_t cflags, lazymask;
    double alpha, overlap, latency;
    // warp-uniform engine state
    unsigned L;
    double now;
    uint32_t a_idx, a_rank;
    int a_prof;
    double a_t, a_svc;
    uint64_t a_key;  // time_key(a_t)
    uint32_t q_head, q_tail;
    uint32_t cseq_ctr, mseq_ctr;
    uint32_t n_ev, n_handler, n_tl;
    uint32_t n_mig, n_reconf, n_enq, n_deq;
    int max_arr, max_intra, max_inter;
    uint32_t n_plan_iter;
    // The armed (timer-carrying: Running, WaitingStart, Draining) slots as a
    // list in shared memory (act[0 .. n_act), apos: slot -> index), SPL >= 2
    // only: C2 averages 6.6 armed slots of 64 and exceeds 16 in 0.1% of
    // events, so the timer scan visits one list entry per lane instead of
    // SPL slots.
    static constexpr bool kAct = SPL >= 2;
    unsigned n_act;
    bool snap_mode;
    double tl_sum, tl_mean;
    unsigned tl_from;  // first GPU whose cost changed since the last timeline sum (G: none)
    // RunJob::last_update of EVERY running job equals the time of the last
    // handler: advance_all stamps all of them, start_service stamps `now`,
    // moves carry it (sim.cpp:153-165,212-218).  So dt is warp-uniform.
    double t_prev;
    double my_f;     // lanes 0..6: slowdown(L+1) = 1 + alpha*L
    double inv_g;    // 1/G when G is a power of two (then x/G == x*inv_g exactly)

    // ---------------------------------------------------------------- tables
    MSG_DI unsigned rank2(unsigned bc, unsigned bm) const {
        return tb->cost2rank[wp::popc(bc) * 256 + bm];
    }
    MSG_DI unsigned k2w(unsigned w) const { return tb->rank2k[rank2(w_bc(w), w_bm(w))]; }
    // frag_cost(gpu) (frag.cpp:60-65): 4-mask cost, busy drives ideal and
    // blocked drives feasibility; tabulated exactly on the host.
    MSG_DI double cost4w(unsigned w) const {
        const unsigned row = (unsigned)wp::popc(w_bc(w)) * 9u + (unsigned)wp::popc(w_bm(w));
        return tb->cost4val[tb->cost4pair[tb->idealid[row] * 32u + tb->feasid[w_km(w)]]];
    }

    // --------------------------------------------------------------- events
    MSG_DI void emit(uint8_t kind, int32_t job, unsigned gpu, unsigned gpu2, unsigned prof,
                     unsigned start, unsigned start2, unsigned flags, uint64_t aux) {
        if (DETAIL && (oflags & OF_EVENTS) && n_ev < ev_cap && L == 0) {
            EventRec r;
            r.t = now;
            r.aux = aux;
            r.job = job;
            r.gpu = (uint16_t)gpu;
            r.gpu2 = (uint16_t)gpu2;
            r.kind = kind;
            r.profile = (uint8_t)prof;
            r.start = (uint8_t)start;
            r.start2 = (uint8_t)start2;
            r.flags = (uint8_t)flags;
            r.pad[0] = r.pad[1] = r.pad[2] = 0;
            evs[n_ev] = r;
        }
        ++n_ev;
    }

    // ---------------------------------------------------------------- setup
    MSG_DI void setup(const SimArgs& a, const DevTables* tables, WS* ws, uint32_t t) {
        L = wp::lane();
        sm = ws;
        tb = tables;
        const DevTrace tr = a.traces[t];
        const DevConfig c = a.configs[tr.cfg];
        N = tr.n_jobs;
        arr = a.arrival + tr.job_off;
        svc = a.service + tr.job_off;
        prf = a.profile + tr.job_off;
        perm = tr.has_perm ? a.perm + tr.job_off : nullptr;
        oflags = a.out_flags;
        if (IO && a.zc_arrival) {  // zero-copy inputs: blocks fetched by load_arrival (zc_fetch_block)
            oflags |= OF_ZC;
            perm = nullptr;
            if (L == 0) {
                sm->zc_a = a.zc_arrival + tr.job_off;
                sm->zc_s = a.zc_service + tr.job_off;
                sm->zc_p = a.zc_profile + tr.job_off;
            }
        } else if (a.profile32) {  // direct inputs: the caller's int32 profiles, narrowed once per trace
            uint8_t* dst = const_cast<uint8_t*>(prf);
            const int32_t* src = a.profile32 + tr.job_off;
            for (uint32_t j = L; j < N; j += 32) dst[j] = (uint8_t)src[j];
            wp::sync();
        }
        queue = a.queue + tr.job_off;
        jobs = a.jobs + tr.job_off;
        jobs_h = a.jobs_host ? a.jobs_host + tr.job_off : nullptr;
        if (IO && jobs_h && L == 0) {
            double* base = reinterpret_cast<double*>(a.jobs_host);
            sm->rows_s = base + tr.job_off;
            sm->rows_d = base + a.rows_soa + tr.job_off;
            sm->rows_gm = reinterpret_cast<uint64_t*>(base + 2 * a.rows_soa) + tr.job_off;
        }
        if (IO && jobs_h && a.prog_host) {
            oflags |= OF_PROG;
            prog_mask = a.prog_mask | 31u;
            if (L == 0) {
                sm->prog_h = a.prog_host + t;
                sm->prog = 0;
                sm->prog_epoch = a.done_epoch;
            }
            for (uint32_t j = L; j < N; j += 32) jobs[j].gpu = -1;  // not completed (rows_flush)
        }
        evs = a.events ? a.events + tr.ev_off : nullptr;
        tl = a.timeline ? a.timeline + 2 * tr.tl_off : nullptr;
        ev_cap = tr.ev_cap;
        tl_cap = tr.tl_cap;
        if (!evs) oflags &= ~OF_EVENTS;
        if (!tl) oflags &= ~OF_TIMELINE;
        G = c.G;
        cflags = c.flags;
        lazymask = c.lazymask;
        alpha = c.alpha;
        overlap = ND ? 0.0 : c.overlap;
        latency = ND ? 0.0 : c.latency;
        init_factors();
        now = 0.0;
        a_idx = 0;
        q_head = q_tail = 0;
        mseq_ctr = 0;
        n_ev = n_handler = n_tl = 0;
        n_mig = n_reconf = n_enq = n_deq = 0;
        max_arr = max_intra = max_inter = 0;
        n_plan_iter = 0;
        snap_mode = false;
        tl_sum = 0.0;
        tl_mean = 0.0;
        tl_from = 0;
        n_act = 0;
#pragma unroll
        for (int i = 0; i < SPL; ++i) {
            const int slot = L + 32 * i;
            sm->st[slot] = ST_EMPTY;
            sm->mig[slot] = 0;
        }
        if (L < (unsigned)WS::NG) {
            sm->gw[L] = 0;
            sm->gcost[L] = 0.0;  // empty GPU: cost 0 (every ratio is 1)
        }
        wp::sync();
        // Static layout: pre-provisioned idle instances (sim.cpp:86-95).
        if (L == 0) {
            for (uint32_t k = 0; k < c.n_init; ++k) {
                const uint32_t v = a.init_slots[c.init_off + k];
                const int slot = (int)(v & 0xFFFFFFu);
                sm->st[slot] = ST_IDLE;
                sm->prof[slot] = (uint8_t)(v >> 24);
                sm->cseq[slot] = k;
            }
        }
        cseq_ctr = c.n_init;
        if (c.n_init) {
            for (int g = 0; g < G; ++g) refresh_gpu(g);
        }
        load_arrival();
        wp::sync();
    }

    // Decision-level mode (decide.cu): load one cluster snapshot instead of
    // a trace.  Busy instances load as ST_RUN (running vs waiting does not
    // matter to the scheduler or the planners), draining ones as ST_DRAIN.
    MSG_DI void setup_snapshot(const SnapArgs& a, const DevTables* tables, WS* ws, uint32_t i) {
        L = wp::lane();
        sm = ws;
        tb = tables;
        G = a.G;
        cflags = a.cflags;
        lazymask = a.lazymask;
        alpha = 0.0;
        overlap = a.overlap;
        latency = 0.0;
        init_factors();
        N = 0;
        a_idx = 0;
        now = 0.0;
        q_head = 0;
        q_tail = a.q_len ? a.q_len[i] : 0;
        queue = a.queue ? const_cast<int32_t*>(a.queue) + (size_t)i * a.q_cap : nullptr;
        prf = a.rank_profile ? a.rank_profile + (size_t)i * a.rank_cap : nullptr;
        svc = nullptr;
        arr = nullptr;
        perm = nullptr;
        jobs = a.scratch ? a.scratch + (size_t)i * a.rank_cap : nullptr;
        jobs_h = nullptr;
        evs = a.events + (size_t)i * a.ev_cap;
        ev_cap = a.ev_cap;
        tl = nullptr;
        tl_cap = 0;
        oflags = OF_EVENTS;
        mseq_ctr = 0;
        n_ev = n_handler = n_tl = 0;
        n_mig = n_reconf = n_enq = n_deq = 0;
        max_arr = max_intra = max_inter = 0;
        n_plan_iter = 0;
        snap_mode = true;
        tl_sum = tl_mean = 0.0;
        tl_from = 0;
        const size_t base = (size_t)i * (size_t)G * 8;
        unsigned maxseq = 0;
        bool any = false;
#pragma unroll
        for (int k = 0; k < SPL; ++k) {
            const int slot = L + 32 * k;
            if (slot < G * 8) {
                const uint32_t v = a.slot_in[base + slot];
                sm->st[slot] = (uint8_t)(v & 0xFu);
                sm->prof[slot] = (uint8_t)((v >> 4) & 0xFu);
                sm->cseq[slot] = v >> 8;
                sm->jm[slot].job = a.job_in[base + slot];
                sm->mig[slot] = 0;
                if ((v & 0xFu) != ST_EMPTY) {
                    maxseq = (v >> 8) > maxseq ? (v >> 8) : maxseq;
                    any = true;
                }
            } else {
                sm->st[slot] = ST_EMPTY;
            }
        }
        const unsigned mx = NONE - wp::rmin(NONE - maxseq);
        cseq_ctr = wp::ballot(any) ? mx + 1u : 0u;
        wp::sync();
        n_act = 0;
        if (kAct) {  // the snapshot's armed slots, in slot order
            const unsigned lt = (1u << L) - 1u;
#pragma unroll
            for (int k = 0; k < SPL; ++k) {
                const int slot = L + 32 * k;
                const bool armed = sm->st[slot] >= ST_RUN;
                const unsigned bl = wp::ballot(armed);
                const unsigned e = n_act + (unsigned)wp::popc(bl & lt);
                if (armed) {
                    sm->act[e] = (uint8_t)slot;
                    sm->apos[slot] = (uint8_t)e;
                }
                n_act += (unsigned)wp::popc(bl);
            }
            wp::sync();
        }
        for (int g = 0; g < G; ++g) refresh_gpu(g);
    }

    MSG_DI void store_snapshot(const SnapArgs& a, uint32_t i) {
        wp::sync();
        const size_t base = (size_t)i * (size_t)G * 8;
#pragma unroll
        for (int k = 0; k < SPL; ++k) {
            const int slot = L + 32 * k;
            if (slot < G * 8) {
                const uint8_t s = sm->st[slot];
                const bool busy = s == ST_RUN || s == ST_WAIT;
                a.slot_out[base + slot] = (uint32_t)(busy ? ST_RUN : s) | ((uint32_t)sm->prof[slot] << 4) |
                                          (sm->cseq[slot] << 8);
                a.job_out[base + slot] = busy ? sm->jm[slot].job : -1;
            }
        }
    }

    // Prefetch the next arrival timer (pushed in trace order, popped in
    // (time, job id) order: sim.cpp:118-120 with TimerLater).
    MSG_DI void load_arrival() {
        if (a_idx < N) {
            if (IO && (oflags & (OF_ZC | OF_PROG)) && ((a_idx & 31u) == 0 || a_idx == kZcFirst)) {
                if (oflags & OF_ZC)
                    zc_fetch_block(sm, const_cast<double*>(arr), const_cast<double*>(svc), const_cast<uint8_t*>(prf),
                                   a_idx, N);
                if ((oflags & OF_PROG) && a_idx && (a_idx & prog_mask) == 0) rows_flush_block(sm, jobs, N);
            }
            const uint32_t r = perm ? perm[a_idx] : a_idx;
            a_rank = r;
            a_t = arr[r];
            a_key = time_key(a_t);
            a_prof = prf[r];
            a_svc = svc[r];
        }
    }

    // ---------------------------------------------------------- GPU masks
    // Recompute GPU g's word from its 8 slots: busy/blocked masks
    // (gpu.cpp:10-48) and the running count running_on_ (sim.cpp:405).
    MSG_DI unsigned refresh_gpu(int g) {
        wp::sync();
        unsigned c = 0, r = 0;
        if (L < 8) {
            const int sl = g * 8 + (int)L;
            const uint8_t s = sm->st[sl];
            if (s >= ST_RUN) {
                const int p = sm->prof[sl];
                const unsigned m = fpm(p, (int)L);
                c = (s == ST_DRAIN) ? (m << 16) : (fpc(p, (int)L) | (m << 8) | (m << 16));
                r = (s == ST_RUN) ? 1u : 0u;
            }
        }
        const unsigned w = wp::ror(c) | (wp::radd(r) << 24);
        const double nc = cost4w(w), oc = sm->gcost[g];
        wp::sync();
        if (L == 0) {
            sm->gw[g] = w;
            sm->gcost[g] = nc;
        }
        // only a changed cost re-opens the timeline sum, from this GPU on
        if (wp::dbits(nc) != wp::dbits(oc) && (unsigned)g < tl_from) tl_from = (unsigned)g;
        wp::sync();
        return w;
    }

    // One instance's share of its GPU's word.  Instances on a GPU are pairwise
    // memory-disjoint (gpu.cpp:146-156) and compute bits lie inside memory
    // bits, so the word is the bitwise SUM of these shares and every
    // lifecycle transition updates it exactly by adding / subtracting them:
    // the same word refresh_gpu would rebuild from the 8 slots, without the
    // slot loads and the two warp reductions.
    MSG_DI unsigned share(unsigned st, int p, int s) const {
        if (st < ST_RUN) return 0u;
        const unsigned t = tb->share_run[p * 8 + s];  // Running: busy c/m, blocked m, one running job
        return st == ST_RUN ? t : (st == ST_WAIT ? t - (1u << 24) : (t & 0xFF0000u));
    }

    // Store GPU g's new word (warp-uniform) and its timeline cost, as
    // refresh_gpu does.
    MSG_DI unsigned set_gpu(int g, unsigned w) {
        const double nc = cost4w(w), oc = sm->gcost[g];
        wp::sync();
        if (L == 0) {
            sm->gw[g] = w;
            sm->gcost[g] = nc;
        }
        if (wp::dbits(nc) != wp::dbits(oc) && (unsigned)g < tl_from) tl_from = (unsigned)g;
        wp::sync();
        return w;
    }

    // ------------------------------------------------ armed-slot list
    MSG_DI void act_add(int slot) {
        if (!kAct) return;
        if (L == 0) {
            sm->act[n_act] = (uint8_t)slot;
            sm->apos[slot] = (uint8_t)n_act;
        }
        ++n_act;
    }
    // `slot` must be in the list: the last entry takes its place.
    MSG_DI void act_remove(int slot) {
        if (!kAct) return;
        --n_act;
        if (L == 0) {
            const unsigned p = sm->apos[slot], last = sm->act[n_act];
            sm->act[p] = (uint8_t)last;
            sm->apos[last] = (uint8_t)p;
        }
    }

    // ------------------------------------------------- contention model
    // slowdown(k) = 1 + alpha*(k-1) (sim.cpp:26-31): DMUL then DADD.
    MSG_DI double factor(unsigned k) const {
        return wp::dadd(1.0, wp::dmul(alpha, (double)((int)k - 1)));
    }

    MSG_DI void init_factors() {
        my_f = factor(L < 7 ? L + 1u : 1u);
        inv_g = ((G & (G - 1)) == 0) ? 1.0 / (double)G : 0.0;
        t_prev = 0.0;
    }

    // sample_timeline (sim.cpp:177-181): sequential sum in GPU order / G.
    // The running prefix sums are kept, so after a change on GPU g only the
    // tail g .. G-1 of the chain is re-added (same additions, same order).
    MSG_DI void sample() {
        if (tl_from < (unsigned)G) {
            wp::sync();
            double tot = tl_from ? sm->tlp[tl_from] : 0.0;
            for (int g = (int)tl_from; g < G; ++g) {
                tot = wp::dadd(tot, sm->gcost[g]);
                if (L == 0) sm->tlp[g + 1] = tot;
            }
            tl_mean = inv_g != 0.0 ? wp::dmul(tot, inv_g) : wp::ddiv(tot, (double)G);
            tl_from = (unsigned)G;
            wp::sync();
        }
        if (DETAIL && (oflags & OF_TIMELINE) && n_tl < tl_cap && L == 0) {
            tl[2 * n_tl] = now;
            tl[2 * n_tl + 1] = tl_mean;
        }
        ++n_tl;
        tl_sum = wp::dadd(tl_sum, tl_mean);
    }

    // -------------------------------------------------------------- events
    // reschedule_completions (sim.cpp:167-175) fused with the next timer pop
    // (Engine::execute, sim.cpp:123-141) and with the popped handler's
    // advance_all (sim.cpp:153-165, the first step of every handler): one
    // pass over the slots recomputes every Running slot's prediction
    // now + max(rem,0)*f and forms the (time, kind, job, push seq) keys of
    // all armed timers; once the warp-wide argmin fixes the new `now`, the
    // same registers give rem -= dt / slowdown(k), and each Running slot's
    // (rem, prediction) pair is stored with one 16-byte store.  The <= 7
    // distinct quotients dt / slowdown(k) are computed once (lane k-1) and
    // fetched by shuffle; dt is warp-uniform (see t_prev).  Returns -1 none,
    // 0 completion, 1 migration end, 2 service start, 3 arrival.
    MSG_DI int resched_next(int& ev_slot) {
        wp::sync();
        unsigned bhi = NONE, blo = NONE, btie = NONE, bms = NONE;
        int bsl = -1;
        double bt = 0.0;
        // With SPL >= 2 the scan visits the armed-slot list (act), one
        // entry per lane while n_act <= 32.
        constexpr bool kCompact = kAct;
        const unsigned na = n_act;
        // every load before the first store (the stores could alias them)
        uint8_t sv[SPL];
        int slv[SPL];
        unsigned kv[SPL], jv[SPL], mv[SPL];
        double rv[SPL], tv[SPL], pv[SPL];
#pragma unroll
        for (int i = 0; i < SPL; ++i) {
            sv[i] = ST_EMPTY;
            slv[i] = 0;
            kv[i] = 1u;
            if (kCompact && i > 0 && na <= 32u * (unsigned)i) continue;
            int slot;
            bool valid = true;
            if (kCompact) {
                valid = L + 32u * (unsigned)i < na;
                slot = valid ? (int)sm->act[L + 32 * i] : 0;
                const uint8_t x = sm->st[slot];
                sv[i] = valid ? x : (uint8_t)ST_EMPTY;
            } else {
                slot = L + 32 * i;
                sv[i] = sm->st[slot];
            }
            slv[i] = slot;
            kv[i] = sv[i] == ST_RUN ? w_k(sm->gw[slot >> 3]) : 1u;
            // a lane past the list reads nothing of slot 0's timer (another
            // lane may own and rewrite it below)
            rv[i] = tv[i] = 0.0;
            jv[i] = mv[i] = 0u;
            if (valid) {
                const typename WS::RT x = sm->rt[slot];
                rv[i] = x.rem;
                tv[i] = x.tkey;
                const typename WS::JM y = sm->jm[slot];
                jv[i] = (unsigned)y.job;
                mv[i] = y.mseq;
            }
        }
#pragma unroll
        for (int i = 0; i < SPL; ++i) {
            if (kCompact && i > 0 && na <= 32u * (unsigned)i) continue;
            // branch-free: every entry forms its key, unarmed ones an all-NONE
            // key that never wins
            const int slot = slv[i];
            const uint8_t s = sv[i];
            // (ND: only Running slots carry timers)
            const bool armed = s >= ST_RUN, run = ND ? armed : s == ST_RUN, drain = !ND && s == ST_DRAIN;
            const double f = wp::shfl(my_f, (int)kv[i] - 1);
            const double r = rv[i] < 0.0 ? 0.0 : rv[i];  // std::max(rem, 0.0)
            const double tp = wp::dadd(now, wp::dmul(r, f));
            pv[i] = tp;
            const double t = run ? tp : tv[i];
            const uint64_t tk = time_key(t);
            const unsigned hi = armed ? (unsigned)(tk >> 32) : NONE, lo = armed ? (unsigned)tk : NONE;
            const unsigned kind = run ? 0u : (drain ? 1u : 2u);
            const unsigned tie = armed ? ((kind << 28) | jv[i]) : NONE;
            const unsigned ms = armed ? (drain ? mv[i] : 0u) : NONE;
            const uint64_t ka = ((uint64_t)hi << 32) | lo, kb = ((uint64_t)tie << 32) | ms;
            const uint64_t ba = ((uint64_t)bhi << 32) | blo, bb = ((uint64_t)btie << 32) | bms;
            // the first entry needs no compare (an unarmed one carries the all-NONE key)
            const bool better = i == 0 || ka < ba || (ka == ba && kb < bb);
            bhi = better ? hi : bhi;
            blo = better ? lo : blo;
            btie = better ? tie : btie;
            bms = better ? ms : bms;
            bsl = better ? slot : bsl;
            bt = better ? t : bt;
        }
        const unsigned mhi = wp::rmin(bhi);
        const bool have_arrival = a_idx < N;
        int kind = 3;
        if (mhi == NONE) {
            if (!have_arrival) return -1;  // the run is over: predictions are no longer needed
            now = a_t;
        } else {
            const unsigned mlo = wp::rmin(bhi == mhi ? blo : NONE);
            const unsigned mtie = wp::rmin((bhi == mhi && blo == mlo) ? btie : NONE);
            bool match = bhi == mhi && blo == mlo && btie == mtie;
            if (!ND && (mtie >> 28) == 1u) {  // same job, same time MigrationEnds: push order
                const unsigned mms = wp::rmin(match ? bms : NONE);
                match = match && bms == mms;
            }
            if (have_arrival && time_key(a_t) < (((uint64_t)mhi << 32) | mlo)) {  // arrivals rank last on equal time
                now = a_t;
            } else {
                const int wl = wp::ffs(wp::ballot(match)) - 1;
                ev_slot = wp::shfl(bsl, wl);
                now = wp::shfl(bt, wl);
                kind = (int)(mtie >> 28);
            }
        }
        // advance_all of the popped handler: dt <= 0 leaves rem unchanged
        const double dt = wp::dsub(now, t_prev);
        t_prev = now;
        const bool adv = dt > 0.0;
        double q = 0.0;
        if (adv) q = wp::ddiv(dt, my_f);
#pragma unroll
        for (int i = 0; i < SPL; ++i) {
            if (kCompact && i > 0 && na <= 32u * (unsigned)i) continue;
            const double qk = wp::shfl(q, (int)kv[i] - 1);
            if (sv[i] == ST_RUN) {
                typename WS::RT x;
                x.rem = adv ? wp::dsub(rv[i], qk) : rv[i];
                x.tkey = pv[i];
                sm->rt[slv[i]] = x;
            }
        }
        return kind;
    }

    // ------------------------------------------------------------ schedule
    // schedule() (scheduler.cpp:47-81) / first_fit_schedule() (:83-98) /
    // dispatch_schedule() (:100-104) on the warp's cluster.
    MSG_DI Decision dispatch(int p) {
        wp::sync();
        Decision d;
        const unsigned smask = startmask_of(p);
        const bool dyn = (cflags & CF_DYN) != 0;
        if (cflags & CF_LB) {
            unsigned kmin = NONE, nl = 0, nb = 0;
#pragma unroll
            for (int i = 0; i < SPL; ++i) {
                // branch-free: every slot scores, non-candidates (illegal
                // start, unavailable, beyond G) drop out of the min and counts
                const int slot = L + 32 * i;
                const int g = slot >> 3, s = slot & 7;
                const unsigned w = sm->gw[g];
                const bool exact = sm->st[slot] == ST_IDLE && sm->prof[slot] == p;
                const unsigned fm = fpm(p, s);
                const bool cand = g < G && ((smask >> s) & 1u) && (dyn || exact) &&
                                  !(fm & w_km(w));  // candidate_starts + avail
                const unsigned rk = rank2((w_bc(w) | fpc(p, s)) & 0x7Fu, (w_bm(w) | fm) & 0xFFu);
                const unsigned lazy = (lazymask >> wp::popc(w_bc(w))) & 1u;
                const unsigned key = ((lazy ^ 1u) << 31) | (rk << 26) | ((exact ? 0u : 1u) << 25) |
                                     ((unsigned)g << 3) | (unsigned)s;
                kmin = cand && key < kmin ? key : kmin;
                nl += cand ? lazy : 0u;
                nb += cand ? (lazy ^ 1u) : 0u;
            }
            const unsigned k = wp::rmin(kmin);
            const unsigned cnt = wp::radd(nl | (nb << 16));  // <= 8 candidates per lane
            const unsigned NL = cnt & 0xFFFFu, NB = cnt >> 16;
            d.evals = NL + (NL == 0 ? NB : 0u);  // Busy pass only if Lazy found nothing
            d.placed = k != NONE;
            d.g = (int)((k >> 3) & 0x3FFFFFu);
            d.s = (int)(k & 7u);
            d.reused = ((k >> 25) & 1u) == 0;
        } else {
            unsigned kmin = NONE;
#pragma unroll
            for (int i = 0; i < SPL; ++i) {
                const int slot = L + 32 * i;
                const int g = slot >> 3, s = slot & 7;
                if (g < G && ((smask >> s) & 1u)) {
                    const unsigned w = sm->gw[g];
                    const bool exact = sm->st[slot] == ST_IDLE && sm->prof[slot] == p;
                    if ((dyn || exact) && !(fpm(p, s) & w_km(w))) {
                        const unsigned key = ((unsigned)g << 3) | (unsigned)s;
                        kmin = key < kmin ? key : kmin;
                    }
                }
            }
            const unsigned k = wp::rmin(kmin);
            d.evals = 0;  // first_fit_schedule reports no evaluations
            d.placed = k != NONE;
            d.g = (int)(k >> 3);
            d.s = (int)(k & 7u);
            d.reused = false;
            if (d.placed) {
                const int slot = (int)k;
                d.reused = sm->st[slot] == ST_IDLE && sm->prof[slot] == p;
            }
        }
        return d;
    }

    // ------------------------------------------------------ create_instance
    // gpu.cpp:71-101: reuse an exact idle instance (0 ops) or destroy every
    // idle instance overlapping the footprint (creation order) and create.
    // Leaves the destination slot ST_RUN as a placeholder; the caller binds
    // the job state.
    MSG_DI CreateRes create(int g, int p, int s) {
        wp::sync();
        CreateRes cr;
        const int sl = g * 8 + (int)(L & 7u);
        const uint8_t mst = L < 8 ? sm->st[sl] : ST_EMPTY;
        const unsigned mpr = L < 8 ? sm->prof[sl] : 0u;
        const unsigned mseq = L < 8 ? sm->cseq[sl] : 0u;
        cr.reused = wp::ballot(L == (unsigned)s && mst == ST_IDLE && mpr == (unsigned)p) != 0;
        cr.dprof = mpr;
        cr.dseq = mseq;
        cr.dmask = 0;
        if (!cr.reused) {
            const bool d = L < 8 && mst == ST_IDLE && (fpm((int)mpr, (int)L) & fpm(p, s)) != 0;
            cr.dmask = wp::ballot(d);
            if (d) sm->st[sl] = ST_EMPTY;
        }
        wp::sync();
        if (L == 0) {
            const int dst = g * 8 + s;
            sm->st[dst] = ST_RUN;
            if (!cr.reused) {
                sm->prof[dst] = (uint8_t)p;
                sm->cseq[dst] = cseq_ctr;
            }
        }
        if (!cr.reused) ++cseq_ctr;
        wp::sync();
        return cr;
    }

    // Reconfig events of one create_instance: destroys in instance-vector
    // (creation) order, then the create (gpu.cpp:88-98, sim.cpp:183-195).
    MSG_DI void emit_reconfig(int g, int p, int s, const CreateRes& cr) {
        if (!DETAIL || !(oflags & OF_EVENTS)) {  // no records: only the count (destroy order is irrelevant)
            const uint32_t n = (uint32_t)wp::popc(cr.dmask) + (cr.reused ? 0u : 1u);
            n_reconf += n;
            n_ev += n;  // emit() counts every event, stored or not
            return;
        }
        unsigned m = cr.dmask;
        while (m) {
            int lw;
            if ((m & (m - 1u)) == 0) {
                lw = wp::ffs(m) - 1;
            } else {
                const unsigned c = (L < 8 && ((m >> L) & 1u)) ? cr.dseq : NONE;
                const unsigned mn = wp::rmin(c);
                lw = wp::ffs(wp::ballot(c == mn && c != NONE)) - 1;
            }
            const int pr = wp::shfl((int)cr.dprof, lw);
            emit(EV_RECONFIG, -1, (unsigned)g, 0, (unsigned)pr, (unsigned)lw, 0, EF_DESTROY, 0);
            ++n_reconf;
            m &= ~(1u << lw);
        }
        if (!cr.reused) {
            emit(EV_RECONFIG, -1, (unsigned)g, 0, (unsigned)p, (unsigned)s, 0, 0, 0);
            ++n_reconf;
        }
    }

    // apply_placement + start_service (sim.cpp:199-218).
    MSG_DI double apply_placement(int g, int p, int s, int32_t r, double sv, unsigned nops) {
        const double delay = wp::dmul((double)nops, latency);
        const double ss = wp::dadd(now, delay);
        const int slot = g * 8 + s;
        // the destination held no instance or an idle one, and create only
        // destroys idle ones: the GPU gains exactly the new instance's share
        const unsigned w = sm->gw[g] + share(delay > 0.0 ? ST_WAIT : ST_RUN, p, s);
        act_add(slot);
        if (L == 0) {
            sm->jm[slot].job = r;
            sm->mig[slot] = 0;
            sm->rt[slot].rem = sv;
            sm->st[slot] = delay > 0.0 ? ST_WAIT : ST_RUN;  // WAIT: ServiceStart timer at ss
            sm->rt[slot].tkey = ss;
            jobs[r].sched = ss;
        }
        set_gpu(g, w);
        return ss;
    }

    // Place job r (profile p) per decision d; emits the placement event
    // (Arrival or Dequeue) followed by its reconfig ops.
    MSG_DI void place(const Decision& d, int32_t r, int p, double sv, uint8_t kind) {
        const CreateRes cr = create(d.g, p, d.s);
        const unsigned nops = (unsigned)wp::popc(cr.dmask) + (cr.reused ? 0u : 1u);
        const double ss = apply_placement(d.g, p, d.s, r, sv, nops);
        emit(kind, r, (unsigned)d.g, 0, (unsigned)p, (unsigned)d.s, 0, EF_PLACED | (cr.reused ? EF_REUSED : 0),
             snap_mode ? (uint64_t)d.evals : wp::dbits(ss));
        emit_reconfig(d.g, p, d.s, cr);
    }

    // dequeue_pass / try_dequeue: strict FCFS, stop at the first head that
    // cannot be placed (sim.cpp:325-344, scheduler.cpp:106-121).
    MSG_DI void dequeue_pass() {
        while (q_head < q_tail) {
            wp::sync();
            const int32_t h = queue[q_head];
            const int p = prf[h];
            const double sv = svc ? svc[h] : 0.0;
            const Decision d = dispatch(p);
            if (!d.placed) break;
            max_arr = max_arr > (int)d.evals ? max_arr : (int)d.evals;
            ++q_head;
            place(d, h, p, sv, EV_DEQUEUE);
            ++n_deq;
        }
    }

    // ----------------------------------------------------------- migration
    // apply_move (migration.cpp:35-69) + record_plan bookkeeping
    // (sim.cpp:346-396): replica-first move of the job in from_slot to
    // (tg, ts); costs are the end-state (busy-mask) costs before/after.
    MSG_DI void apply_move(int from_slot, int tg, int ts, bool inter) {
        wp::sync();
        const int fg = from_slot >> 3, fs = from_slot & 7;
        const int q = sm->prof[from_slot];
        const int32_t r = sm->jm[from_slot].job;
        const uint8_t jst = sm->st[from_slot];
        const double jrem = sm->rt[from_slot].rem, jtk = sm->rt[from_slot].tkey;
        const unsigned jmig = sm->mig[from_slot];
        const unsigned wf = sm->gw[fg], wt = sm->gw[tg];
        const unsigned fcb = k2w(wf);
        const unsigned tcb = k2w(wt);
        // source: the job's share leaves, a draining replica's (blocked
        // memory only) stays while overlap > 0; destination: the job's share
        const unsigned sh_to = share(jst, q, ts);
        unsigned nwf = wf - share(jst, q, fs) + (overlap > 0.0 ? share(ST_DRAIN, q, fs) : 0u);
        if (tg == fg) nwf += sh_to;
        wp::sync();
        if (L == 0) sm->st[from_slot] = ST_DRAIN;  // start_draining
        const CreateRes cr = create(tg, q, ts);
        if (L == 0) {
            const int dst = tg * 8 + ts;
            sm->st[dst] = jst;
            sm->jm[dst].job = r;
            sm->mig[dst] = (uint16_t)(jmig + 1u);
            sm->rt[dst].rem = jrem;
            sm->rt[dst].tkey = jtk;
            if (overlap <= 0.0) {
                sm->st[from_slot] = ST_IDLE;  // finish_draining at once
            } else {
                sm->rt[from_slot].tkey = wp::dadd(now, overlap);
                sm->jm[from_slot].mseq = mseq_ctr;
            }
        }
        if (overlap > 0.0) ++mseq_ctr;
        act_add(tg * 8 + ts);
        if (overlap <= 0.0) act_remove(from_slot);
        set_gpu(fg, nwf);
        const unsigned nwt = tg != fg ? set_gpu(tg, wt + sh_to) : nwf;
        const uint64_t costs = (uint64_t)fcb | ((uint64_t)k2w(nwf) << 16) | ((uint64_t)tcb << 32) |
                               ((uint64_t)k2w(nwt) << 48);
        emit(EV_MIGRATION_START, r, (unsigned)fg, (unsigned)tg, (unsigned)q, (unsigned)fs, (unsigned)ts,
             inter ? EF_INTER : 0, costs);
        ++n_mig;
        emit_reconfig(tg, q, ts, cr);
        if (overlap <= 0.0) emit(EV_MIGRATION_END, r, (unsigned)fg, 0, 0, 0, 0, 0, 0);
    }

    // plan_intra (migration.cpp:71-123): greedy, strictly improving moves of
    // one busy job to another legal start on the same GPU; key
    // (cost, job id, start).
    MSG_DI void plan_intra(int g) {
        for (;;) {
            wp::sync();
            const unsigned w = sm->gw[g];
            const unsigned bc = w_bc(w), bm = w_bm(w), km = w_km(w);
            const unsigned cur = rank2(bc, bm);
            const int own = (int)(L & 7u);
            const int sl = g * 8 + own;
            const uint8_t s = sm->st[sl];
            unsigned kmin = NONE, cnt = 0;
            if (s == ST_RUN || s == ST_WAIT) {
                const int q = sm->prof[sl];
                const unsigned r = (unsigned)sm->jm[sl].job;
                const unsigned ofc = fpc(q, own), ofm = fpm(q, own);
                const unsigned n = count_of(q), stride = stride_of(q);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const unsigned j = (L >> 3) + 4u * (unsigned)h;
                    if (j < n) {
                        const int t = (int)(j * stride);
                        if (t != own && !(fpm(q, t) & km)) {
                            const unsigned rk = rank2((bc & ~ofc) | fpc(q, t), (bm & ~ofm) | fpm(q, t));
                            const unsigned key = (rk << 27) | (r << 3) | (unsigned)t;
                            kmin = key < kmin ? key : kmin;
                            ++cnt;
                        }
                    }
                }
            }
            const unsigned best = wp::rmin(kmin);
            const int evals = (int)wp::radd(cnt);
            max_intra = max_intra > evals ? max_intra : evals;
            ++n_plan_iter;
            if (best == NONE || (best >> 27) >= cur) break;  // strict improvement only
            const int wl = wp::ffs(wp::ballot(kmin == best)) - 1;
            apply_move(g * 8 + (wl & 7), g, (int)(best & 7u), false);
        }
    }

    // plan_inter (migration.cpp:125-210): move jobs from Busy GPUs to the
    // Lazy GPU g0 while the move leaves g0 less loaded than the source;
    // source key (cost without the job, gpu, job id), destination key
    // (cost with the job, start).  Lazy-ness of g0 is not re-checked.
    MSG_DI void plan_inter(int g0) {
        for (;;) {
            wp::sync();
            const unsigned w0 = sm->gw[g0];
            const unsigned lazy_cs = (unsigned)wp::popc(w_bc(w0));
            const unsigned km0 = w_km(w0);
            const unsigned pl = tb->placeable[km0];
            unsigned kmin = NONE, cnt = 0;
            int bsl = -1;
            const unsigned na = n_act;
#pragma unroll
            for (int i = 0; i < SPL; ++i) {
                // sources are busy slots: with the armed-slot list, one entry per lane
                if (kAct && i > 0 && na <= 32u * (unsigned)i) continue;
                const bool in = !kAct || L + 32u * (unsigned)i < na;
                const int slot = kAct ? (in ? (int)sm->act[L + 32 * i] : 0) : L + 32 * i;
                const int g = slot >> 3, s = slot & 7;
                if (in && g < G && g != g0) {
                    const uint8_t st = sm->st[slot];
                    if (st == ST_RUN || st == ST_WAIT) {
                        const unsigned w = sm->gw[g];
                        const unsigned src_cs = (unsigned)wp::popc(w_bc(w));
                        const int q = sm->prof[slot];
                        const unsigned cs = cs_of(q);
                        if (!((lazymask >> src_cs) & 1u) && lazy_cs + cs < src_cs - cs && ((pl >> q) & 1u)) {
                            const unsigned rk = rank2(w_bc(w) & ~fpc(q, s), w_bm(w) & ~fpm(q, s));
                            const unsigned key = (rk << 27) | ((unsigned)g << 22) | (unsigned)sm->jm[slot].job;
                            if (key < kmin) {
                                kmin = key;
                                bsl = slot;
                            }
                            ++cnt;
                        }
                    }
                }
            }
            const unsigned best = wp::rmin(kmin);
            int evals = (int)wp::radd(cnt);
            ++n_plan_iter;
            if (best == NONE) {
                max_inter = max_inter > evals ? max_inter : evals;
                break;
            }
            const int wl = wp::ffs(wp::ballot(kmin == best)) - 1;
            const int from_slot = wp::shfl(bsl, wl);
            const int q = sm->prof[from_slot];
            // Destination: minimum (cost, start) on g0; lane L < 8 = start L.
            const bool cand = L < 8 && ((startmask_of(q) >> L) & 1u) && !(fpm(q, (int)L) & km0);
            const unsigned dk = cand ? ((rank2(w_bc(w0) | fpc(q, (int)L), w_bm(w0) | fpm(q, (int)L)) << 3) | L)
                                     : NONE;
            const unsigned dbest = wp::rmin(dk);
            evals += (int)wp::radd(cand ? 1u : 0u);
            max_inter = max_inter > evals ? max_inter : evals;
            apply_move(from_slot, g0, (int)(dbest & 7u), true);
        }
    }

    // on_departure (migration.cpp:212-220): Busy -> intra, Lazy -> inter.
    MSG_DI void on_departure(int g) {
        wp::sync();
        const unsigned w = sm->gw[g];
        if ((lazymask >> wp::popc(w_bc(w))) & 1u) plan_inter(g);
        else plan_intra(g);
    }

    // ------------------------------------------------------------ handlers
    // Handler bodies (sim.cpp:220-323), laid out so the steps every handler
    // shares (advance_all first, reschedule + sample last, the dequeue pass)
    // exist once in the instruction stream:
    //   Arrival:      advance; place or enqueue;                       reschedule; sample
    //   Completion:   advance; release; log; sample; dequeue; [plan; dequeue]; reschedule; sample
    //   MigrationEnd: advance; finish draining; log; dequeue;          reschedule; sample
    //   ServiceStart: advance; start service;                          reschedule; sample
    MSG_DI void handle_arrival() {  // sim.cpp:220-267
        const int32_t r = (int32_t)a_rank;
        const int p = a_prof;
        const double sv = a_svc;
        ++a_idx;
        load_arrival();
        bool enq = q_head < q_tail;  // never overtake a non-empty queue
        if (!enq) {
            const Decision d = dispatch(p);
            max_arr = max_arr > (int)d.evals ? max_arr : (int)d.evals;
            if (d.placed) place(d, r, p, sv, EV_ARRIVAL);
            else enq = true;
        }
        if (enq) {
            emit(EV_ARRIVAL, r, 0, 0, (unsigned)p, 0, 0, 0, 0);
            if (L == 0) queue[q_tail] = r;
            ++q_tail;
            emit(EV_ENQUEUE, r, 0, 0, 0, 0, 0, 0, 0);
            ++n_enq;
        }
    }

    // Completion (sim.cpp:269-301) and MigrationEnd (sim.cpp:303-315).
    MSG_DI void handle_departure(int slot, bool completion) {
        wp::sync();
        const int g = slot >> 3;
        const int32_t r = sm->jm[slot].job;
        const int m = sm->mig[slot];
        const unsigned w = sm->gw[g] - share(sm->st[slot], sm->prof[slot], slot & 7);
        act_remove(slot);
        wp::sync();
        if (L == 0) {
            sm->st[slot] = ST_IDLE;  // release_job / finish_draining: the instance stays, idle
            if (completion) {
                jobs[r].done = now;
                jobs[r].gpu = g;
                jobs[r].mig = m;
            }
        }
        set_gpu(g, w);
        emit(completion ? EV_COMPLETION : EV_MIGRATION_END, r, (unsigned)g, 0, 0, 0, 0, 0, 0);
        if (completion) sample();  // post-departure level
        const int passes = (completion && (cflags & CF_MIG)) ? 2 : 1;
        for (int pass = 0; pass < passes; ++pass) {
            if (pass) on_departure(g);
            dequeue_pass();
        }
    }

    MSG_DI void handle_service_start(int slot) {  // sim.cpp:317-323
        wp::sync();
        const unsigned w = sm->gw[slot >> 3] + (1u << 24);  // WaitingStart -> Running: one more running job
        if (L == 0) {
            sm->st[slot] = ST_RUN;  // start_service: rem already holds service_s
        }
        set_gpu(slot >> 3, w);
    }

    MSG_DI void run() {  // Engine::execute (sim.cpp:123-141)
#ifdef MSG_SIM_PHASES
        unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        long long c0 = clock64();
#define MSG_SIM_PH(k) do { const long long c1 = clock64(); ph[k] += (unsigned long long)(c1 - c0); c0 = c1; } while (0)
#else
#define MSG_SIM_PH(k) ((void)0)
#endif
        for (;;) {
            int slot = -1;
            // reschedules the previous handler's completions, pops the next
            // timer and advances every running job to it
            const int kind = resched_next(slot);
            MSG_SIM_PH(0);
            if (kind < 0) break;
            ++n_handler;
            if (kind == 3) {
                handle_arrival();
                MSG_SIM_PH(1);
            } else if (kind == 2) {
                handle_service_start(slot);
                MSG_SIM_PH(2);
            } else {
                handle_departure(slot, kind == 0);
                MSG_SIM_PH(3);
            }
            sample();
            MSG_SIM_PH(4);
        }
#ifdef MSG_SIM_PHASES
        if (L == 0)
            for (int k = 0; k < 5; ++k) atomicAdd(&g_simph[k], ph[k]);
#endif
#undef MSG_SIM_PH
    }

    // metrics (sim.cpp:414-502): sums in job-id order, then divide.
    MSG_DI void finish(DevSummary* out, DevSummary* out_host = nullptr) {
        wp::sync();
        DevSummary s;
        s.status = q_head < q_tail ? STATUS_JOBS_PENDING : STATUS_OK;
        s.reserved = 0;
        s.pending_rank = -1;
        double sw = 0.0, se = 0.0, st = 0.0, first = 0.0, lastc = 0.0;
        if (s.status == STATUS_OK) {
            const uint32_t pub = (IO && (oflags & OF_PROG)) ? sm->prog : 0u;  // rows already on the host
            double fa = 0.0, lc = 0.0;      // min arrival / max completion so far (this lane's jobs)
            unsigned fj = NONE, lj = NONE;  // ... and the first job holding it
            for (uint32_t base = 0; base < N; base += 32) {
                const uint32_t j = base + L;
                double w = 0.0, e = 0.0, t = 0.0, a = 0.0, d = 0.0;
                if (j < N) {
                    a = arr[j];
                    const JobOut jo = jobs[j];
                    if (IO && jobs_h && j >= pub)
                        store_row_host(sm, j, jo);  // SoA: three coalesced 256-byte stores per warp
                    else if (!IO && jobs_h)
                        jobs_h[j] = jo;  // coalesced: a warp stores 32 consecutive records
                    const double sc = jo.sched;
                    d = jo.done;
                    w = wp::dsub(sc, a);
                    e = wp::dsub(d, sc);
                    t = wp::dadd(w, e);
                }
                if (j < N) {  // lane-local: jobs j ascend, so a strict compare keeps the earliest on ties
                    if (fj == NONE || a < fa) fa = a, fj = j;
                    if (lj == NONE || lc < d) lc = d, lj = j;
                }
                const uint32_t n = N - base < 32 ? N - base : 32;
                for (uint32_t k = 0; k < n; ++k) {  // the sums: sequential, in job-id order
                    const double wk = wp::shfl(w, (int)k), ek = wp::shfl(e, (int)k), tk = wp::shfl(t, (int)k);
                    sw = wp::dadd(sw, wk);
                    se = wp::dadd(se, ek);
                    st = wp::dadd(st, tk);
                }
            }
            // std::min(first, a) / std::max(last, c) over job-id order keep the
            // earliest job among equal values: a (value, job) tree with that rule
            for (int off = 16; off > 0; off >>= 1) {
                const int src = (int)(L ^ (unsigned)off);
                const double oa = wp::shfl(fa, src), oc = wp::shfl(lc, src);
                const unsigned oj = wp::shfl(fj, src), ol = wp::shfl(lj, src);
                if (oj != NONE && (fj == NONE || oa < fa || (!(fa < oa) && oj < fj))) fa = oa, fj = oj;
                if (ol != NONE && (lj == NONE || lc < oc || (!(oc < lc) && ol < lj))) lc = oc, lj = ol;
            }
            first = fa;
            lastc = lc;
        } else {
            unsigned mn = NONE;
            for (uint32_t i = q_head + L; i < q_tail; i += 32) {
                const unsigned r = (unsigned)queue[i];
                mn = r < mn ? r : mn;
            }
            s.pending_rank = (int32_t)wp::rmin(mn);
        }
        if (N > 0 && s.status == STATUS_OK) {
            const double n = (double)N;
            s.mean_wait = wp::ddiv(sw, n);
            s.mean_exec = wp::ddiv(se, n);
            s.mean_turn = wp::ddiv(st, n);
            s.makespan = wp::dsub(lastc, first);
        } else {
            s.mean_wait = s.mean_exec = s.mean_turn = s.makespan = 0.0;
        }
        s.handler_events = n_handler;
        s.n_events = n_ev;
        s.timeline_samples = n_tl;
        s.migrations = n_mig;
        s.reconfig_ops = n_reconf;
        s.enqueues = n_enq;
        s.dequeues = n_deq;
        s.max_arr = max_arr;
        s.max_intra = max_intra;
        s.max_inter = max_inter;
        s.tl_sum = tl_sum;
        if (L == 0) {
            *out = s;
            if (out_host) *out_host = s;
        }
    }
};

// One warp, one trace: the body shared by the CUDA kernel and the CPU-side
// unit-test emulation.
template <int SPL, bool DETAIL = true, bool IO = false, bool ND = false>
MSG_DI void simulate_trace(const SimArgs& a, const DevTables* tables, WarpSmem<SPL>* ws, uint32_t t) {
    TraceSim<SPL, DETAIL, IO, ND> sim;
    sim.setup(a, tables, ws, t);
    sim.run();
    sim.finish(a.summary + t, a.summary_host ? a.summary_host + t : nullptr);
    if (a.done_host) {  // publish: every lane's host stores, then the trace's flag
        wp::gfence_sys();
        wp::sync();
        if (wp::lane() == 0) *(volatile uint32_t*)(a.done_host + t) = a.done_epoch;
    }
}

// One decision-level operation on one cluster snapshot (decide.cu): the
// body shared by the CUDA kernel and the CPU-side unit-test emulation.
template <int SPL>
MSG_DI void snapshot_op(const SnapArgs& a, const DevTables* tb, WarpSmem<SPL>* ws, uint32_t i) {
    TraceSim<SPL> sim;
    sim.setup_snapshot(a, tb, ws, i);
    int32_t out[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int arg = a.arg ? a.arg[i] : 0;
    if (a.op <= SOP_DISPATCH) {
        if (a.op == SOP_SCHEDULE) sim.cflags |= CF_LB;
        if (a.op == SOP_FIRST_FIT) sim.cflags &= ~CF_LB;
        const Decision d = sim.dispatch(arg);
        out[0] = d.placed;
        out[1] = d.placed ? d.g : 0;
        out[2] = d.placed ? d.s : 0;
        out[3] = d.placed ? (int)ms_of(arg) : 0;
        out[4] = d.placed && d.reused;
        out[5] = (int)d.evals;
    } else if (a.op == SOP_TRY_DEQUEUE) {
        sim.dequeue_pass();
        out[0] = (int)sim.q_head;  // placed heads
        out[1] = (int)sim.n_ev;
        sim.store_snapshot(a, i);
    } else {
        // on_departure (migration.cpp:212-220) / plan_intra / plan_inter
        int kind = -1, status = 0;
        const unsigned w0 = ws->gw[arg];
        const bool lazy = (sim.lazymask >> wp::popc(w0 & 0x7Fu)) & 1u;
        if (a.op == SOP_ON_DEPARTURE) {
            if (a.enabled) {
                kind = lazy ? 1 : 0;
                if (lazy) sim.plan_inter(arg);
                else sim.plan_intra(arg);
            }
        } else if (a.op == SOP_PLAN_INTRA) {
            kind = 0;
            sim.plan_intra(arg);
        } else {
            if (!lazy) {
                status = 5;  // NotLazy (migration.cpp:127-129)
            } else {
                kind = 1;
                sim.plan_inter(arg);
            }
        }
        out[0] = status;
        out[1] = kind;
        out[2] = (int)sim.n_mig;
        out[3] = (int)sim.n_plan_iter;
        out[4] = kind == 0 ? sim.max_intra : sim.max_inter;
        out[5] = (int)sim.n_ev;
        sim.store_snapshot(a, i);
    }
    if (sim.L == 0)
        for (int k = 0; k < 8; ++k) a.out[(size_t)i * 8 + k] = out[k];
}

}  // namespace msgk
