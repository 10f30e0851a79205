/*
 * ORACLE / TEST INFRASTRUCTURE — never linked into the product.
 *
 * oracle_port.c: a plain-C restatement of the reference's scheduler hot
 * path (arXiv 2512.16099 "migsched", /root/reference/proj), written as a
 * straightforward scalar program: instance vectors, an explicit binary heap
 * of timers including stale completions, a linear FCFS queue.  Each function
 * cites the reference file:line it follows (paths relative to proj/).  It
 * emits the record formats of include/migsched_b200.h so tests can diff it
 * against the GPU engine and against the reference library itself
 * (tests/test_oracle_port.py pins it to the reference and to the golden
 * vectors in tests/golden/).
 *
 * Built by oracle/Makefile with -O2 -ffp-contract=off (no FMA: SURVEY §7).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "migsched_b200.h"

/* ---- MIG geometry: profiles.cpp:8-15 ------------------------------------ */
static const int P_CS[6] = {7, 4, 3, 2, 1, 1};
static const int P_MS[6] = {8, 4, 4, 2, 2, 1};
static const int P_NSTART[6] = {1, 1, 2, 3, 4, 7};
static const int P_STARTS[6][7] = {
    {0}, {0}, {0, 4}, {0, 2, 4}, {0, 2, 4, 6}, {0, 1, 2, 3, 4, 5, 6}};

static int legal_start(int p, int s) { /* valid(): profiles.cpp:31-37 */
    for (int i = 0; i < P_NSTART[p]; ++i)
        if (P_STARTS[p][i] == s) return 1;
    return 0;
}
static unsigned run_mask(int start, int count) { /* slice_mask: profiles.cpp:43-45 */
    return (((1u << count) - 1u) << start) & 0xFFu;
}
static unsigned fp_c(int p, int s) { return run_mask(s, P_CS[p]); } /* slice_footprint :49-57 */
static unsigned fp_m(int p, int s) { return run_mask(s, P_MS[p]); }

/* ---- GPU occupancy model: gpu.hpp:18-97, gpu.cpp ------------------------ */
typedef struct {
    uint64_t id;
    int profile, start;
    int has_job;
    int64_t job;
    int draining;
} Inst;

typedef struct {
    int id;
    Inst inst[16];
    int n;
    uint64_t next_id;
} Gpu;

static int inst_busy(const Inst* i) { return i->has_job; }
static int inst_idle(const Inst* i) { return !i->has_job && !i->draining; }
static int inst_blocks(const Inst* i) { return i->has_job || i->draining; }

static unsigned busy_c(const Gpu* g) { /* gpu.cpp:10-16 */
    unsigned m = 0;
    for (int k = 0; k < g->n; ++k)
        if (inst_busy(&g->inst[k])) m |= fp_c(g->inst[k].profile, g->inst[k].start);
    return m;
}
static unsigned busy_m(const Gpu* g) { /* gpu.cpp:18-24 */
    unsigned m = 0;
    for (int k = 0; k < g->n; ++k)
        if (inst_busy(&g->inst[k])) m |= fp_m(g->inst[k].profile, g->inst[k].start);
    return m;
}
static unsigned blocked_c(const Gpu* g) { /* gpu.cpp:26-32 */
    unsigned m = 0;
    for (int k = 0; k < g->n; ++k)
        if (inst_blocks(&g->inst[k])) m |= fp_c(g->inst[k].profile, g->inst[k].start);
    return m;
}
static unsigned blocked_m(const Gpu* g) { /* gpu.cpp:34-40 */
    unsigned m = 0;
    for (int k = 0; k < g->n; ++k)
        if (inst_blocks(&g->inst[k])) m |= fp_m(g->inst[k].profile, g->inst[k].start);
    return m;
}

static const Inst* find_idle_exact(const Gpu* g, int p, int s) { /* gpu.cpp:64-69 */
    for (int k = 0; k < g->n; ++k)
        if (inst_idle(&g->inst[k]) && g->inst[k].profile == p && g->inst[k].start == s) return &g->inst[k];
    return NULL;
}

/* avail(): gpu.cpp:158-166 */
static int avail(const Gpu* g, int p, int s) {
    return (fp_c(p, s) & blocked_c(g)) == 0 && (fp_m(p, s) & blocked_m(g)) == 0;
}

static double utilization(const Gpu* g) { /* gpu.cpp:168-170 */
    return (double)__builtin_popcount(busy_c(g)) / 7.0;
}
static int is_lazy(const Gpu* g, double threshold) { /* classify: gpu.cpp:172-177 */
    return utilization(g) < threshold;
}

typedef struct {
    int action; /* 0 create, 1 destroy */
    int profile, start;
} Op;

typedef struct {
    uint64_t instance;
    int reused;
    Op ops[16];
    int n_ops;
} CreateRes;

/* create_instance: gpu.cpp:71-101.  Returns 0 or a msg status. */
static int create_instance(Gpu* g, int p, int s, int64_t job, CreateRes* out) {
    out->reused = 0;
    out->n_ops = 0;
    if (!legal_start(p, s)) return MSG_ERR_INVALID_PLACEMENT;
    if ((fp_c(p, s) & blocked_c(g)) || (fp_m(p, s) & blocked_m(g))) return MSG_ERR_SLICES_BUSY;
    for (int k = 0; k < g->n; ++k) {
        Inst* i = &g->inst[k];
        if (inst_idle(i) && i->profile == p && i->start == s) {
            i->has_job = 1;
            i->job = job;
            out->instance = i->id;
            out->reused = 1;
            return MSG_OK;
        }
    }
    /* erase_if keeps the survivors' order; each erased idle instance is one
       destroy op in vector order */
    int w = 0;
    for (int k = 0; k < g->n; ++k) {
        Inst* i = &g->inst[k];
        const int hit = inst_idle(i) && ((fp_c(i->profile, i->start) & fp_c(p, s)) ||
                                         (fp_m(i->profile, i->start) & fp_m(p, s)));
        if (hit) {
            out->ops[out->n_ops++] = (Op){1, i->profile, i->start};
        } else {
            g->inst[w++] = *i;
        }
    }
    g->n = w;
    Inst created = {g->next_id++, p, s, 1, job, 0};
    out->instance = created.id;
    out->ops[out->n_ops++] = (Op){0, p, s};
    g->inst[g->n++] = created;
    return MSG_OK;
}

/* add_idle_instance: gpu.cpp:103-113 */
static int add_idle(Gpu* g, int p, int s) {
    if (p < 0 || p >= 6) return MSG_ERR_UNKNOWN_PROFILE;
    if (!legal_start(p, s)) return MSG_ERR_INVALID_PLACEMENT;
    for (int k = 0; k < g->n; ++k) {
        const Inst* i = &g->inst[k];
        if ((fp_c(i->profile, i->start) & fp_c(p, s)) || (fp_m(i->profile, i->start) & fp_m(p, s)))
            return MSG_ERR_SLICES_BUSY;
    }
    g->inst[g->n++] = (Inst){g->next_id++, p, s, 0, 0, 0};
    return MSG_OK;
}

static int release_job(Gpu* g, int64_t job) { /* gpu.cpp:115-123 */
    for (int k = 0; k < g->n; ++k)
        if (g->inst[k].has_job && g->inst[k].job == job) {
            g->inst[k].has_job = 0;
            return MSG_OK;
        }
    return MSG_ERR_UNKNOWN_JOB;
}

static uint64_t start_draining(Gpu* g, int64_t job) { /* gpu.cpp:125-135 */
    for (int k = 0; k < g->n; ++k)
        if (g->inst[k].has_job && g->inst[k].job == job) {
            g->inst[k].has_job = 0;
            g->inst[k].draining = 1;
            return g->inst[k].id;
        }
    return 0;
}

static void finish_draining(Gpu* g, uint64_t id) { /* gpu.cpp:137-144 */
    for (int k = 0; k < g->n; ++k)
        if (g->inst[k].id == id) {
            g->inst[k].draining = 0;
            return;
        }
}

/* ---- fragmentation metric: frag.cpp:10-58 ------------------------------ */
typedef struct {
    long num, den;
} Frac;

static int frac_cmp(Frac a, Frac b) { /* frag.hpp:20-25: cross-multiplication */
    const long long l = (long long)a.num * b.den, r = (long long)b.num * a.den;
    return l < r ? -1 : l > r ? 1 : 0;
}

static Frac frag_cost4(unsigned bc, unsigned bm, unsigned kc, unsigned km) {
    const int rc = 7 - __builtin_popcount(bc), rm = 8 - __builtin_popcount(bm);
    long sum = 0;
    int counted = 0;
    for (int p = 0; p < 6; ++p) {
        const int a = rc / P_CS[p], b = rm / P_MS[p];
        const int ideal = a < b ? a : b; /* ideal_from_masks: frag.cpp:12-16 */
        if (ideal == 0) continue;
        int feasible = 0; /* feasible_from_masks: frag.cpp:18-26 */
        for (int i = 0; i < P_NSTART[p]; ++i) {
            const int s = P_STARTS[p][i];
            if (!(fp_c(p, s) & kc) && !(fp_m(p, s) & km)) ++feasible;
        }
        sum += (long)feasible * (420 / ideal);
        ++counted;
    }
    if (counted == 0) return (Frac){0, 1};
    const long den = 420L * counted;
    return (Frac){den - sum, den};
}
static Frac frag_cost2(unsigned bc, unsigned bm) { return frag_cost4(bc, bm, bc, bm); }
static double frac_d(Frac f) { return (double)f.num / (double)f.den; }
static double frag_cost_gpu(const Gpu* g) { /* frag.cpp:60-65 */
    return frac_d(frag_cost4(busy_c(g), busy_m(g), blocked_c(g), blocked_m(g)));
}

/* ---- scheduler: scheduler.cpp:19-121 ------------------------------------ */
typedef struct {
    int placed, gpu, start, reused, evals;
} Decision;

typedef struct {
    double threshold;
    int lb, dyn;
} SchedCfg;

/* schedule(): scheduler.cpp:47-81 (Lazy pass, then Busy) */
static Decision schedule(int p, const Gpu* gpus, int G, const SchedCfg* c) {
    Decision d = {0, -1, 0, 0, 0};
    for (int pass = 0; pass < 2; ++pass) {
        int have = 0;
        Frac bcost = {0, 1};
        int breused = 0, bgpu = 0, bstart = 0;
        for (int gi = 0; gi < G; ++gi) {
            const Gpu* g = &gpus[gi];
            if (is_lazy(g, c->threshold) != (pass == 0)) continue;
            const unsigned bc = busy_c(g), bm = busy_m(g);
            for (int i = 0; i < P_NSTART[p]; ++i) { /* candidate_starts: :19-28 */
                const int s = P_STARTS[p][i];
                if (!c->dyn && !find_idle_exact(g, p, s)) continue;
                if (!avail(g, p, s)) continue;
                const Frac cost = frag_cost2(bc | fp_c(p, s), bm | fp_m(p, s));
                const int reused = find_idle_exact(g, p, s) != NULL;
                ++d.evals;
                /* better_than: cost, reuse, gpu, start (:37-42) */
                int better = !have;
                if (have) {
                    const int cmp = frac_cmp(cost, bcost);
                    if (cmp != 0) better = cmp < 0;
                    else if (reused != breused) better = reused;
                    else if (g->id != bgpu) better = g->id < bgpu;
                    else better = s < bstart;
                }
                if (better) {
                    have = 1;
                    bcost = cost;
                    breused = reused;
                    bgpu = g->id;
                    bstart = s;
                }
            }
        }
        if (have) {
            d.placed = 1;
            d.gpu = bgpu;
            d.start = bstart;
            d.reused = breused;
            return d;
        }
    }
    return d;
}

/* first_fit_schedule(): scheduler.cpp:83-98 */
static Decision first_fit(int p, const Gpu* gpus, int G, const SchedCfg* c) {
    Decision d = {0, -1, 0, 0, 0};
    for (int gi = 0; gi < G; ++gi) {
        const Gpu* g = &gpus[gi];
        for (int i = 0; i < P_NSTART[p]; ++i) {
            const int s = P_STARTS[p][i];
            if (!c->dyn && !find_idle_exact(g, p, s)) continue;
            if (!avail(g, p, s)) continue;
            d.placed = 1;
            d.gpu = g->id;
            d.start = s;
            d.reused = find_idle_exact(g, p, s) != NULL;
            return d;
        }
    }
    return d;
}

static Decision dispatch(int p, const Gpu* gpus, int G, const SchedCfg* c) { /* :100-104 */
    return c->lb ? schedule(p, gpus, G, c) : first_fit(p, gpus, G, c);
}

/* ---- migration: migration.cpp:35-220 ------------------------------------ */
typedef struct {
    int64_t job;
    int profile, from_gpu, from_start, to_gpu, to_start, inter;
    double overlap;
    uint64_t source_instance;
    CreateRes create;
    double fcb, fca, tcb, tca;
} Move;

typedef struct {
    Move* moves;
    int n, cap;
    int kind; /* -1 none, 0 intra, 1 inter */
    int max_evals, n_iter;
} Plan;

static void plan_push(Plan* pl, const Move* m) {
    if (pl->n == pl->cap) {
        pl->cap = pl->cap ? 2 * pl->cap : 8;
        pl->moves = (Move*)realloc(pl->moves, sizeof(Move) * pl->cap);
    }
    pl->moves[pl->n++] = *m;
}
static void plan_iter(Plan* pl, int evals) {
    ++pl->n_iter;
    if (evals > pl->max_evals) pl->max_evals = evals;
}

static double end_cost(const Gpu* g) { return frac_d(frag_cost2(busy_c(g), busy_m(g))); }

/* apply_move(): migration.cpp:35-69 (replica first) */
static void apply_move(Gpu* gpus, Move* m) {
    Gpu* from = &gpus[m->from_gpu];
    Gpu* to = &gpus[m->to_gpu];
    m->fcb = end_cost(from);
    m->tcb = end_cost(to);
    m->source_instance = start_draining(from, m->job);
    create_instance(to, m->profile, m->to_start, m->job, &m->create);
    if (m->overlap <= 0.0) finish_draining(from, m->source_instance);
    m->fca = end_cost(from);
    m->tca = end_cost(to);
}

/* plan_intra(): migration.cpp:71-123 */
static void plan_intra(Gpu* gpus, int gi, double overlap, Plan* pl) {
    Gpu* g = &gpus[gi];
    pl->kind = 0;
    for (;;) {
        const unsigned bc = busy_c(g), bm = busy_m(g), kc = blocked_c(g), km = blocked_m(g);
        const Frac cur = frag_cost2(bc, bm);
        int evals = 0, have = 0;
        Frac best = {0, 1};
        int64_t bjob = 0;
        int bstart = 0, bprof = 0, bfrom = 0;
        for (int k = 0; k < g->n; ++k) {
            const Inst* i = &g->inst[k];
            if (!inst_busy(i)) continue;
            const int p = i->profile;
            const unsigned oc = fp_c(p, i->start), om = fp_m(p, i->start);
            for (int j = 0; j < P_NSTART[p]; ++j) {
                const int s = P_STARTS[p][j];
                if (s == i->start) continue;
                if ((fp_c(p, s) & kc) || (fp_m(p, s) & km)) continue;
                const Frac cost = frag_cost2((bc & ~oc) | fp_c(p, s), (bm & ~om) | fp_m(p, s));
                ++evals;
                int better = !have;
                if (have) { /* cost, job id, start */
                    const int cmp = frac_cmp(cost, best);
                    if (cmp != 0) better = cmp < 0;
                    else if (i->job != bjob) better = i->job < bjob;
                    else better = s < bstart;
                }
                if (better) {
                    have = 1;
                    best = cost;
                    bjob = i->job;
                    bstart = s;
                    bprof = p;
                    bfrom = i->start;
                }
            }
        }
        plan_iter(pl, evals);
        if (!have || frac_cmp(best, cur) >= 0) break; /* strict improvement */
        Move m;
        memset(&m, 0, sizeof(m));
        m.job = bjob;
        m.profile = bprof;
        m.from_gpu = gi;
        m.from_start = bfrom;
        m.to_gpu = gi;
        m.to_start = bstart;
        m.inter = 0;
        m.overlap = overlap;
        apply_move(gpus, &m);
        plan_push(pl, &m);
    }
}

/* plan_inter(): migration.cpp:125-210 */
static int plan_inter(Gpu* gpus, int G, int lazy_id, double threshold, double overlap, Plan* pl) {
    Gpu* lazy = &gpus[lazy_id];
    if (!is_lazy(lazy, threshold)) return MSG_ERR_NOT_LAZY;
    pl->kind = 1;
    for (;;) {
        int evals = 0, have = 0;
        Frac best = {0, 1};
        int bgpu = 0, bprof = 0, bfrom = 0;
        int64_t bjob = 0;
        const int lazy_cs = __builtin_popcount(busy_c(lazy));
        for (int gi = 0; gi < G; ++gi) {
            Gpu* src = &gpus[gi];
            if (gi == lazy_id) continue;
            if (is_lazy(src, threshold)) continue;
            const int src_cs = __builtin_popcount(busy_c(src));
            for (int k = 0; k < src->n; ++k) {
                const Inst* i = &src->inst[k];
                if (!inst_busy(i)) continue;
                const int p = i->profile;
                if (lazy_cs + P_CS[p] >= src_cs - P_CS[p]) continue;
                int placeable = 0;
                for (int j = 0; j < P_NSTART[p] && !placeable; ++j) placeable = avail(lazy, p, P_STARTS[p][j]);
                if (!placeable) continue;
                const Frac cost = frag_cost2(busy_c(src) & ~fp_c(p, i->start), busy_m(src) & ~fp_m(p, i->start));
                ++evals;
                int better = !have;
                if (have) { /* cost, gpu id, job id */
                    const int cmp = frac_cmp(cost, best);
                    if (cmp != 0) better = cmp < 0;
                    else if (gi != bgpu) better = gi < bgpu;
                    else better = i->job < bjob;
                }
                if (better) {
                    have = 1;
                    best = cost;
                    bgpu = gi;
                    bjob = i->job;
                    bprof = p;
                    bfrom = i->start;
                }
            }
        }
        if (!have) {
            plan_iter(pl, evals);
            break;
        }
        int dhave = 0, dstart = 0;
        Frac dbest = {0, 1};
        for (int j = 0; j < P_NSTART[bprof]; ++j) { /* destination: min cost, lowest start */
            const int s = P_STARTS[bprof][j];
            if (!avail(lazy, bprof, s)) continue;
            const Frac cost = frag_cost2(busy_c(lazy) | fp_c(bprof, s), busy_m(lazy) | fp_m(bprof, s));
            ++evals;
            if (!dhave || frac_cmp(cost, dbest) < 0) {
                dhave = 1;
                dbest = cost;
                dstart = s;
            }
        }
        plan_iter(pl, evals);
        Move m;
        memset(&m, 0, sizeof(m));
        m.job = bjob;
        m.profile = bprof;
        m.from_gpu = bgpu;
        m.from_start = bfrom;
        m.to_gpu = lazy_id;
        m.to_start = dstart;
        m.inter = 1;
        m.overlap = overlap;
        apply_move(gpus, &m);
        plan_push(pl, &m);
    }
    return MSG_OK;
}

/* ---- discrete-event engine: sim.cpp:33-410 ------------------------------ */
enum { T_COMPLETION = 0, T_MIGRATION_END = 1, T_SERVICE_START = 2, T_ARRIVAL = 3 };
enum { J_PENDING, J_QUEUED, J_WAITING, J_RUNNING, J_DONE };

typedef struct {
    double time;
    int kind;
    int64_t job;
    long gen;
    int gpu;
    uint64_t instance;
    uint64_t seq;
} Timer;

static int timer_later(const Timer* a, const Timer* b) { /* TimerLater: sim.cpp:49-56 */
    if (a->time != b->time) return a->time > b->time;
    if (a->kind != b->kind) return a->kind > b->kind;
    if (a->job != b->job) return a->job > b->job;
    return a->seq > b->seq;
}

typedef struct {
    Timer* v;
    size_t n, cap;
} Heap;

static void heap_push(Heap* h, Timer t) {
    if (h->n == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->v = (Timer*)realloc(h->v, sizeof(Timer) * h->cap);
    }
    size_t i = h->n++;
    h->v[i] = t;
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (!timer_later(&h->v[p], &h->v[i])) break;
        Timer x = h->v[p];
        h->v[p] = h->v[i];
        h->v[i] = x;
        i = p;
    }
}
static Timer heap_pop(Heap* h) {
    Timer top = h->v[0];
    h->v[0] = h->v[--h->n];
    size_t i = 0;
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < h->n && timer_later(&h->v[m], &h->v[l])) m = l;
        if (r < h->n && timer_later(&h->v[m], &h->v[r])) m = r;
        if (m == i) break;
        Timer x = h->v[m];
        h->v[m] = h->v[i];
        h->v[i] = x;
        i = m;
    }
    return top;
}

typedef struct {
    int64_t id;
    double arrival, service;
    int profile;
    int state, gpu;
    uint64_t instance;
    double rem, last;
    long gen;
    int migrations;
} RJob;

typedef struct {
    msg_event* v;
    size_t n, cap;
} Log;

static msg_event* log_add(Log* l, double t, int kind) {
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 256;
        l->v = (msg_event*)realloc(l->v, sizeof(msg_event) * l->cap);
    }
    msg_event* e = &l->v[l->n++];
    memset(e, 0, sizeof(*e));
    e->time_s = t;
    e->kind = kind;
    return e;
}

typedef struct {
    /* config */
    int G;
    SchedCfg sc;
    int migration;
    double alpha, overlap, latency;
    /* state */
    Gpu* gpus;
    RJob* jobs;
    size_t nj;
    int64_t* sorted_ids; /* index_by_id_: sorted (id, index) */
    uint32_t* sorted_idx;
    int64_t* queue;
    size_t qh, qt;
    Heap timers;
    Log log;
    int* running_on;
    msg_timeline_point* tl;
    size_t ntl, captl;
    int max_arr, max_intra, max_inter;
    double now;
    uint64_t seq;
    uint64_t handler;
    int err;
} Sim;

static RJob* job_ref(Sim* s, int64_t id) { /* index_by_id_.at(id) */
    size_t lo = 0, hi = s->nj;
    while (lo < hi) {
        size_t mid = (lo + hi) / 2;
        if (s->sorted_ids[mid] < id) lo = mid + 1;
        else hi = mid;
    }
    return &s->jobs[s->sorted_idx[lo]];
}

static void push_timer(Sim* s, double t, int kind, int64_t job, long gen, int gpu, uint64_t inst) {
    Timer x = {t, kind, job, gen, gpu, inst, s->seq++};
    heap_push(&s->timers, x);
}

static double slowdown(int k, double alpha) { return 1.0 + alpha * (double)(k - 1); } /* sim.cpp:26-31 */

static void advance_all(Sim* s) { /* sim.cpp:153-165 */
    for (size_t i = 0; i < s->nj; ++i) {
        RJob* j = &s->jobs[i];
        if (j->state != J_RUNNING) continue;
        const double dt = s->now - j->last;
        if (dt > 0.0) {
            const double f = slowdown(s->running_on[j->gpu], s->alpha);
            j->rem -= dt / f;
        }
        j->last = s->now;
    }
}

static void reschedule(Sim* s) { /* sim.cpp:167-175 */
    for (size_t i = 0; i < s->nj; ++i) {
        RJob* j = &s->jobs[i];
        if (j->state != J_RUNNING) continue;
        const double f = slowdown(s->running_on[j->gpu], s->alpha);
        const double r = j->rem < 0.0 ? 0.0 : j->rem;
        ++j->gen;
        push_timer(s, s->now + r * f, T_COMPLETION, j->id, j->gen, -1, 0);
    }
}

static void sample(Sim* s) { /* sim.cpp:177-181 */
    double total = 0.0;
    for (int g = 0; g < s->G; ++g) total += frag_cost_gpu(&s->gpus[g]);
    if (s->ntl == s->captl) {
        s->captl = s->captl ? 2 * s->captl : 256;
        s->tl = (msg_timeline_point*)realloc(s->tl, sizeof(msg_timeline_point) * s->captl);
    }
    s->tl[s->ntl++] = (msg_timeline_point){s->now, total / (double)s->G};
}

static void emit_ops(Sim* s, int gpu, const CreateRes* c) { /* sim.cpp:183-195 */
    for (int k = 0; k < c->n_ops; ++k) {
        msg_event* e = log_add(&s->log, s->now, MSG_EV_RECONFIG);
        e->gpu = gpu;
        e->action = c->ops[k].action;
        e->profile = c->ops[k].profile;
        e->start = c->ops[k].start;
        e->size = P_MS[c->ops[k].profile];
        e->present = MSG_HAS_GPU | MSG_HAS_ACTION | MSG_HAS_PROFILE | MSG_HAS_START | MSG_HAS_SIZE;
    }
}

static void start_service(Sim* s, RJob* j) { /* sim.cpp:212-218 */
    j->state = J_RUNNING;
    j->rem = j->service;
    j->last = s->now;
    ++s->running_on[j->gpu];
}

static double apply_placement(Sim* s, RJob* j, int gpu, const CreateRes* c) { /* sim.cpp:199-210 */
    j->gpu = gpu;
    j->instance = c->instance;
    const double delay = (double)c->n_ops * s->latency;
    const double ss = s->now + delay;
    if (delay > 0.0) {
        j->state = J_WAITING;
        push_timer(s, ss, T_SERVICE_START, j->id, 0, -1, 0);
    } else {
        start_service(s, j);
    }
    return ss;
}

static void place_event(msg_event* e, const RJob* j, const Decision* d, const CreateRes* c, double ss) {
    e->job = j->id;
    e->gpu = d->gpu;
    e->start = d->start;
    e->size = P_MS[j->profile];
    e->reused = c->reused;
    e->scheduled_s = ss;
    e->present |= MSG_HAS_JOB | MSG_HAS_GPU | MSG_HAS_START | MSG_HAS_SIZE | MSG_HAS_REUSED | MSG_HAS_SCHEDULED;
}

static void dequeue_pass(Sim* s) { /* sim.cpp:325-344 with try_dequeue scheduler.cpp:106-121 */
    while (s->qh < s->qt) {
        RJob* j = job_ref(s, s->queue[s->qh]);
        const Decision d = dispatch(j->profile, s->gpus, s->G, &s->sc);
        if (!d.placed) break;
        ++s->qh;
        CreateRes c;
        create_instance(&s->gpus[d.gpu], j->profile, d.start, j->id, &c);
        if (d.evals > s->max_arr) s->max_arr = d.evals;
        const double ss = apply_placement(s, j, d.gpu, &c);
        place_event(log_add(&s->log, s->now, MSG_EV_DEQUEUE), j, &d, &c, ss);
        emit_ops(s, d.gpu, &c);
    }
}

static void record_plan(Sim* s, const Plan* pl) { /* sim.cpp:346-396 */
    if (pl->n_iter) {
        if (pl->kind == 0) {
            if (pl->max_evals > s->max_intra) s->max_intra = pl->max_evals;
        } else if (pl->max_evals > s->max_inter) {
            s->max_inter = pl->max_evals;
        }
    }
    for (int k = 0; k < pl->n; ++k) {
        const Move* m = &pl->moves[k];
        RJob* j = job_ref(s, m->job);
        if (j->state == J_RUNNING) {
            --s->running_on[m->from_gpu];
            ++s->running_on[m->to_gpu];
        }
        j->gpu = m->to_gpu;
        j->instance = m->create.instance;
        ++j->migrations;
        msg_event* e = log_add(&s->log, s->now, MSG_EV_MIGRATION_START);
        e->job = m->job;
        e->profile = m->profile;
        e->from_gpu = m->from_gpu;
        e->from_start = m->from_start;
        e->to_gpu = m->to_gpu;
        e->to_start = m->to_start;
        e->move_kind = m->inter;
        e->overlap_s = m->overlap;
        e->from_cost_before = m->fcb;
        e->from_cost_after = m->fca;
        e->to_cost_before = m->tcb;
        e->to_cost_after = m->tca;
        e->present = MSG_HAS_JOB | MSG_HAS_PROFILE | MSG_HAS_FROM_GPU | MSG_HAS_FROM_START | MSG_HAS_TO_GPU |
                     MSG_HAS_TO_START | MSG_HAS_MOVE_KIND | MSG_HAS_OVERLAP | MSG_HAS_COSTS;
        emit_ops(s, m->to_gpu, &m->create);
        if (m->overlap > 0.0) {
            push_timer(s, s->now + m->overlap, T_MIGRATION_END, m->job, 0, m->from_gpu, m->source_instance);
        } else {
            msg_event* x = log_add(&s->log, s->now, MSG_EV_MIGRATION_END);
            x->job = m->job;
            x->gpu = m->from_gpu;
            x->present = MSG_HAS_JOB | MSG_HAS_GPU;
        }
    }
}

static void handle_arrival(Sim* s, const Timer* t) { /* sim.cpp:220-267 */
    advance_all(s);
    RJob* j = job_ref(s, t->job);
    msg_event* e = log_add(&s->log, s->now, MSG_EV_ARRIVAL);
    e->job = j->id;
    e->profile = j->profile;
    e->present = MSG_HAS_JOB | MSG_HAS_PROFILE;
    int enqueue = s->qh < s->qt;
    if (!enqueue) {
        const Decision d = dispatch(j->profile, s->gpus, s->G, &s->sc);
        if (d.evals > s->max_arr) s->max_arr = d.evals;
        if (d.placed) {
            CreateRes c;
            create_instance(&s->gpus[d.gpu], j->profile, d.start, j->id, &c);
            const double ss = apply_placement(s, j, d.gpu, &c);
            place_event(&s->log.v[s->log.n - 1], j, &d, &c, ss);
            emit_ops(s, d.gpu, &c);
        } else {
            enqueue = 1;
        }
    }
    if (enqueue) {
        j->state = J_QUEUED;
        s->queue[s->qt++] = j->id;
        msg_event* q = log_add(&s->log, s->now, MSG_EV_ENQUEUE);
        q->job = j->id;
        q->present = MSG_HAS_JOB;
    }
    reschedule(s);
    sample(s);
}

static void handle_completion(Sim* s, const Timer* t) { /* sim.cpp:269-301 */
    RJob* j = job_ref(s, t->job);
    if (j->state != J_RUNNING || t->gen != j->gen) return; /* superseded prediction */
    ++s->handler;
    advance_all(s);
    j->state = J_DONE;
    j->rem = 0.0;
    const int g = j->gpu;
    --s->running_on[g];
    release_job(&s->gpus[g], j->id);
    msg_event* e = log_add(&s->log, s->now, MSG_EV_COMPLETION);
    e->job = j->id;
    e->gpu = g;
    e->present = MSG_HAS_JOB | MSG_HAS_GPU;
    sample(s);
    dequeue_pass(s);
    if (s->migration) {
        Plan pl;
        memset(&pl, 0, sizeof(pl));
        pl.kind = -1;
        /* on_departure: migration.cpp:212-220 */
        if (!is_lazy(&s->gpus[g], s->sc.threshold)) plan_intra(s->gpus, g, s->overlap, &pl);
        else plan_inter(s->gpus, s->G, g, s->sc.threshold, s->overlap, &pl);
        record_plan(s, &pl);
        free(pl.moves);
        dequeue_pass(s);
    }
    reschedule(s);
    sample(s);
}

static void handle_migration_end(Sim* s, const Timer* t) { /* sim.cpp:303-315 */
    advance_all(s);
    finish_draining(&s->gpus[t->gpu], t->instance);
    msg_event* e = log_add(&s->log, s->now, MSG_EV_MIGRATION_END);
    e->job = t->job;
    e->gpu = t->gpu;
    e->present = MSG_HAS_JOB | MSG_HAS_GPU;
    dequeue_pass(s);
    reschedule(s);
    sample(s);
}

static void handle_service_start(Sim* s, const Timer* t) { /* sim.cpp:317-323 */
    advance_all(s);
    start_service(s, job_ref(s, t->job));
    reschedule(s);
    sample(s);
}

/* ---- result handle -------------------------------------------------------- */
typedef struct {
    int status;
    char message[256];
    msg_trace_summary summary;
    msg_event* events;
    size_t n_events;
    msg_job_row* jobs;
    size_t n_jobs;
    msg_timeline_point* timeline;
    size_t n_tl;
} PortResult;

static int cmp_pair(const void* a, const void* b) {
    const int64_t* x = (const int64_t*)a;
    const int64_t* y = (const int64_t*)b;
    return x[0] < y[0] ? -1 : x[0] > y[0] ? 1 : 0;
}

static const char* const NAMES[] = {"Ok", "InvalidPlacement", "SlicesBusy", "UnknownJob", "UnknownGpu",
                                    "NotLazy", "UnknownProfile", "BadThreshold", "BadConfig", "BadSpec",
                                    "TraceUnsorted", "BadConcurrency", "JobsPending", "ParseError"};

static PortResult* fail(PortResult* r, int st, const char* msg) {
    r->status = st;
    r->summary.status = st;
    snprintf(r->message, sizeof r->message, "%s: %s", NAMES[st], msg);
    return r;
}

/* metrics(): sim.cpp:414-502 — per job in id order from the log. */
static void metrics(Sim* s, PortResult* r) {
    const size_t n = s->nj;
    double* sched = (double*)malloc(sizeof(double) * (n ? n : 1));
    double* done = (double*)malloc(sizeof(double) * (n ? n : 1));
    int* has_s = (int*)calloc(n ? n : 1, sizeof(int));
    int* has_d = (int*)calloc(n ? n : 1, sizeof(int));
    int* gpu = (int*)malloc(sizeof(int) * (n ? n : 1));
    int* mig = (int*)calloc(n ? n : 1, sizeof(int));
    for (size_t i = 0; i < n; ++i) gpu[i] = -1;
    for (size_t k = 0; k < s->log.n; ++k) {
        const msg_event* e = &s->log.v[k];
        size_t lo = 0, hi = n; /* position in id order */
        if (e->present & MSG_HAS_JOB) {
            while (lo < hi) {
                size_t mid = (lo + hi) / 2;
                if (s->sorted_ids[mid] < e->job) lo = mid + 1;
                else hi = mid;
            }
        }
        switch (e->kind) {
            case MSG_EV_ARRIVAL:
                if (e->present & MSG_HAS_SCHEDULED) has_s[lo] = 1, sched[lo] = e->scheduled_s;
                if (e->present & MSG_HAS_GPU) gpu[lo] = e->gpu;
                break;
            case MSG_EV_DEQUEUE:
                has_s[lo] = 1;
                sched[lo] = e->scheduled_s;
                gpu[lo] = e->gpu;
                break;
            case MSG_EV_COMPLETION:
                has_d[lo] = 1;
                done[lo] = e->time_s;
                gpu[lo] = e->gpu;
                break;
            case MSG_EV_MIGRATION_START: ++mig[lo]; ++r->summary.migration_count; break;
            case MSG_EV_RECONFIG: ++r->summary.reconfig_op_count; break;
            case MSG_EV_ENQUEUE: ++r->summary.enqueue_count; break;
            default: break;
        }
        if (e->kind == MSG_EV_DEQUEUE) ++r->summary.dequeue_count;
    }
    for (size_t i = 0; i < n; ++i)
        if (!has_s[i] || !has_d[i]) {
            char msg[96];
            snprintf(msg, sizeof msg, "job %lld did not complete", (long long)s->sorted_ids[i]);
            fail(r, MSG_ERR_JOBS_PENDING, msg);
            goto out;
        }
    r->jobs = (msg_job_row*)calloc(n ? n : 1, sizeof(msg_job_row));
    r->n_jobs = n;
    double sw = 0.0, se = 0.0, st = 0.0, first = 0.0, last = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const RJob* j = &s->jobs[s->sorted_idx[i]];
        msg_job_row* row = &r->jobs[i];
        row->id = j->id;
        row->arrival_s = j->arrival;
        row->scheduled_s = sched[i];
        row->completed_s = done[i];
        row->wait_s = row->scheduled_s - row->arrival_s;
        row->execution_s = row->completed_s - row->scheduled_s;
        row->turnaround_s = row->wait_s + row->execution_s;
        row->profile = j->profile;
        row->gpu = gpu[i];
        row->migrations = mig[i];
        sw += row->wait_s;
        se += row->execution_s;
        st += row->turnaround_s;
        if (i == 0) {
            first = row->arrival_s;
            last = row->completed_s;
        } else {
            first = row->arrival_s < first ? row->arrival_s : first;
            last = last < row->completed_s ? row->completed_s : last;
        }
    }
    if (n) {
        r->summary.mean_wait_s = sw / (double)n;
        r->summary.mean_execution_s = se / (double)n;
        r->summary.mean_turnaround_s = st / (double)n;
        r->summary.workload_makespan_s = last - first;
    }
out:
    free(sched);
    free(done);
    free(has_s);
    free(has_d);
    free(gpu);
    free(mig);
}

static PortResult* run_one(const msg_trace_batch* b, uint32_t t, const msg_config* c, int want_detail) {
    PortResult* r = (PortResult*)calloc(1, sizeof(PortResult));
    r->summary.gpu_count = c->gpu_count;
    /* Engine::Engine validation: sim.cpp:73-116 */
    if (c->gpu_count < 1) return fail(r, MSG_ERR_BAD_CONFIG, "cluster must contain at least one GPU");
    if (c->threshold < 0.0 || c->threshold > 1.0)
        return fail(r, MSG_ERR_BAD_THRESHOLD, "load-balancing threshold must be in [0,1]");
    if (!c->dynamic_partitioning && !c->has_static_layout)
        return fail(r, MSG_ERR_BAD_CONFIG, "dynamic partitioning is off but no static layout is configured");
    Sim s;
    memset(&s, 0, sizeof(s));
    s.G = c->gpu_count;
    s.sc.threshold = c->threshold;
    s.sc.lb = c->load_balancing;
    s.sc.dyn = c->dynamic_partitioning;
    s.migration = c->migration;
    s.alpha = c->contention_alpha;
    s.overlap = c->migration_overlap_s;
    s.latency = c->reconfig_latency_s;
    s.gpus = (Gpu*)calloc((size_t)s.G, sizeof(Gpu));
    for (int g = 0; g < s.G; ++g) s.gpus[g].id = g, s.gpus[g].next_id = 1;
    s.running_on = (int*)calloc((size_t)s.G, sizeof(int));
    int err = MSG_OK;
    char emsg[128] = "";
    if (!c->dynamic_partitioning) {
        if (c->layout_gpus != c->gpu_count) {
            err = MSG_ERR_BAD_CONFIG;
            snprintf(emsg, sizeof emsg, "static layout must list every GPU in the cluster");
        }
        for (int g = 0; g < c->layout_gpus && !err; ++g)
            for (int i = c->layout_offsets[g]; i < c->layout_offsets[g + 1] && !err; ++i) {
                err = add_idle(&s.gpus[g], c->layout_profile[i], c->layout_start[i]);
                if (err) snprintf(emsg, sizeof emsg, "invalid static layout entry");
            }
    }
    const uint64_t lo = b->offsets[t], hi = b->offsets[t + 1];
    s.nj = hi - lo;
    s.jobs = (RJob*)calloc(s.nj ? s.nj : 1, sizeof(RJob));
    double prev = -1.0;
    for (uint64_t i = 0; i < s.nj && !err; ++i) {
        const uint64_t k = lo + i;
        RJob* j = &s.jobs[i];
        j->id = b->job_id[k];
        j->arrival = b->arrival_s[k];
        j->service = b->service_s[k];
        j->profile = b->profile[k];
        j->gpu = -1;
        if (j->profile < 0 || j->profile >= 6) {
            err = MSG_ERR_UNKNOWN_PROFILE;
            snprintf(emsg, sizeof emsg, "job %lld requests an unknown profile", (long long)j->id);
        } else if (j->arrival < prev) {
            err = MSG_ERR_TRACE_UNSORTED;
            snprintf(emsg, sizeof emsg, "job %lld arrives out of order", (long long)j->id);
        } else if (j->service <= 0.0) {
            err = MSG_ERR_BAD_SPEC;
            snprintf(emsg, sizeof emsg, "job %lld has non-positive service demand", (long long)j->id);
        } else if (isnan(j->arrival) || isnan(j->service)) {
            err = MSG_ERR_BAD_SPEC; /* engine contract: NaN times rejected */
            snprintf(emsg, sizeof emsg, "job %lld has a NaN time", (long long)j->id);
        } else {
            for (uint64_t q = 0; q < i; ++q)
                if (s.jobs[q].id == j->id) {
                    err = MSG_ERR_BAD_SPEC;
                    snprintf(emsg, sizeof emsg, "duplicate job id %lld", (long long)j->id);
                    break;
                }
        }
        prev = j->arrival;
    }
    if (!err) {
        /* index_by_id_: sorted (id, index) pairs */
        int64_t* pairs = (int64_t*)malloc(sizeof(int64_t) * 2 * (s.nj ? s.nj : 1));
        for (size_t i = 0; i < s.nj; ++i) pairs[2 * i] = s.jobs[i].id, pairs[2 * i + 1] = (int64_t)i;
        qsort(pairs, s.nj, 2 * sizeof(int64_t), cmp_pair);
        s.sorted_ids = (int64_t*)malloc(sizeof(int64_t) * (s.nj ? s.nj : 1));
        s.sorted_idx = (uint32_t*)malloc(sizeof(uint32_t) * (s.nj ? s.nj : 1));
        for (size_t i = 0; i < s.nj; ++i) s.sorted_ids[i] = pairs[2 * i], s.sorted_idx[i] = (uint32_t)pairs[2 * i + 1];
        free(pairs);
        s.queue = (int64_t*)malloc(sizeof(int64_t) * (s.nj ? s.nj : 1));
        for (size_t i = 0; i < s.nj; ++i) push_timer(&s, s.jobs[i].arrival, T_ARRIVAL, s.jobs[i].id, 0, -1, 0);
        /* execute(): sim.cpp:123-141 */
        while (s.timers.n) {
            const Timer x = heap_pop(&s.timers);
            s.now = x.time;
            switch (x.kind) {
                case T_ARRIVAL: ++s.handler; handle_arrival(&s, &x); break;
                case T_COMPLETION: handle_completion(&s, &x); break;
                case T_MIGRATION_END: ++s.handler; handle_migration_end(&s, &x); break;
                default: ++s.handler; handle_service_start(&s, &x); break;
            }
        }
        metrics(&s, r);
        if (r->status == MSG_OK) {
            r->summary.handler_events = s.handler;
            r->summary.n_events = s.log.n;
            r->summary.timeline_samples = s.ntl;
            r->summary.n_jobs = s.nj;
            r->summary.max_arrival_frag_evals = s.max_arr;
            r->summary.max_intra_iter_frag_evals = s.max_intra;
            r->summary.max_inter_iter_frag_evals = s.max_inter;
            double sum = 0.0;
            for (size_t i = 0; i < s.ntl; ++i) sum += s.tl[i].mean_frag_cost;
            r->summary.timeline_sum = sum;
            if (want_detail) {
                r->events = s.log.v;
                r->n_events = s.log.n;
                s.log.v = NULL;
                r->timeline = s.tl;
                r->n_tl = s.ntl;
                s.tl = NULL;
            }
        } else {
            memset(&r->summary, 0, sizeof(r->summary));
            r->summary.status = r->status;
            r->summary.gpu_count = c->gpu_count;
            free(r->jobs);
            r->jobs = NULL;
            r->n_jobs = 0;
        }
        if (!want_detail) {
            free(r->jobs);
            r->jobs = NULL;
            r->n_jobs = 0;
        }
    } else {
        fail(r, err, emsg);
    }
    free(s.gpus);
    free(s.running_on);
    free(s.jobs);
    free(s.sorted_ids);
    free(s.sorted_idx);
    free(s.queue);
    free(s.timers.v);
    free(s.log.v);
    free(s.tl);
    return r;
}

void* port_run(const msg_trace_batch* b, uint32_t t, const msg_config* c) { return run_one(b, t, c, 1); }
int port_result_status(void* h) { return ((PortResult*)h)->status; }
const char* port_result_message(void* h) { return ((PortResult*)h)->message; }
const msg_trace_summary* port_result_summary(void* h) { return &((PortResult*)h)->summary; }
const msg_event* port_result_events(void* h, uint64_t* n) {
    *n = ((PortResult*)h)->n_events;
    return ((PortResult*)h)->events;
}
const msg_job_row* port_result_jobs(void* h, uint64_t* n) {
    *n = ((PortResult*)h)->n_jobs;
    return ((PortResult*)h)->jobs;
}
const msg_timeline_point* port_result_timeline(void* h, uint64_t* n) {
    *n = ((PortResult*)h)->n_tl;
    return ((PortResult*)h)->timeline;
}
void port_result_free(void* h) {
    PortResult* r = (PortResult*)h;
    free(r->events);
    free(r->jobs);
    free(r->timeline);
    free(r);
}

/* Summaries only, single thread (a scalar port); returns wall seconds. */
double port_run_batch(const msg_trace_batch* b, const msg_config* cfgs, uint32_t n_cfgs, msg_trace_summary* out) {
    (void)n_cfgs;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (uint32_t t = 0; t < b->n_traces; ++t) {
        const uint32_t ci = b->config_index ? b->config_index[t] : 0;
        PortResult* r = run_one(b, t, &cfgs[ci], 0);
        out[t] = r->summary;
        port_result_free(r);
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* Cost numerator over 25200 of frag_cost_masks(bc, bm, kc, km). */
int32_t port_frag_k(uint8_t bc, uint8_t bm, uint8_t kc, uint8_t km) {
    const Frac f = frag_cost4(bc, bm, kc, km);
    return (int32_t)(f.num * (25200 / f.den));
}
