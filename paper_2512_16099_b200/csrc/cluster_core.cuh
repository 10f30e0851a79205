// cluster_core.cuh — the event loop for LARGE clusters (G > 32 GPUs, up to
// the 16384-GPU C4 configuration): one thread-block CLUSTER of S CTAs
// replays one trace of the reference's discrete-event scheduler
// (proj/src/sim.cpp:71-410); S = 1 is a single block.
//
// Sharding.  CTA `sh` (a SHARD) owns the contiguous GPU range
// [G*sh/S, G*(sh+1)/S) and everything that lives on it:
//   * per GPU: mask word (busy compute | busy memory | blocked memory |
//     running count), idle-exact placement bits, 4-mask cost id — in SHARED
//     memory (9 B/GPU), else global;
//   * per (GPU, start) slot: instance state, profile, creation sequence,
//     migrations of the bound job, position in the active list — in SHARED
//     memory too when the shard's 105 B/GPU fit (C4 at 16 shards: 105 KiB),
//     else global (L2-resident);
//   * the shard's ACTIVE list: every slot of its GPUs that carries a timer
//     (running, waiting for service start, draining) with the timer data
//     stored densely by list index (time, state, job, remaining work,
//     MigrationEnd order): the per-event scans (next event, advance_all,
//     reschedule, plan_inter sources) are coalesced loops over ~R/S entries;
//   * the shard's part of the integer fragmentation-cost total.
// Replicated in every shard (identical, because every input to them is
// either replicated or exchanged): the clock, the arrival cursor, the FCFS
// queue, the decision counters.
//
// Exchange.  Every decision that spans shards is one EXCHANGE: each shard
// reduces its own candidates block-wide (per-warp REDUX chain, one
// __syncthreads, the same chain over the warp winners) into one 96-byte
// record; lane k of warp 0 pushes it into CTA k's shared-memory inbox with
// st.async (distributed shared memory, completing on CTA k's mbarrier), and
// once its own barrier has counted all S records, warp 0 of every shard
// reduces them identically from local shared memory: lexicographic minimum key
// (with the winner's payload: the migrating job's slot, state, remaining
// work and timer), sums (candidate counts, cost-total parts) and ORs (the
// GPU word its owner broadcasts).  Inboxes and barriers are
// double-buffered by round parity; there is no cluster-wide barrier and no
// global-memory fence on this path.  Exchanges per handler:
//   next event (always; its record also carries the winning slot's GPU word,
//   which every shard then follows through the dequeue pass to classify a
//   completed job's GPU without an exchange) · one per placement attempt
//   (arrival, dequeue pass) · on a completion with migration onto a Lazy
//   GPU, one per plan_inter iteration.
// plan_intra, create_instance and the placement itself are owner-local.
// Fragmentation-timeline samples are deferred: each shard queues its part
// of the cost total at the sample point and the next exchange sums them.
//
// The MigrationEnd tie order (same job, same time: push order,
// sim.cpp:49-56) uses the job's migration count at the move, which grows
// with every move of the job — equivalent to the reference's global push
// sequence for every comparison that can tie, and shard-independent.
//
// Bit-exact with the reference, except the fragmentation timeline above
// kExactTimelineGpus GPUs: there the per-sample mean is
// RN(RN(sum_g k_g / 25200) / G) from the exact integer sum of the per-GPU
// cost numerators instead of the reference's sequential double sum (relative
// difference <= G * 2^-53, i.e. < 2e-12 at 16384 GPUs; SURVEY §7 hard part
// 6).  Sharding (S > 1 or D > 1) is used only above that size and without
// the event log.
//
// Device groups.  The same trace can be split further over D device groups
// (one cluster each; B200s of one NVLink/NVSwitch domain, or clusters of one
// GPU): shard gs = dv * S + sh of D * S.  An exchange then has two levels —
// the cluster level above, giving every CTA of a group the group's record,
// and one cross-group step in which CTA sh of each group stores that record
// into the inbox of every group (peer memory over NVLink, 96 B + a stamp
// written with st.release.sys) and waits on its own inbox stamps
// (ld.acquire.sys): a device-initiated all-reduce of packed keys per
// decision, no host round trip and no NCCL call on the path.  Job rows go
// to group 0's memory; the summary and timeline are written by group 0.
#pragma once
#include "engine_core.cuh"

namespace msgk {

#ifdef MSG_PHASE_PROF
// Development build only (tools/c4_phases.sh): SM cycles per phase of the
// event loop on CTA 0 of group 0 — 0 timer scan, 1 speculative placement
// search, 2 exchanges, 3 advance, 4 arrival, 5 departure, 6 service start,
// 7 reschedule + sample; [8] exchanges, [9] events.
__device__ unsigned long long g_phase[16];
#define MSG_PH(k) ph_mark(k)
#else
#define MSG_PH(k) ((void)0)
#endif

struct BlockScratch {
    unsigned hi[2][32], lo[2][32], tie[2][32], ms[2][32];
    int pay[2][32];
    unsigned sum[2][32];
    unsigned kh[2][32], kl[2][32], nl[2][32], nb[2][32];  // next_event: the fused placement search's partials
    double q[8];       // dt / slowdown(k), k = 1..7
    double f[8];       // slowdown(k)
    unsigned u[8];     // small broadcasts from one thread / warp 0
    int dl_slot[8];    // create_instance: destroyed starts in creation order
    int dl_prof[8];
    unsigned long long ksum;  // this shard's sum of per-GPU 4-mask cost numerators
    double tl;
    XRec xin[2][kMaxShards];  // records pushed by every shard, by round parity
    XInbox* ib[kMaxDev];      // every device group's inbox for this trace
    double pend_t[2];         // deferred timeline samples: time, this shard's cost total
    unsigned long long pend_k[2];
    XRec xr;                  // reduced record (within the cluster)
    XRec xr2;                 // reduced record (across device groups)
    uint64_t xbar[2];         // mbarriers counting the pushed bytes, by round parity
};

// ---- pieces of the block engine used at several call sites -----------------
// Free functions.  All kept out of line (MSG_DNI) they cut the C4 kernel
// from 25,880 to 13,744 SASS instructions (r02f ncu: 79% i-cache hit rate,
// 'no_instruction' the third stall), but most calls cost more than the
// misses they save: 20K-arrival C4 prefix 0.367 s vs 0.341 s inlined
// (profiles/r02, c4_variants_r02t.log); only the exchange reduction pays
// (r02u).  CL_OOL_* select each for A/B builds.
#ifndef C4_DISPATCH_UNROLL
#define C4_DISPATCH_UNROLL 1
#endif
constexpr int kC4DispatchUnroll = C4_DISPATCH_UNROLL;
#ifndef C4_SCAN_UNROLL
#define C4_SCAN_UNROLL 8
#endif
constexpr int kC4ScanUnroll = C4_SCAN_UNROLL;
#ifndef C4_HELD
#define C4_HELD 8  // active entries per thread kept in registers from the timer scan to advance_all
#endif
#ifndef C4_FUSED_SUMS
#define C4_FUSED_SUMS 1
#endif
#ifndef C4_DROP_BARRIERS
#define C4_DROP_BARRIERS 1
#endif
#ifndef CL_OOL_WORD
#define CL_OOL_WORD MSG_DI
#endif
#ifndef CL_OOL_TL
#define CL_OOL_TL MSG_DI
#endif
#ifndef CL_OOL_XRED
#define CL_OOL_XRED MSG_DNI  // out of line: 0.332 vs 0.337 s inlined (r02u)
#endif

// Idle-exact bit of placement (p, s): the profile's first bit + the start's
// index among its legal starts (strides are powers of two).
MSG_DI unsigned cl_pidx(int p, int s) {
    return ((0x00B74210u >> (4 * p)) & 0xFu) + ((unsigned)s >> ((0x011233u >> (4 * p)) & 0xFu));
}

// GPU word (busy/blocked masks, running count), idle-exact bits and 4-mask
// cost id from the GPU's 8 slots (gpu.cpp:10-48).
struct GpuWord {
    unsigned w, x, id;
};
CL_OOL_WORD GpuWord cl_gpu_word(const uint8_t* st8, const uint8_t* pr8, const DevTables* tb) {
    unsigned bc = 0, bm = 0, km = 0, k = 0, x = 0;
    for (int s = 0; s < 8; ++s) {
        const uint8_t v = st8[s];
        if (v == ST_EMPTY) continue;
        const int p = pr8[s];
        const unsigned m = fpm(p, s);
        if (v == ST_IDLE) {
            x |= 1u << cl_pidx(p, s);
        } else if (v == ST_DRAIN) {
            km |= m;
        } else {
            bc |= fpc(p, s);
            bm |= m;
            km |= m;
            k += v == ST_RUN;
        }
    }
    GpuWord r;
    r.w = bc | (bm << 8) | (km << 16) | (k << 24);
    r.x = x;
    const unsigned row = (unsigned)wp::popc(bc) * 9u + (unsigned)wp::popc(bm);
    r.id = tb->cost4pair[tb->idealid[row] * 32u + tb->feasid[km]];
    return r;
}

// Timeline mean of a cost total (numerators over 25200) over G GPUs.
CL_OOL_TL double cl_tl_mean(unsigned long long ktot, double inv_g, int G) {
    const double tot = wp::ddiv((double)ktot, 25200.0);
    return inv_g != 0.0 ? wp::dmul(tot, inv_g) : wp::ddiv(tot, (double)G);
}

// dt / slowdown(k)
CL_OOL_TL double cl_ddiv(double a, double b) { return wp::ddiv(a, b); }

// Lexicographic (hi, lo, tie, ms) minimum within the warp; every lane ends
// with the winning tuple and its payload.
MSG_DI void cl_warp_lexmin(unsigned& hi, unsigned& lo, unsigned& tie, unsigned& ms, int& pay) {
    const unsigned mhi = wp::rmin(hi);
    const unsigned mlo = wp::rmin(hi == mhi ? lo : NONE);
    const unsigned mtie = wp::rmin((hi == mhi && lo == mlo) ? tie : NONE);
    const bool m3 = hi == mhi && lo == mlo && tie == mtie;
    const unsigned mms = wp::rmin(m3 ? ms : NONE);
    const int wl = wp::ffs(wp::ballot(m3 && ms == mms)) - 1;
    pay = wp::shfl(pay, wl < 0 ? 0 : wl);
    hi = mhi;
    lo = mlo;
    tie = mtie;
    ms = mms;
}

MSG_DI XRec cl_xnone() {
    XRec r;
    r.hi = r.lo = r.tie = r.ms = NONE;
    r.slot = -1;
    r.job = -1;
    r.info = 0;
    r.w = 0;
    r.rem = r.tkey = 0.0;
    r.c[0] = r.c[1] = r.c[2] = r.c[3] = 0;
    r.mx = 0;
    r.pad = 0;
    r.ks[0] = r.ks[1] = 0;
    r.pad2 = ~0ull;
    return r;
}

// One warp: the identical reduction of records in[0 .. n) (one per lane;
// lanes >= n contribute cl_xnone()) — lexicographic minimum with the
// winner's payload, sums, OR, max — stored by lane 0 into *out.
CL_OOL_XRED void cl_xreduce(const XRec* in, unsigned n, XRec* out) {
    const unsigned L = wp::lane();
    const XRec x = L < n ? in[L] : cl_xnone();
    int pay = (int)L;
    unsigned hi = x.hi, lo = x.lo, tie = x.tie, ms = x.ms;
    cl_warp_lexmin(hi, lo, tie, ms, pay);
    XRec o;
    o.hi = hi;
    o.lo = lo;
    o.tie = tie;
    o.ms = ms;
    o.slot = wp::shfl(x.slot, pay);
    o.job = wp::shfl(x.job, pay);
    o.info = wp::shfl(x.info, pay);
    o.rem = wp::shfl(x.rem, pay);
    o.tkey = wp::shfl(x.tkey, pay);
    o.w = wp::ror(x.w);
    for (int k = 0; k < 4; ++k) o.c[k] = wp::radd(x.c[k]);
    o.mx = wp::rmax(x.mx);
    o.pad = 0;
    {  // pad2: a second 64-bit minimum (the speculative arrival decision key)
        const unsigned h = wp::rmin((unsigned)(x.pad2 >> 32));
        const unsigned l = wp::rmin((unsigned)(x.pad2 >> 32) == h ? (unsigned)x.pad2 : NONE);
        o.pad2 = ((uint64_t)h << 32) | l;
    }
    for (int k = 0; k < 2; ++k) {  // parts < 2^35: 20-bit split keeps the lane sums in 32 bits
        const unsigned lo20 = wp::radd((unsigned)(x.ks[k] & 0xFFFFFu));
        const unsigned hi20 = wp::radd((unsigned)(x.ks[k] >> 20));
        o.ks[k] = ((unsigned long long)hi20 << 20) + lo20;
    }
    if (L == 0) *out = o;
}

template <bool DETAIL>
struct ClusterSim {
    BlockScratch* sc;
    const DevTables* tb;
    const uint16_t* stab;  // per-word placement table (host_tables.h, build_score_table) or null
    // per slot (global slot index 8g + s)
    uint8_t* st;
    uint8_t* prof;
    uint16_t* mig;
    uint32_t* cseq;
    int32_t* apos;
    // per active entry of this shard
    int32_t* aslot;
    uint8_t* ast;
    int32_t* ajob;
    uint32_t* amseq;
    double* arem;
    double* atkey;
    // per owned GPU (index g - g_lo)
    uint32_t* gw;
    uint32_t* gx;
    uint8_t* gcid;
    const double* arr;
    const double* svc;
    const uint8_t* prf;
    const uint32_t* perm;
    int32_t* queue;
    JobOut* jobs;
    EventRec* evs;
    double* tl;
    uint32_t N, ev_cap, tl_cap, oflags;
    int G;
    uint32_t cflags, lazymask;
    double alpha, overlap, latency, inv_g;
    // shard geometry: S CTAs per cluster (rank sh), D device groups (this
    // one dv); global shard gs = dv * S + sh of NS = D * S
    unsigned S, sh, D, dv, gs, NS, epoch;
    int g_lo, g_hi;
    // block-uniform state (every thread holds the same values)
    unsigned T, W, L, w, NT;  // thread, warp, lane, warps, threads
    int bph;                  // scratch double-buffer parity
    uint32_t xround;          // exchanges so far
    double now, t_prev;
    uint32_t a_idx, a_rank;
    int a_prof;
    double a_t, a_svc;
    uint32_t q_head, q_tail, n_act;
    uint32_t cseq_ctr;
    uint32_t n_ev, n_handler, n_tl, n_mig, n_reconf, n_enq, n_deq;
    int max_arr, max_intra, max_inter;
    double tl_sum, tl_mean;
    bool tl_dirty;
    // deferred timeline samples (sharded)
    uint32_t npend;
    // sharded: the GPU word of the last completion's GPU, tracked by every
    // shard (from the next-event record, then through the placements of the
    // dequeue pass), so on_departure needs no exchange to classify it
    int dep_g;
    unsigned dep_w;
    // sharded: the pending arrival's decision, searched in the next-event exchange
    bool spec;
    uint64_t spec_key;
    unsigned spec_nl, spec_nb;
    // next_event -> advance_all: this thread's first kHeld active entries
    static constexpr int kHeld = C4_HELD;
    double held_rem[kHeld];
    unsigned held_k[kHeld];  // running count of the entry's GPU, 0: not Running

    // ------------------------------------------------------------- tables
    MSG_DI unsigned rank2(unsigned bc, unsigned bm) const { return tb->cost2rank[wp::popc(bc) * 256 + bm]; }
    MSG_DI unsigned k2w(unsigned wd) const { return tb->rank2k[rank2(w_bc(wd), w_bm(wd))]; }
    MSG_DI static unsigned pidx(int p, int s) {  // idle-exact bit of placement (p, s)
        return cl_pidx(p, s);
    }
    MSG_DI bool own(int g) const { return g >= g_lo && g < g_hi; }
    MSG_DI unsigned& W_(int g) { return gw[g - g_lo]; }  // owned GPU's mask word

    // ----------------------------------------------------- block reductions
    // Lexicographic (hi, lo, tie, ms) minimum within the warp; every lane
    // ends with the winning tuple and its payload.
    MSG_DI void warp_lexmin(unsigned& hi, unsigned& lo, unsigned& tie, unsigned& ms, int& pay) {
        cl_warp_lexmin(hi, lo, tie, ms, pay);
    }
    // ... and over the whole block (one __syncthreads).
    MSG_DI void block_lexmin(unsigned& hi, unsigned& lo, unsigned& tie, unsigned& ms, int& pay) {
        warp_lexmin(hi, lo, tie, ms, pay);
        if (L == 0) {
            sc->hi[bph][W] = hi;
            sc->lo[bph][W] = lo;
            sc->tie[bph][W] = tie;
            sc->ms[bph][W] = ms;
            sc->pay[bph][W] = pay;
        }
        wp::bsync();
        const bool v = L < w;
        hi = v ? sc->hi[bph][L] : NONE;
        lo = v ? sc->lo[bph][L] : NONE;
        tie = v ? sc->tie[bph][L] : NONE;
        ms = v ? sc->ms[bph][L] : NONE;
        pay = v ? sc->pay[bph][L] : -1;
        warp_lexmin(hi, lo, tie, ms, pay);
        bph ^= 1;
    }
    // block_lexmin and two block sums in one shared-memory round (one barrier).
    MSG_DI void block_lexmin_sums(unsigned& hi, unsigned& lo, unsigned& tie, unsigned& ms, int& pay, unsigned& c0,
                                  unsigned& c1) {
        warp_lexmin(hi, lo, tie, ms, pay);
        c0 = wp::radd(c0);
        c1 = wp::radd(c1);
        if (L == 0) {
            sc->hi[bph][W] = hi;
            sc->lo[bph][W] = lo;
            sc->tie[bph][W] = tie;
            sc->ms[bph][W] = ms;
            sc->pay[bph][W] = pay;
            sc->nl[bph][W] = c0;
            sc->nb[bph][W] = c1;
        }
        wp::bsync();
        const bool v = L < w;
        hi = v ? sc->hi[bph][L] : NONE;
        lo = v ? sc->lo[bph][L] : NONE;
        tie = v ? sc->tie[bph][L] : NONE;
        ms = v ? sc->ms[bph][L] : NONE;
        pay = v ? sc->pay[bph][L] : -1;
        c0 = wp::radd(v ? sc->nl[bph][L] : 0u);
        c1 = wp::radd(v ? sc->nb[bph][L] : 0u);
        warp_lexmin(hi, lo, tie, ms, pay);
        bph ^= 1;
    }
    MSG_DI unsigned block_sum(unsigned x) {
        x = wp::radd(x);
        if (L == 0) sc->sum[bph][W] = x;
        wp::bsync();
        x = wp::radd(L < w ? sc->sum[bph][L] : 0u);
        bph ^= 1;
        return x;
    }

    // ----------------------------------------------------------- exchange
    MSG_DI static XRec xnone() { return cl_xnone(); }

    // Cluster-wide reduction of one record per shard (see the header).  The
    // caller passes a block-uniform record; every thread of every shard
    // returns the same reduced record.  Deferred timeline samples ride along.
    MSG_DI void exchange(XRec& r) {
        if (NS == 1) return;
#ifdef MSG_PHASE_PROF
        const int ph_saved = ph_cur;
        MSG_PH(2);
#endif
        wp::sync();  // warp 0's lanes see thread 0's deferred samples
        r.ks[0] = npend > 0 ? sc->pend_k[0] : 0ull;
        r.ks[1] = npend > 1 ? sc->pend_k[1] : 0ull;
        const unsigned par = xround & 1u, use = xround >> 1;
        if (S > 1) {  // level 1: the CTAs of this cluster, over distributed shared memory
            if (W == 0) {
                // lane k pushes this shard's record into CTA k's inbox slot [par][sh]
                if (L == 0) wp::xbar_arm(&sc->xbar[par], S * (unsigned)sizeof(XRec));
                if (L < S)
                    wp::xpush(&sc->xin[par][sh], reinterpret_cast<const uint4*>(&r), (int)(sizeof(XRec) / 16), L,
                              &sc->xbar[par]);
                wp::xwait(&sc->xbar[par], use, S);
                cl_xreduce(sc->xin[par], S, &sc->xr);
            }
            wp::bsync();
            r = sc->xr;
        }
        if (D > 1) {  // level 2: CTA sh of every device group, over (peer) global memory
            if (W == 0) {
                const uint64_t stamp = ((uint64_t)epoch << 32) | (xround + 1u);
                if (L < D) {  // push the group's record to group L, then its stamp (release)
                    XInbox* dst = sc->ib[L];
                    uint4* q = reinterpret_cast<uint4*>(&dst->rec[par][sh][dv]);
                    const uint4* src = reinterpret_cast<const uint4*>(&r);
                    for (int i = 0; i < (int)(sizeof(XRec) / 16); ++i) q[i] = src[i];
                    wp::st_release_sys(&dst->stamp[par][sh][dv], stamp);
                }
                XInbox* me = sc->ib[dv];
                if (L < D) {
                    const uint64_t t0 = wp::gtime_ns();
                    unsigned spins = 0;
                    while (wp::ld_acquire_sys(&me->stamp[par][sh][L]) != stamp) {
                        wp::spin_pause();
                        if ((++spins & 1023u) == 0 && wp::gtime_ns() - t0 > 30000000000ull) wp::fail_stop();
                    }
                }
                cl_xreduce(me->rec[par][sh], D, &sc->xr2);
            }
            wp::bsync();
            r = sc->xr2;
        }
        ++xround;
        // deferred timeline samples, in order
        for (uint32_t i = 0; i < npend; ++i) record_sample(sc->pend_t[i], r.ks[i]);
        npend = 0;
#ifdef MSG_PHASE_PROF
        MSG_PH(ph_saved);
#endif
    }

    // --------------------------------------------------------------- events
    // Only the shard that owns an event emits (and counts) it; replicated
    // events belong to shard 0.
    MSG_DI void emit(uint8_t kind, int32_t jb, unsigned gpu, unsigned gpu2, unsigned pr, unsigned start,
                     unsigned start2, unsigned flags, uint64_t aux) {
        if (DETAIL && (oflags & OF_EVENTS) && n_ev < ev_cap && T == 0) {
            EventRec r;
            r.t = now;
            r.aux = aux;
            r.job = jb;
            r.gpu = (uint16_t)gpu;
            r.gpu2 = (uint16_t)gpu2;
            r.kind = kind;
            r.profile = (uint8_t)pr;
            r.start = (uint8_t)start;
            r.start2 = (uint8_t)start2;
            r.flags = (uint8_t)flags;
            r.pad[0] = r.pad[1] = r.pad[2] = 0;
            evs[n_ev] = r;
        }
        ++n_ev;
    }

    // ---------------------------------------------------------------- setup
    // gpu_smem: dynamic shared memory for the owned GPUs — 9 B per GPU (mask
    // words, cost ids), plus 96 B per GPU for its 8 slots when slots_smem —
    // or nullptr (everything global).
#ifdef MSG_PHASE_PROF
    long long ph_t = 0;
    int ph_cur = 0;
    MSG_DI void ph_mark(int k) {
        if (T == 0 && sh == 0 && gs == 0) {
            const long long c = clock64();
            if (ph_t) atomicAdd(&g_phase[ph_cur], (unsigned long long)(c - ph_t));
            ph_t = c;
            if (k == 2) atomicAdd(&g_phase[8], 1ull);
        }
        ph_cur = k;
    }
#endif
    MSG_DI void setup(const SimArgs& a, const DevTables* tables, BlockScratch* scratch, unsigned char* gpu_smem,
                      bool slots_smem, uint32_t t) {
        T = wp::tid();
        L = wp::lane();
        W = T >> 5;
        NT = wp::nthreads();
        w = NT >> 5;
        bph = 0;
        sc = scratch;
        tb = tables;
        stab = a.score_tab;
        S = wp::cluster_size();
        sh = wp::cluster_rank();
        D = a.n_dev < 1 ? 1u : a.n_dev;
        const unsigned vd = a.vdev < 1 ? 1u : a.vdev;
        dv = a.dev0 + (wp::cluster_id() % vd);
        gs = dv * S + sh;
        NS = D * S;
        epoch = a.epoch;
        // inbox of group k for this trace: a.inbox[k] holds one XInbox per large trace
        if (T < D) sc->ib[T] = reinterpret_cast<XInbox*>(a.inbox[T]) + wp::cluster_id() / vd;
        xround = 0;
        npend = 0;
        dep_g = -1;
        dep_w = 0;
        spec = false;
        const DevTrace tr = a.traces[t];
        const DevConfig c = a.configs[tr.cfg];
        G = c.G;
        g_lo = (int)((uint64_t)G * gs / NS);
        g_hi = (int)((uint64_t)G * (gs + 1) / NS);
        const uint64_t go = tr.cl_goff, so = 8 * go;
        st = a.c_st + so;
        prof = a.c_prof + so;
        mig = a.c_mig + so;
        cseq = a.c_cseq + so;
        apos = a.c_apos + so;
        const uint64_t ao = so + 8ull * (uint64_t)g_lo;  // this shard's active-list arena (8 per owned GPU)
        aslot = a.c_aslot + ao;
        ast = a.c_ast + ao;
        ajob = a.c_ajob + ao;
        amseq = a.c_amseq + ao;
        arem = a.c_arem + ao;
        atkey = a.c_atkey + ao;
        const int ng = g_hi - g_lo;
        if (gpu_smem) {
            unsigned char* p = gpu_smem;
            gw = reinterpret_cast<uint32_t*>(p);
            p += 4 * ng;
            gx = reinterpret_cast<uint32_t*>(p);
            p += 4 * ng;
            if (slots_smem) {  // indexed by global slot: bases offset by the shard's first slot
                const int s0 = 8 * g_lo;
                apos = reinterpret_cast<int32_t*>(p) - s0;
                p += 32 * ng;
                cseq = reinterpret_cast<uint32_t*>(p) - s0;
                p += 32 * ng;
                mig = reinterpret_cast<uint16_t*>(p) - s0;
                p += 16 * ng;
                st = p - s0;
                p += 8 * ng;
                prof = p - s0;
                p += 8 * ng;
            }
            gcid = p;
        } else {
            gw = a.c_gw + go + g_lo;
            gx = a.c_gx + go + g_lo;
            gcid = a.c_gcid + go + g_lo;
        }
        N = tr.n_jobs;
        arr = a.arrival + tr.job_off;
        svc = a.service + tr.job_off;
        prf = a.profile + tr.job_off;
        perm = tr.has_perm ? a.perm + tr.job_off : nullptr;
        queue = a.queue + tr.job_off;
        jobs = a.jobs + tr.job_off;
        evs = a.events ? a.events + tr.ev_off : nullptr;
        tl = a.timeline ? a.timeline + 2 * tr.tl_off : nullptr;
        ev_cap = tr.ev_cap;
        tl_cap = tr.tl_cap;
        oflags = a.out_flags;
        if (!evs) oflags &= ~OF_EVENTS;
        if (!tl) oflags &= ~OF_TIMELINE;
        cflags = c.flags;
        lazymask = c.lazymask;
        alpha = c.alpha;
        overlap = c.overlap;
        latency = c.latency;
        inv_g = ((G & (G - 1)) == 0) ? 1.0 / (double)G : 0.0;
        now = t_prev = 0.0;
        a_idx = 0;
        q_head = q_tail = 0;
        n_act = 0;
        n_ev = n_handler = n_tl = n_mig = n_reconf = n_enq = n_deq = 0;
        max_arr = max_intra = max_inter = 0;
        tl_sum = tl_mean = 0.0;
        tl_dirty = true;
        for (uint64_t i = 8ull * g_lo + T; i < 8ull * g_hi; i += NT) {
            st[i] = ST_EMPTY;
            mig[i] = 0;
            apos[i] = -1;
        }
        // empty GPU: masks 0, cost id of frag 0 (every profile fully feasible)
        const uint8_t empty_id = tb->cost4pair[tb->idealid[0] * 32u + tb->feasid[0]];
        for (int g = (int)T; g < ng; g += (int)NT) {
            gw[g] = 0;
            gx[g] = 0;
            gcid[g] = empty_id;
        }
        if (T < 7) sc->f[T] = wp::dadd(1.0, wp::dmul(alpha, (double)(int)T));  // slowdown(T+1)
        if (T == 0) sc->ksum = (unsigned long long)tb->cost4k[empty_id] * (unsigned long long)ng;
        if (S > 1) {  // exchange barriers live before any shard pushes
            if (T == 0) {
                wp::xbar_init(&sc->xbar[0]);
                wp::xbar_init(&sc->xbar[1]);
            }
            wp::cluster_sync();
        }
        wp::bsync();
        // static layout (sim.cpp:86-95), owned instances
        if (T == 0) {
            for (uint32_t k = 0; k < c.n_init; ++k) {
                const uint32_t v = a.init_slots[c.init_off + k];
                const int slot = (int)(v & 0xFFFFFFu);
                if (!own(slot >> 3)) continue;
                st[slot] = ST_IDLE;
                prof[slot] = (uint8_t)(v >> 24);
                cseq[slot] = k;
            }
            for (uint32_t k = 0; k < c.n_init; ++k) {
                const int g = (int)((a.init_slots[c.init_off + k] & 0xFFFFFFu) >> 3);
                if (own(g)) refresh_gpu(g);
            }
        }
        cseq_ctr = c.n_init;
        load_arrival();
        wp::bsync();
    }

    MSG_DI void load_arrival() {
        if (a_idx < N) {
            const uint32_t r = perm ? perm[a_idx] : a_idx;
            a_rank = r;
            a_t = arr[r];
            a_prof = prf[r];
            a_svc = svc[r];
        }
    }

    // ------------------------------------------- GPU words (single thread)
    // busy/blocked masks (gpu.cpp:10-48), running count, idle-exact
    // placements, 4-mask cost id; keeps the shard's integer cost total current.
    MSG_DI void refresh_gpu(int g) {
        const GpuWord r = cl_gpu_word(st + 8 * g, prof + 8 * g, tb);
        const int l = g - g_lo;
        gw[l] = r.w;
        gx[l] = r.x;
        sc->ksum += (unsigned long long)tb->cost4k[r.id] - (unsigned long long)tb->cost4k[gcid[l]];
        gcid[l] = (uint8_t)r.id;
    }

    // ------------------------------------------ active list (single thread)
    MSG_DI void act_add(uint32_t i, int slot, uint8_t s, int32_t jb, double r, double tk, uint32_t ms) {
        aslot[i] = slot;
        ast[i] = s;
        ajob[i] = jb;
        arem[i] = r;
        atkey[i] = tk;
        amseq[i] = ms;
        apos[slot] = (int32_t)i;
    }
    MSG_DI void act_remove(int slot, uint32_t n) {  // n = list size before removal
        const int i = apos[slot];
        const uint32_t last = n - 1;
        if ((uint32_t)i != last) {
            const int ls = aslot[last];
            aslot[i] = ls;
            ast[i] = ast[last];
            ajob[i] = ajob[last];
            arem[i] = arem[last];
            atkey[i] = atkey[last];
            amseq[i] = amseq[last];
            apos[ls] = i;
        }
        apos[slot] = -1;
    }

    // ---------------------------------------------------- contention model
    MSG_DI void advance_all() {  // sim.cpp:153-165 (uniform dt, see engine_core.cuh)
        const double dt = wp::dsub(now, t_prev);
        t_prev = now;
        if (!(dt > 0.0)) return;
        // dt / slowdown(k): lane k-1 of every warp, fetched by shuffle
        const double q = L < 7 ? cl_ddiv(dt, sc->f[L]) : 0.0;
#pragma unroll
        for (int h = 0; h < kHeld; ++h) {
            const uint32_t i = T + (uint32_t)h * NT;
            const unsigned k = i < n_act ? held_k[h] : 0u;
            const double qk = wp::shfl(q, k ? (int)k - 1 : 0);
            if (k) arem[i] = wp::dsub(held_rem[h], qk);
        }
        if (n_act <= (uint32_t)kHeld * NT) return;
        if (W == 0 && L < 7) sc->q[L] = q;
        wp::bsync();
#pragma unroll 4
        for (uint32_t i = T + (uint32_t)kHeld * NT; i < n_act; i += NT)
            if (ast[i] == ST_RUN) arem[i] = wp::dsub(arem[i], sc->q[w_k(W_(aslot[i] >> 3)) - 1]);
        // no trailing barrier: every reader of arem starts with one, and
        // the next timer scan revisits entry i on the same thread
    }

    // A deferred sample (sharded engine): its mean and the running sum are
    // kept by one thread of the last warp only (finish reads them back), off
    // warp 0, which runs the exchanges and the owner's serial steps.
    MSG_DI void record_sample(double t, unsigned long long ktot) {
        if (T == NT - 1) {
            tl_mean = cl_tl_mean(ktot, inv_g, G);
            if (DETAIL && (oflags & OF_TIMELINE) && n_tl < tl_cap && gs == 0) {
                tl[2 * n_tl] = t;
                tl[2 * n_tl + 1] = tl_mean;
            }
            tl_sum = wp::dadd(tl_sum, tl_mean);
        }
        ++n_tl;
    }

    MSG_DI void sample() {  // sim.cpp:177-181
        if (NS > 1) {  // deferred: the next exchange sums the shards' parts
            if (T == 0) {  // thread 0 also keeps ksum (refresh_gpu): no barrier needed here
                sc->pend_t[npend] = now;
                sc->pend_k[npend] = sc->ksum;
            }
            ++npend;
            return;
        }
        if (tl_dirty) {
            wp::bsync();
            if (T == 0) {
                if (G <= kExactTimelineGpus) {
                    double tot = 0.0;
                    for (int g = 0; g < G; ++g) tot = wp::dadd(tot, tb->cost4val[gcid[g]]);
                    sc->tl = inv_g != 0.0 ? wp::dmul(tot, inv_g) : wp::ddiv(tot, (double)G);
                } else {
                    const double tot = wp::ddiv((double)sc->ksum, 25200.0);
                    sc->tl = inv_g != 0.0 ? wp::dmul(tot, inv_g) : wp::ddiv(tot, (double)G);
                }
            }
            wp::bsync();
            tl_mean = sc->tl;
            tl_dirty = false;
        }
        if (DETAIL && (oflags & OF_TIMELINE) && n_tl < tl_cap && T == 0) {
            tl[2 * n_tl] = now;
            tl[2 * n_tl + 1] = tl_mean;
        }
        ++n_tl;
        tl_sum = wp::dadd(tl_sum, tl_mean);
    }

    // --------------------------------------------------------- next event
    // reschedule_completions (sim.cpp:167-175: every Running job's
    // prediction now + max(rem,0)*f) fused with the scan for the next timer.
    // Returns the kind (-1 none, 0 completion, 1 migration end, 2 service
    // start, 3 arrival); for slot timers `slot` is the global slot and
    // `ev_i` its index in this shard's active list (-1 on other shards).
    MSG_DI int next_event(int& slot, int& ev_i) {
        wp::bsync();
        unsigned bhi = NONE, blo = NONE, btie = NONE, bms = NONE;
        int bi = -1;
        // This thread's first kHeld entries keep (remaining work, running
        // count) in registers for advance_all (nothing changes them between
        // the scan and the advance): its update needs no reload, no barrier.
#pragma unroll kC4ScanUnroll
        for (uint32_t i = T, j = 0; i < n_act; i += NT, ++j) {
            const uint8_t s = ast[i];
            double t;
            if (s == ST_RUN) {
                const double r0 = arem[i];
                const unsigned k = w_k(W_(aslot[i] >> 3));
                const double r = r0 < 0.0 ? 0.0 : r0;
                t = wp::dadd(now, wp::dmul(r, sc->f[k - 1]));
                atkey[i] = t;
#pragma unroll
                for (int h = 0; h < kHeld; ++h)
                    if (j == (uint32_t)h) held_rem[h] = r0, held_k[h] = k;
            } else {
                t = atkey[i];
#pragma unroll
                for (int h = 0; h < kHeld; ++h)
                    if (j == (uint32_t)h) held_k[h] = 0;
            }
            const uint64_t tk = time_key(t);
            const unsigned hi = (unsigned)(tk >> 32), lo = (unsigned)tk;
            const unsigned kind = s == ST_RUN ? 0u : (s == ST_DRAIN ? 1u : 2u);
            const unsigned tie = (kind << 28) | (unsigned)ajob[i];
            const unsigned ms = s == ST_DRAIN ? amseq[i] : 0u;
            const bool better =
                hi < bhi || (hi == bhi && (lo < blo || (lo == blo && (tie < btie || (tie == btie && ms < bms)))));
            if (better) {
                bhi = hi;
                blo = lo;
                btie = tie;
                bms = ms;
                bi = (int)i;
            }
        }
        // The pending arrival's placement search rides in the next-event
        // exchange when it would dispatch at once (empty queue): the masks
        // it reads do not change before handle_arrival.  Its scan shares the
        // timer scan's pass and block reduction (one barrier for both).
        spec = NS > 1 && a_idx < N && q_head == q_tail;
        uint64_t skey = ~0ull;
        unsigned snl = 0, snb = 0;
        if (spec) {
            MSG_PH(1);
            scan_dispatch(a_prof, skey, snl, snb);
            MSG_PH(0);
            warp_lexmin(bhi, blo, btie, bms, bi);
            const unsigned kh = wp::rmin((unsigned)(skey >> 32));
            const unsigned kl = wp::rmin((unsigned)(skey >> 32) == kh ? (unsigned)skey : NONE);
            snl = wp::radd(snl);
            snb = wp::radd(snb);
            if (L == 0) {
                sc->hi[bph][W] = bhi;
                sc->lo[bph][W] = blo;
                sc->tie[bph][W] = btie;
                sc->ms[bph][W] = bms;
                sc->pay[bph][W] = bi;
                sc->kh[bph][W] = kh;
                sc->kl[bph][W] = kl;
                sc->nl[bph][W] = snl;
                sc->nb[bph][W] = snb;
            }
            wp::bsync();
            const bool v = L < w;
            bhi = v ? sc->hi[bph][L] : NONE;
            blo = v ? sc->lo[bph][L] : NONE;
            btie = v ? sc->tie[bph][L] : NONE;
            bms = v ? sc->ms[bph][L] : NONE;
            bi = v ? sc->pay[bph][L] : -1;
            const unsigned h2 = v ? sc->kh[bph][L] : NONE, l2 = v ? sc->kl[bph][L] : NONE;
            snl = wp::radd(v ? sc->nl[bph][L] : 0u);
            snb = wp::radd(v ? sc->nb[bph][L] : 0u);
            bph ^= 1;
            warp_lexmin(bhi, blo, btie, bms, bi);
            const unsigned mh = wp::rmin(h2);
            const unsigned ml = wp::rmin(h2 == mh ? l2 : NONE);
            skey = ((uint64_t)mh << 32) | ml;
            if (!(cflags & CF_LB)) snl = snb = 0;
        } else {
            block_lexmin(bhi, blo, btie, bms, bi);
        }
        double tmin = 0.0;
        slot = -1;
        unsigned winfo = 0;
        if (bhi != NONE) {
            tmin = atkey[bi];
            slot = aslot[bi];
            winfo = (W_(slot >> 3) & 0x0FFFFFFFu) | ((unsigned)prof[slot] << 28);  // GPU word | slot profile
        }
        if (NS > 1) {
            XRec r = xnone();
            if (spec) {
                r.pad2 = skey;
                r.c[0] = snl;
                r.c[1] = snb;
            }
            r.hi = bhi;
            r.lo = blo;
            r.tie = btie;
            r.ms = bms;
            r.slot = slot;
            r.tkey = tmin;
            r.info = winfo;
            exchange(r);
            if (spec) {
                spec_key = r.pad2;
                spec_nl = r.c[0];
                spec_nb = r.c[1];
            }
            bhi = r.hi;
            blo = r.lo;
            btie = r.tie;
            slot = r.slot;
            tmin = r.tkey;
            winfo = r.info;
        }
        const bool have_arrival = a_idx < N;
        ev_i = -1;
        if (bhi == NONE) {
            if (!have_arrival) return -1;
            now = a_t;
            return 3;
        }
        if (have_arrival && time_key(a_t) < (((uint64_t)bhi << 32) | blo)) {
            now = a_t;
            return 3;
        }
        if (own(slot >> 3)) ev_i = apos[slot];
        now = tmin;
        if ((btie >> 28) == 0u) {  // a completion: its GPU's word once the slot is idle (gpu.cpp:113-125)
            const int q = (int)(winfo >> 28), s0 = slot & 7;
            const unsigned m = fpm(q, s0);
            dep_g = slot >> 3;
            dep_w = (winfo & ~(fpc(q, s0) | (m << 8) | (m << 16))) & 0x00FFFFFFu;
        }
        return (int)(btie >> 28);
    }

    // ------------------------------------------------------------ schedule
    // This shard's candidates for a job of profile p (scheduler.cpp:47-104):
    // the block-wide minimum packed key and the Lazy / Busy candidate counts.
    MSG_DI void local_dispatch(int p, uint64_t& key, unsigned& NL, unsigned& NB) {
        wp::bsync();
        uint64_t kmin;
        unsigned nl, nb;
        scan_dispatch(p, kmin, nl, nb);
        unsigned hi = (unsigned)(kmin >> 32), lo = (unsigned)kmin, z0 = 0, z1 = 0;
        int pay = 0;
#if C4_FUSED_SUMS
        block_lexmin_sums(hi, lo, z0, z1, pay, nl, nb);
        NL = (cflags & CF_LB) ? nl : 0u;
        NB = (cflags & CF_LB) ? nb : 0u;
#else
        block_lexmin(hi, lo, z0, z1, pay);
        NL = NB = 0;
        if (cflags & CF_LB) {
            const unsigned x = block_sum(nl | (nb << 16));
            NL = x & 0xFFFFu;
            NB = x >> 16;
        }
#endif
        key = ((uint64_t)hi << 32) | lo;
    }

    // This thread's part of local_dispatch: its GPUs' minimum key and
    // Lazy / Busy candidate counts (no barrier).
    MSG_DI void scan_dispatch(int p, uint64_t& kmin_out, unsigned& nl_out, unsigned& nb_out) {
        const unsigned n = count_of(p), stride = stride_of(p);
        const unsigned pb = pidx(p, 0);
        const bool dyn = (cflags & CF_DYN) != 0;
        const bool lb = (cflags & CF_LB) != 0;
        uint64_t kmin = ~0ull;
        unsigned nl = 0, nb = 0;
        // With load balancing and dynamic partitioning, a GPU without a
        // draining instance (blocked memory == busy memory) is scored by one
        // lookup in the scorer's per-word table (score.cu: lowest
        // post-placement rank, the starts reaching it, the candidate count);
        // the rest take the per-start loop below.
        const uint16_t* Tp = (lb && dyn && stab) ? stab + p * 2048 : nullptr;
#pragma unroll kC4DispatchUnroll
        for (int g = g_lo + (int)T; g < g_hi; g += (int)NT) {
            if (Tp) {
                const unsigned wd = gw[g - g_lo];
                const unsigned bm = w_bm(wd);
                if (w_km(wd) == bm) {
                    const unsigned pc = (unsigned)wp::popc(w_bc(wd));
                    const unsigned e = Tp[pc * 256u + bm];
                    const unsigned cnt = e & 7u;
                    const unsigned lazy = (lazymask >> pc) & 1u;
                    const unsigned mm = (e >> 3) & 0x7Fu, r = mm & (gx[g - g_lo] >> pb);
                    const unsigned j = (unsigned)wp::ffs(r ? r : mm) - 1u;
                    const uint64_t k = ((uint64_t)(lazy ^ 1u) << 47) | ((uint64_t)(e >> 10) << 42) |
                                       ((uint64_t)(r ? 0u : 1u) << 41) | ((uint64_t)g << 3) | (uint64_t)(j * stride);
                    kmin = cnt && k < kmin ? k : kmin;
                    nl += lazy ? cnt : 0u;
                    nb += lazy ? 0u : cnt;
                    continue;
                }
            }
            const unsigned wd = gw[g - g_lo];
            const unsigned ex = gx[g - g_lo] >> pb;
            const unsigned lazy = (lazymask >> wp::popc(w_bc(wd))) & 1u;
            for (unsigned j = 0; j < n; ++j) {
                const int s = (int)(j * stride);
                const bool exact = (ex >> j) & 1u;
                if ((dyn || exact) && !(fpm(p, s) & w_km(wd))) {
                    uint64_t k;
                    if (lb) {
                        const unsigned rk = rank2(w_bc(wd) | fpc(p, s), w_bm(wd) | fpm(p, s));
                        k = ((uint64_t)(lazy ^ 1u) << 47) | ((uint64_t)rk << 42) | ((uint64_t)(exact ? 0u : 1u) << 41) |
                            ((uint64_t)g << 3) | (uint64_t)s;
                        nl += lazy;
                        nb += lazy ^ 1u;
                    } else {
                        k = ((uint64_t)g << 3) | (uint64_t)s;
                    }
                    kmin = k < kmin ? k : kmin;
                }
            }
        }
        kmin_out = kmin;
        nl_out = nl;
        nb_out = nb;
    }

    // The decision from the global minimum key and counts.
    MSG_DI Decision decide(int p, uint64_t k, unsigned NL, unsigned NB) {
        const bool lb = (cflags & CF_LB) != 0;
        Decision d;
        d.placed = k != ~0ull;
        d.evals = lb ? NL + (NL == 0 ? NB : 0u) : 0u;
        d.g = (int)((k >> 3) & 0x3FFFFFFFFull);
        d.s = (int)(k & 7u);
        d.reused = false;
        if (d.placed) {
            if (lb) d.reused = ((k >> 41) & 1u) == 0;
            else if (own(d.g)) d.reused = (gx[d.g - g_lo] >> pidx(p, d.s)) & 1u;
        }
        return d;
    }

    MSG_DI Decision dispatch(int p) {  // scheduler.cpp:47-104
        uint64_t k;
        unsigned NL, NB;
        local_dispatch(p, k, NL, NB);
        if (NS > 1) {
            XRec r = xnone();
            r.hi = (unsigned)(k >> 32);
            r.lo = (unsigned)k;
            r.tie = r.ms = 0;
            r.c[0] = NL;
            r.c[1] = NB;
            exchange(r);
            k = ((uint64_t)r.hi << 32) | r.lo;
            NL = r.c[0];
            NB = r.c[1];
        }
        return decide(p, k, NL, NB);
    }

    // ---------------------------------------------------- create_instance
    // gpu.cpp:71-101 on one thread of the GPU's owner; destroyed instances
    // are listed in creation order for the Reconfig events.
    MSG_DI CreateRes create(int g, int p, int s) {
        wp::bsync();
        if (T == 0) {
            const int b = 8 * g;
            const bool reused = st[b + s] == ST_IDLE && prof[b + s] == p;
            unsigned dmask = 0;
            int nd = 0;
            if (!reused) {
                for (int t = 0; t < 8; ++t) {
                    if (st[b + t] == ST_IDLE && (fpm(prof[b + t], t) & fpm(p, s))) {
                        dmask |= 1u << t;
                        int i = nd++;  // insertion by creation sequence
                        while (i > 0 && cseq[b + sc->dl_slot[i - 1]] > cseq[b + t]) {
                            sc->dl_slot[i] = sc->dl_slot[i - 1];
                            sc->dl_prof[i] = sc->dl_prof[i - 1];
                            --i;
                        }
                        sc->dl_slot[i] = t;
                        sc->dl_prof[i] = prof[b + t];
                    }
                }
                for (int t = 0; t < 8; ++t)
                    if ((dmask >> t) & 1u) st[b + t] = ST_EMPTY;
                prof[b + s] = (uint8_t)p;
                cseq[b + s] = cseq_ctr;
            }
            st[b + s] = ST_RUN;  // placeholder, the caller binds the job
            sc->u[0] = reused;
            sc->u[1] = dmask;
        }
        wp::bsync();
        CreateRes cr;
        cr.reused = sc->u[0] != 0;
        cr.dmask = sc->u[1];
        cr.dprof = 0;
        cr.dseq = 0;
        if (!cr.reused) ++cseq_ctr;
        // no trailing barrier: sc->u is next written by thread 0 after the
        // leading barrier of a later create_instance
#if !C4_DROP_BARRIERS
        wp::bsync();
#endif
        return cr;
    }

    MSG_DI void emit_reconfig(int g, int p, int s, const CreateRes& cr) {
        const int nd = wp::popc(cr.dmask);
        for (int i = 0; i < nd; ++i) {
            emit(EV_RECONFIG, -1, (unsigned)g, 0, (unsigned)sc->dl_prof[i], (unsigned)sc->dl_slot[i], 0, EF_DESTROY, 0);
            ++n_reconf;
        }
        if (!cr.reused) {
            emit(EV_RECONFIG, -1, (unsigned)g, 0, (unsigned)p, (unsigned)s, 0, 0, 0);
            ++n_reconf;
        }
    }

    MSG_DI double apply_placement(int g, int s, int32_t r, double sv, unsigned nops) {  // sim.cpp:199-218
        const double delay = wp::dmul((double)nops, latency);
        const double ss = wp::dadd(now, delay);
        const int slot = 8 * g + s;
        if (T == 0) {
            const uint8_t v = delay > 0.0 ? ST_WAIT : ST_RUN;
            st[slot] = v;
            mig[slot] = 0;
            act_add(n_act, slot, v, r, sv, ss, 0);
            jobs[r].sched = ss;
            refresh_gpu(g);
        }
        ++n_act;
        tl_dirty = true;
        wp::bsync();
        return ss;
    }

    // The decided placement, on the GPU's owner only.
    MSG_DI void place(const Decision& d, int32_t r, int p, double sv, uint8_t kind) {
        if (d.g == dep_g) {  // every shard follows the departed GPU's masks (create_instance never
            const unsigned m = fpm(p, d.s);  // touches busy masks of other instances)
            dep_w |= fpc(p, d.s) | (m << 8) | (m << 16);
        }
        if (!own(d.g)) return;
        const CreateRes cr = create(d.g, p, d.s);
        const unsigned nops = (unsigned)wp::popc(cr.dmask) + (cr.reused ? 0u : 1u);
        const double ss = apply_placement(d.g, d.s, r, sv, nops);
        emit(kind, r, (unsigned)d.g, 0, (unsigned)p, (unsigned)d.s, 0, EF_PLACED | (cr.reused ? EF_REUSED : 0),
             wp::dbits(ss));
        emit_reconfig(d.g, p, d.s, cr);
    }

    MSG_DI void dequeue_pass() {  // sim.cpp:325-344
        while (q_head < q_tail) {
            wp::bsync();
            const int32_t h = queue[q_head];
            const int p = prf[h];
            const double sv = svc[h];
            const Decision d = dispatch(p);
            if (!d.placed) break;
            max_arr = max_arr > (int)d.evals ? max_arr : (int)d.evals;
            ++q_head;
            place(d, h, p, sv, EV_DEQUEUE);
            ++n_deq;
        }
    }

    // ------------------------------------------------------------ migration
    // apply_move (migration.cpp:35-69) within one GPU (plan_intra, owner
    // only): the job keeps its active entry (its remaining work and timer
    // move with it); with overlap > 0 the source slot gets a new entry
    // carrying its MigrationEnd timer.
    MSG_DI void apply_move_intra(int from_slot, int ts) {
        wp::bsync();
        const int g = from_slot >> 3, fs = from_slot & 7;
        const int q = prof[from_slot];
        const int ia = apos[from_slot];
        const int32_t r = ajob[ia];
        const unsigned jmig = mig[from_slot];
        const uint8_t jst = st[from_slot];
        const unsigned cb = k2w(W_(g));
        wp::bsync();
        if (T == 0) st[from_slot] = ST_DRAIN;  // start_draining
        const CreateRes cr = create(g, q, ts);
        if (T == 0) {
            const int dst = 8 * g + ts;
            st[dst] = jst;
            mig[dst] = (uint16_t)(jmig + 1u);
            aslot[ia] = dst;  // the job's entry follows it
            apos[dst] = ia;
            apos[from_slot] = -1;
            if (overlap <= 0.0) {
                st[from_slot] = ST_IDLE;
            } else {
                act_add(n_act, from_slot, ST_DRAIN, r, 0.0, wp::dadd(now, overlap), jmig);
            }
            refresh_gpu(g);
        }
        if (overlap > 0.0) ++n_act;
        tl_dirty = true;
        wp::bsync();
        const unsigned ca = k2w(W_(g));
        const uint64_t costs = (uint64_t)cb | ((uint64_t)ca << 16) | ((uint64_t)cb << 32) | ((uint64_t)ca << 48);
        emit(EV_MIGRATION_START, r, (unsigned)g, (unsigned)g, (unsigned)q, (unsigned)fs, (unsigned)ts, 0, costs);
        ++n_mig;
        emit_reconfig(g, q, ts, cr);
        if (overlap <= 0.0) emit(EV_MIGRATION_END, r, (unsigned)g, 0, 0, 0, 0, 0, 0);
    }

    // apply_move of plan_inter: the source side on the source GPU's owner,
    // the destination side on the lazy GPU's owner, from the exchanged
    // record of the winning source (x).  The job's active entry moves with
    // it: removed at the source (which, with overlap > 0, gets a draining
    // entry instead) and re-added at the destination.
    MSG_DI void apply_move_inter(const XRec& x, int tg, int ts) {
        wp::bsync();
        const int from_slot = x.slot;
        const int fg = from_slot >> 3, fs = from_slot & 7;
        const uint8_t jst = (uint8_t)(x.info & 0xFFu);
        const int q = (int)((x.info >> 8) & 0xFFu);
        const unsigned jmig = x.info >> 16;
        const int32_t r = x.job;
        const bool src = own(fg), dst_own = own(tg);
        unsigned fcb = 0, fca = 0, tcb = 0, tca = 0;
        if (src) {
            fcb = k2w(W_(fg));
            wp::bsync();
            if (T == 0) {
                act_remove(from_slot, n_act);
                if (overlap <= 0.0) {
                    st[from_slot] = ST_IDLE;
                } else {
                    st[from_slot] = ST_DRAIN;
                    act_add(n_act - 1, from_slot, ST_DRAIN, r, 0.0, wp::dadd(now, overlap), jmig);
                }
                refresh_gpu(fg);
            }
            if (overlap <= 0.0) --n_act;
            wp::bsync();
            fca = k2w(W_(fg));
        }
        if (dst_own) {
            tcb = k2w(W_(tg));
            const CreateRes cr = create(tg, q, ts);
            if (T == 0) {
                const int dst = 8 * tg + ts;
                st[dst] = jst;
                mig[dst] = (uint16_t)(jmig + 1u);
                act_add(n_act, dst, jst, r, x.rem, x.tkey, 0);
                refresh_gpu(tg);
            }
            ++n_act;
            wp::bsync();
            tca = k2w(W_(tg));
            if (NS == 1) {  // both sides are here: the event log carries all four costs
                const uint64_t costs =
                    (uint64_t)fcb | ((uint64_t)fca << 16) | ((uint64_t)tcb << 32) | ((uint64_t)tca << 48);
                emit(EV_MIGRATION_START, r, (unsigned)fg, (unsigned)tg, (unsigned)q, (unsigned)fs, (unsigned)ts,
                     EF_INTER, costs);
            } else {
                ++n_ev;  // counted; the sharded engine runs without the event log
            }
            ++n_mig;
            emit_reconfig(tg, q, ts, cr);
            if (overlap <= 0.0) emit(EV_MIGRATION_END, r, (unsigned)fg, 0, 0, 0, 0, 0, 0);
        }
        tl_dirty = true;
        wp::bsync();
    }

    MSG_DI void plan_intra(int g) {  // migration.cpp:71-123, on warp 0 of the owner
        for (;;) {
            wp::bsync();
            const unsigned wd = W_(g);
            const unsigned bc = w_bc(wd), bm = w_bm(wd), km = w_km(wd);
            const unsigned cur = rank2(bc, bm);
            if (W == 0) {
                const int own_s = (int)(L & 7u);
                const int sl = 8 * g + own_s;
                const uint8_t s = st[sl];
                unsigned kmin = NONE, cnt = 0;
                if (s == ST_RUN || s == ST_WAIT) {
                    const int q = prof[sl];
                    const unsigned r = (unsigned)ajob[apos[sl]];
                    const unsigned ofc = fpc(q, own_s), ofm = fpm(q, own_s);
                    const unsigned n = count_of(q), stride = stride_of(q);
                    for (int h = 0; h < 2; ++h) {
                        const unsigned j = (L >> 3) + 4u * (unsigned)h;
                        if (j < n) {
                            const int t = (int)(j * stride);
                            if (t != own_s && !(fpm(q, t) & km)) {
                                const unsigned rk = rank2((bc & ~ofc) | fpc(q, t), (bm & ~ofm) | fpm(q, t));
                                const unsigned key = (rk << 27) | (r << 3) | (unsigned)t;
                                kmin = key < kmin ? key : kmin;
                                ++cnt;
                            }
                        }
                    }
                }
                const unsigned best = wp::rmin(kmin);
                const unsigned evals = wp::radd(cnt);
                const int wl = wp::ffs(wp::ballot(kmin == best)) - 1;
                if (L == 0) {
                    sc->u[2] = best;
                    sc->u[3] = evals;
                    sc->u[4] = (unsigned)(wl & 7);
                }
            }
            wp::bsync();
            const unsigned best = sc->u[2];
            const int evals = (int)sc->u[3];
            const int from = (int)sc->u[4];
            max_intra = max_intra > evals ? max_intra : evals;
            wp::bsync();
            if (best == NONE || (best >> 27) >= cur) break;
            apply_move_intra(8 * g + from, (int)(best & 7u));
        }
    }

    // migration.cpp:125-210.  w0 = the lazy GPU's word, replicated in every
    // shard (exchanged by on_departure, then updated by every shard with the
    // same destination choice).
    MSG_DI void plan_inter(int g0, unsigned w0) {
        for (;;) {
            wp::bsync();
            const unsigned lazy_cs = (unsigned)wp::popc(w_bc(w0));
            const unsigned km0 = w_km(w0);
            const unsigned pl = tb->placeable[km0];
            unsigned bhi = NONE, blo = NONE, z0 = 0, z1 = 0, cnt = 0;
            int bi = -1;
            for (uint32_t i = T; i < n_act; i += NT) {
                const uint8_t v = ast[i];
                if (v != ST_RUN && v != ST_WAIT) continue;
                const int slot = aslot[i];
                const int g = slot >> 3, s = slot & 7;
                if (g == g0) continue;
                const unsigned wd = W_(g);
                const unsigned src_cs = (unsigned)wp::popc(w_bc(wd));
                if ((lazymask >> src_cs) & 1u) continue;  // source must be Busy
                const int q = prof[slot];
                const unsigned cs = cs_of(q);
                if (lazy_cs + cs < src_cs - cs && ((pl >> q) & 1u)) {
                    const unsigned rk = rank2(w_bc(wd) & ~fpc(q, s), w_bm(wd) & ~fpm(q, s));
                    // key (cost, gpu, job id): rank:5 | gpu:35 | job:24
                    const uint64_t key = ((uint64_t)rk << 59) | ((uint64_t)g << 24) | (uint64_t)ajob[i];
                    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
                    if (hi < bhi || (hi == bhi && lo < blo)) {
                        bhi = hi;
                        blo = lo;
                        bi = (int)i;
                    }
                    ++cnt;
                }
            }
#if C4_FUSED_SUMS
            unsigned zc = 0;
            block_lexmin_sums(bhi, blo, z0, z1, bi, cnt, zc);
#else
            block_lexmin(bhi, blo, z0, z1, bi);
            cnt = block_sum(cnt);
#endif
            XRec x = xnone();
            x.c[0] = cnt;
            x.hi = bhi;
            x.lo = blo;
            x.tie = x.ms = 0;
            if (bhi != NONE) {
                const int slot = aslot[bi];
                x.slot = slot;
                x.job = ajob[bi];
                x.info = (uint32_t)st[slot] | ((uint32_t)prof[slot] << 8) | ((uint32_t)mig[slot] << 16);
                x.rem = arem[bi];
                x.tkey = atkey[bi];
            }
            exchange(x);
            int evals = (int)x.c[0];
            if (x.hi == NONE) {
                max_inter = max_inter > evals ? max_inter : evals;
                break;
            }
            const int q = (int)((x.info >> 8) & 0xFFu);
            if (W == 0) {  // destination: minimum (cost, start) on g0, lane = start
                const bool cand = L < 8 && ((startmask_of(q) >> L) & 1u) && !(fpm(q, (int)L) & km0);
                const unsigned dk =
                    cand ? ((rank2(w_bc(w0) | fpc(q, (int)L), w_bm(w0) | fpm(q, (int)L)) << 3) | L) : NONE;
                const unsigned dbest = wp::rmin(dk);
                const unsigned dcnt = wp::radd(cand ? 1u : 0u);
                if (L == 0) {
                    sc->u[5] = dbest;
                    sc->u[6] = dcnt;
                }
            }
            wp::bsync();
            const int ts = (int)(sc->u[5] & 7u);
            evals += (int)sc->u[6];
            max_inter = max_inter > evals ? max_inter : evals;
            apply_move_inter(x, g0, ts);
            // the lazy GPU's word after create_instance (destroyed instances were idle)
            const unsigned m = fpm(q, ts);
            w0 = (w0 | fpc(q, ts) | (m << 8) | (m << 16)) + ((x.info & 0xFFu) == ST_RUN ? (1u << 24) : 0u);
        }
    }

    MSG_DI void on_departure(int g) {  // migration.cpp:212-220
        wp::bsync();
        // sharded: every shard tracked g's masks since the completion (the
        // running count, not needed here, is left out)
        const unsigned wd = NS > 1 ? dep_w : W_(g);
        if ((lazymask >> wp::popc(w_bc(wd))) & 1u) plan_inter(g, wd);
        else if (own(g)) plan_intra(g);
    }

    // ------------------------------------------------------------ handlers
    MSG_DI void handle_arrival() {
        const int32_t r = (int32_t)a_rank;
        const int p = a_prof;
        const double sv = a_svc;
        ++a_idx;
        load_arrival();
        bool enq = q_head < q_tail;
        if (!enq) {
            const Decision d = spec ? decide(p, spec_key, spec_nl, spec_nb) : dispatch(p);
            max_arr = max_arr > (int)d.evals ? max_arr : (int)d.evals;
            if (d.placed) place(d, r, p, sv, EV_ARRIVAL);
            else enq = true;
        }
        if (enq) {
            if (gs == 0) emit(EV_ARRIVAL, r, 0, 0, (unsigned)p, 0, 0, 0, 0);
            if (T == 0) queue[q_tail] = r;  // every shard keeps the same queue
            ++q_tail;
            if (gs == 0) emit(EV_ENQUEUE, r, 0, 0, 0, 0, 0, 0, 0);
            ++n_enq;
        }
    }

    MSG_DI void handle_departure(int slot, int ia, bool completion) {
        const int g = slot >> 3;
        if (own(g)) {
            wp::bsync();  // advance_all's stores before act_remove moves an entry
#if C4_DROP_BARRIERS
            int32_t r = -1;  // only thread 0 needs the job (records, emit)
            if (T == 0) {
                r = ajob[ia];
                const int m = mig[slot];
#else
            const int32_t r = ajob[ia];
            const int m = mig[slot];
            wp::bsync();
            if (T == 0) {
#endif
                st[slot] = ST_IDLE;
                act_remove(slot, n_act);
                if (completion) {
                    jobs[r].done = now;
                    jobs[r].gpu = g;
                    jobs[r].mig = m;
                }
                refresh_gpu(g);
            }
            --n_act;
            tl_dirty = true;
            wp::bsync();
            emit(completion ? EV_COMPLETION : EV_MIGRATION_END, r, (unsigned)g, 0, 0, 0, 0, 0, 0);
        }
        if (completion) sample();
        const int passes = (completion && (cflags & CF_MIG)) ? 2 : 1;
        for (int pass = 0; pass < passes; ++pass) {
            if (pass) on_departure(g);
            dequeue_pass();
        }
    }

    MSG_DI void handle_service_start(int slot, int ia) {
        if (!own(slot >> 3)) return;
        wp::bsync();
        if (T == 0) {
            st[slot] = ST_RUN;
            ast[ia] = ST_RUN;  // start_service: arem already holds service_s
            refresh_gpu(slot >> 3);
        }
        tl_dirty = true;
        wp::bsync();
    }

    MSG_DI void run() {
        for (;;) {
            int slot = -1, ia = -1;
            MSG_PH(0);
            const int kind = next_event(slot, ia);
            if (kind < 0) break;
            ++n_handler;
            MSG_PH(3);
            advance_all();
            MSG_PH(kind == 3 ? 4 : kind == 2 ? 6 : 5);
            if (kind == 3) handle_arrival();
            else if (kind == 2) handle_service_start(slot, ia);
            else handle_departure(slot, ia, kind == 0);
            MSG_PH(7);
            sample();  // the completions are rescheduled by the next scan
#ifdef MSG_PHASE_PROF
            if (T == 0 && sh == 0 && gs == 0) atomicAdd(&g_phase[9], 1ull);
#endif
        }
        MSG_PH(0);
    }

    MSG_DI void finish(DevSummary* out) {  // metrics (sim.cpp:414-502), warp 0 of shard 0
        wp::bsync();
        DevSummary s;
        s.status = q_head < q_tail ? STATUS_JOBS_PENDING : STATUS_OK;
        s.reserved = 0;
        s.pending_rank = -1;
        if (NS > 1) {  // flush the last samples, sum the owner-counted totals; job rows become visible
            if (D > 1) wp::gfence_sys();
            else wp::gfence();
            XRec x = xnone();
            x.c[0] = n_mig;
            x.c[1] = n_reconf;
            x.c[2] = n_ev;
            x.mx = (unsigned)max_intra;
            exchange(x);
            n_mig = x.c[0];
            n_reconf = x.c[1];
            n_ev = x.c[2];
            max_intra = (int)x.mx;
            if (S > 1) wp::cluster_sync();  // no CTA leaves while a push to it may be in flight
            if (gs != 0) return;
            if (T == NT - 1) sc->tl = tl_sum;  // record_sample's thread
            wp::bsync();
            tl_sum = sc->tl;
        }
        if (s.status != STATUS_OK) {
            unsigned mn = NONE;
            for (uint32_t i = q_head + T; i < q_tail; i += NT) {
                const unsigned r = (unsigned)queue[i];
                mn = r < mn ? r : mn;
            }
            unsigned z0 = 0, z1 = 0, z2 = 0;
            int pay = 0;
            block_lexmin(mn, z0, z1, z2, pay);
            s.pending_rank = (int32_t)mn;
        }
        if (W != 0) return;
        double sw = 0.0, se = 0.0, stt = 0.0, first = 0.0, lastc = 0.0;
        if (s.status == STATUS_OK) {
            for (uint32_t base = 0; base < N; base += 32) {
                const uint32_t j = base + L;
                double wv = 0.0, e = 0.0, t = 0.0, a = 0.0, dn = 0.0;
                if (j < N) {
                    a = arr[j];
                    const double sc0 = jobs[j].sched;
                    dn = jobs[j].done;
                    wv = wp::dsub(sc0, a);
                    e = wp::dsub(dn, sc0);
                    t = wp::dadd(wv, e);
                }
                const uint32_t n = N - base < 32 ? N - base : 32;
                for (uint32_t k = 0; k < n; ++k) {
                    const double wk = wp::shfl(wv, (int)k), ek = wp::shfl(e, (int)k), tk = wp::shfl(t, (int)k);
                    const double ak = wp::shfl(a, (int)k), dk = wp::shfl(dn, (int)k);
                    sw = wp::dadd(sw, wk);
                    se = wp::dadd(se, ek);
                    stt = wp::dadd(stt, tk);
                    if (base + k == 0) {
                        first = ak;
                        lastc = dk;
                    } else {
                        first = ak < first ? ak : first;
                        lastc = lastc < dk ? dk : lastc;
                    }
                }
            }
        }
        if (N > 0 && s.status == STATUS_OK) {
            const double n = (double)N;
            s.mean_wait = wp::ddiv(sw, n);
            s.mean_exec = wp::ddiv(se, n);
            s.mean_turn = wp::ddiv(stt, n);
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
        if (L == 0) *out = s;
    }
};

template <bool DETAIL>
MSG_DI void simulate_large_trace(const SimArgs& a, const DevTables* tables, BlockScratch* sc,
                                 unsigned char* gpu_smem, bool slots_smem, uint32_t t) {
    ClusterSim<DETAIL> sim;
    sim.setup(a, tables, sc, gpu_smem, slots_smem, t);
    sim.run();
    sim.finish(a.summary + t);
}

}  // namespace msgk
