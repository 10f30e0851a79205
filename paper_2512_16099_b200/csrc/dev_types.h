// Device-side record layouts shared by the kernels (engine_core.cuh) and the
// host runtime (host_runtime.cpp).  Plain PODs, no CUDA types.
#pragma once
#include <stdint.h>

namespace msgk {

// Slot states: one slot per (GPU, start index) — instances on a GPU are
// pairwise slice-disjoint (gpu.cpp:146-156), so a start index names at most
// one instance.  Instance::busy()/idle()/draining (gpu.hpp:18-29) plus the
// job's RunJob state (sim.cpp:58-68) folded in:
enum : uint8_t {
    ST_EMPTY = 0,  // no instance
    ST_IDLE = 1,   // instance without job, not draining
    ST_RUN = 2,    // job bound and Running            (Completion timer)
    ST_WAIT = 3,   // job bound, WaitingStart          (ServiceStart timer)
    ST_DRAIN = 4   // draining source replica          (MigrationEnd timer)
};

// Block engine (cluster_core.cuh): the fragmentation timeline is the
// reference's sequential double sum up to kExactTimelineGpus GPUs; a trace
// is split over up to kMaxShards CTAs (one thread-block cluster) only above
// that size and without the event log.
constexpr int kExactTimelineGpus = 512;
constexpr int kMaxShards = 16;
// A trace can also be split over up to kMaxDev device GROUPS (one cluster
// each): B200s of one box exchanging over NVLink, or clusters of one GPU.
constexpr int kMaxDev = 8;

// One shard's contribution to an exchange (and, after it, the reduction).
struct alignas(16) XRec {
    unsigned hi, lo, tie, ms;  // key, lexicographic minimum wins
    int32_t slot;              // winner payload: global slot
    int32_t job;               //   job rank
    uint32_t info;             //   slot state | profile << 8 | job migrations << 16
    uint32_t w;                // OR: word broadcast by a GPU's owner
    double rem, tkey;          //   remaining work, timer time
    uint32_t c[4];             // sums
    uint32_t mx;               // max
    uint32_t pad;
    uint64_t ks[2];            // sums: deferred timeline samples (cost-total parts)
    uint64_t pad2;             // second minimum: the pending arrival's placement key (next-event exchange)
};
static_assert(sizeof(XRec) == 96, "exchange record layout (6 x 16-byte pushes)");

// A device group's inbox for the cross-group exchange: slot [parity][CTA
// rank][sending group], each validated by a round stamp written with
// release semantics after the record (peer-mapped across GPUs).
struct XInbox {
    XRec rec[2][kMaxShards][kMaxDev];
    uint64_t stamp[2][kMaxShards][kMaxDev];  // epoch << 32 | round + 1
};

// Feature / output flags.
enum : uint32_t {
    CF_LB = 1u,      // FeatureFlags::load_balancing
    CF_DYN = 2u,     // FeatureFlags::dynamic_partitioning
    CF_MIG = 4u      // FeatureFlags::migration
};
enum : uint32_t { OF_JOBS = 1u, OF_EVENTS = 2u, OF_TIMELINE = 4u, OF_ZC = 8u /* in-kernel: zero-copy inputs */,
                   OF_PROG = 16u /* in-kernel: progressive row flushes */ };

struct DevConfig {
    double alpha;     // SimConfig::contention_alpha
    double overlap;   // SimConfig::migration_overlap_s
    double latency;   // SimConfig::reconfig_latency_s
    int32_t G;        // SimConfig::gpu_count
    uint32_t flags;   // CF_*
    uint32_t lazymask;  // bit pc set iff pc/7.0 < threshold (gpu.cpp:168-177)
    uint32_t n_init;    // static-layout instances (sim.cpp:86-95)
    uint32_t init_off;  // offset into the init-slot array
    uint32_t reserved;
};

// Packed static-layout instance: slot | profile << 24 (creation order = array order).
struct DevTrace {
    uint64_t job_off;   // first job (rank order) in the batch arrays
    uint64_t ev_off;    // first event record
    uint64_t tl_off;    // first timeline sample
    uint32_t n_jobs;
    uint32_t cfg;
    uint32_t ev_cap;
    uint32_t tl_cap;
    uint32_t has_perm;  // arrival order differs from rank order
    uint32_t large;     // G > 32: simulated by the block engine (cluster_core.cuh)
    uint64_t cl_goff;   // block engine: first GPU of this trace in the cluster arena
};

// Fixed 32-byte event record written by the kernel (decoded on the host into
// msg_event, include/migsched_b200.h).
struct EventRec {
    double t;
    uint64_t aux;      // bits of scheduled_s; MigrationStart: 4 x u16 cost numerators over 25200
    int32_t job;       // job rank (dense id order), -1 none
    uint16_t gpu;      // gpu / from_gpu
    uint16_t gpu2;     // to_gpu
    uint8_t kind;      // msg EventKind
    uint8_t profile;
    uint8_t start;     // start / from_start
    uint8_t start2;    // to_start
    uint8_t flags;     // EF_*
    uint8_t pad[3];
};
static_assert(sizeof(EventRec) == 32, "EventRec must be 32 bytes");
enum : uint8_t { EF_REUSED = 1, EF_PLACED = 2, EF_DESTROY = 4, EF_INTER = 8 };

struct JobOut {
    double sched;      // service start (scheduled_s)
    double done;       // completion time
    int32_t gpu;       // final GPU
    int32_t mig;       // migrations
};

struct DevSummary {
    int32_t status;
    uint32_t reserved;
    uint64_t handler_events;
    uint64_t n_events;
    uint64_t timeline_samples;
    int64_t migrations;
    int64_t reconfig_ops;
    int64_t enqueues;
    int64_t dequeues;
    int32_t max_arr;
    int32_t max_intra;
    int32_t max_inter;
    int32_t pending_rank;   // smallest queued job rank when JobsPending
    double mean_wait;
    double mean_exec;
    double mean_turn;
    double makespan;
    double tl_sum;
};

// Read-only lookup tables computed on the host from the exact-rational
// fragmentation metric (frag.cpp:44-58) and staged into shared memory.
struct DevTables {
    uint8_t cost2rank[8 * 256];  // [popc(busy_c)][busy_m] -> rank of the 2-mask cost
    double cost4val[256];        // 4-mask cost id -> frag_cost as double (k / 25200.0)
    uint16_t cost4k[256];        // 4-mask cost id -> numerator k over 25200
    uint16_t rank2k[32];         // cost rank -> numerator over 25200
    uint8_t placeable[256];      // blocked_m -> profiles with >= 1 free legal start
    uint8_t feasid[256];         // blocked_m -> id of its per-profile feasible-count vector
    uint8_t idealid[80];         // popc(busy_c) * 9 + popc(busy_m) -> id of its ideal-count vector
    uint8_t cost4pair[32 * 32];  // [ideal id][feasible id] -> 4-mask cost id
    uint32_t share_run[6 * 8];   // [profile][start] -> a Running instance's share of the GPU word
};

// Kernel arguments of the per-trace event loop (engine_core.cuh).
struct SimArgs {
    const DevTrace* traces;
    const DevConfig* configs;
    const uint32_t* init_slots;
    const DevTables* tables;
    const uint16_t* score_tab;  // the arrival scorer's per-word table (host_tables.h, build_score_table), or null
    const double* arrival;   // rank order
    const double* service;
    const uint8_t* profile;
    const int32_t* profile32;  // optional: the caller's int32 profiles (pipelined direct inputs); each
                               // warp narrows its trace's into `profile` before its first event
    const uint32_t* perm;    // arrival order -> rank (only traces with has_perm)
    // optional (pipelined msg_run_batch, page-locked caller arrays, every
    // trace in input order): the caller's arrival / service / int32 profile
    // arrays as mapped host memory, indexed like `arrival`.  Each warp reads
    // its trace over PCIe one 32-job block at a time as its arrivals reach
    // the block and publishes the block into arrival / service / profile
    // (no H2D copy and no host staging before the launch).
    const double* zc_arrival;
    const double* zc_service;
    const int32_t* zc_profile;
    int32_t* queue;          // FCFS queue storage, n_jobs per trace
    JobOut* jobs;
    JobOut* jobs_host;       // optional (pipelined msg_run_batch): a finished trace's records, also
                             // stored by its warp into mapped pinned host memory (no separate D2H)
    EventRec* events;
    double* timeline;        // (t, mean) pairs
    DevSummary* summary;
    DevSummary* summary_host;  // optional (pipelined msg_run_batch): the summary, also in mapped host memory,
    uint32_t* done_host;       // then done_host[t] = done_epoch once the trace's host records are visible
    uint32_t done_epoch;
    // optional (with jobs_host and done_host): progressive row publication.
    // prog_host[t] = done_epoch << 32 | n once the records of the trace's
    // first n jobs (all completed) are in jobs_host; the warp flushes the
    // completed prefix every 64 arrivals (prog_mask), so the host decodes rows while the
    // trace still runs.
    uint64_t* prog_host;
    uint32_t prog_mask;  // flush when the arrival index is a multiple of prog_mask + 1 (a power of two >= 32)
    // IO kernel: jobs_host holds SoA columns over the batch's rows_soa jobs —
    // sched f64 [rows_soa], done f64 [rows_soa], gpu | migrations << 32 u64
    // [rows_soa] — so each warp store covers whole 128-byte lines over PCIe
    uint64_t rows_soa;
    uint32_t n_traces;
    uint32_t out_flags;
    uint32_t no_delay;  // every config: reconfig latency 0 and migration overlap 0 (the ND kernels)
    // block engine (G > 32): cluster arena, indexed by GPU (cl_goff + g) or
    // slot (8 * (cl_goff + g) + s), and the list of large traces
    const uint32_t* large_idx;
    uint32_t n_large;
    uint32_t shards;   // CTAs (GPU-range shards) per large trace: one thread-block cluster
    // per slot (8 per GPU)
    uint8_t* c_st;
    uint8_t* c_prof;
    uint16_t* c_mig;
    uint32_t* c_cseq;
    int32_t* c_apos;   // slot -> index in the active list, -1
    // per active-list entry (capacity 8 per GPU): the slot's timer data
    int32_t* c_aslot;
    uint8_t* c_ast;
    int32_t* c_ajob;
    uint32_t* c_amseq;
    double* c_arem;
    double* c_atkey;
    // per GPU (used only when they do not fit in shared memory)
    uint32_t* c_gw;
    uint32_t* c_gx;
    uint8_t* c_gcid;
    uint32_t smem_gpus;  // per-GPU arrays live in shared memory for G <= smem_gpus (set by launch_cluster)
    uint32_t smem_slots; // ... and so do the per-slot arrays
    // device groups (cluster_core.cuh): n_dev groups per trace; this launch
    // runs groups dev0 .. dev0 + vdev - 1 of every large trace (vdev = n_dev:
    // all groups on this GPU; vdev = 1: one group per GPU, dev0 = rank).
    // inbox[k]: group k's exchange inbox (peer-mapped across GPUs).
    uint32_t n_dev;
    uint32_t dev0;
    uint32_t vdev;
    uint32_t epoch;    // run number of a multi-GPU group (inbox stamps need no reset between runs)
    void* inbox[kMaxDev];
    uint32_t max_gpus;   // largest G among the large traces
};

// Decision-level kernel arguments (decide.cu): one warp per cluster snapshot
// of G <= 32 GPUs.  Slot words: state (ST_*) | profile << 4 | cseq << 8.
enum : int32_t {
    SOP_SCHEDULE = 0,
    SOP_FIRST_FIT = 1,
    SOP_DISPATCH = 2,
    SOP_ON_DEPARTURE = 10,
    SOP_PLAN_INTRA = 11,
    SOP_PLAN_INTER = 12,
    SOP_TRY_DEQUEUE = 20
};
struct SnapArgs {
    const DevTables* tables;
    const uint32_t* slot_in;   // n * G * 8
    const int32_t* job_in;     // n * G * 8 job ranks, -1 none
    uint32_t* slot_out;
    int32_t* job_out;
    const int32_t* arg;        // per snapshot: profile (schedule) or gpu (plans)
    const int32_t* queue;      // try_dequeue: per snapshot q_cap job ranks
    const uint32_t* q_len;     // try_dequeue: per snapshot queue length
    const uint8_t* rank_profile;  // try_dequeue: per snapshot rank_cap profiles, indexed by job rank
    JobOut* scratch;           // per snapshot rank_cap job outputs (unused results)
    int32_t* out;              // per snapshot 8 ints
    EventRec* events;          // per snapshot ev_cap records
    uint32_t ev_cap;
    uint32_t q_cap;
    uint32_t rank_cap;
    uint32_t n;
    int32_t G;
    int32_t op;
    uint32_t cflags;
    uint32_t lazymask;
    double overlap;
    int32_t enabled;
    int32_t reserved;
};

constexpr int kProfileCount = 6;  // profiles.cpp:8-15
// Constant geometry (profiles.cpp:8-15), packed per profile id.
constexpr uint32_t kCsPack = 0x112347u;               // nibble p: compute slices
constexpr uint32_t kMsPack = 0x122448u;               // nibble p: memory slices
constexpr uint64_t kStartMask = 0x00007F5515110101ull;  // byte p: legal starts
constexpr uint32_t kStridePack = 0x122488u;           // nibble p: start stride
constexpr uint32_t kCountPack = 0x743211u;            // nibble p: number of starts

}  // namespace msgk
