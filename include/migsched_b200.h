/*
 * migsched_b200.h — C ABI of the B200-native MIG scheduler engine.
 *
 * Drop-in boundary for the reference's scheduler hot path (arXiv 2512.16099,
 * "migsched").  The reference has no FFI of its own: its policy interface is
 * plain C++ free functions.  Every entry point below replaces
 * one of those functions; the comment on each cites the reference signature
 * (paths relative to /root/reference/proj/).  The C++ façade in
 * include/migsched_b200.hpp re-exports the reference's own signatures on top
 * of this header; INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Conventions
 *  - No entry point throws.  Failures return a msg_status whose name
 *    (msg_status_name) is the reference's migsched::Error code string
 *    (include/migsched/error.hpp:10-19); a human-readable message is
 *    available from msg_engine_last_error / msg_result_message.
 *  - The caller owns every input; results are library-allocated and freed
 *    with msg_result_free.  Device memory is owned by the engine handle.
 *  - An engine handle is externally synchronised (one host thread at a time);
 *    independent handles are reentrant.  One CUDA stream per handle.
 *  - There is no CPU fallback: every msg_run_* / msg_decide_* call executes
 *    sm_100a kernels; without a usable device the call fails with
 *    MSG_ERR_CUDA.
 */
#ifndef MIGSCHED_B200_H
#define MIGSCHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSG_ABI_VERSION 1

/* ---- status codes: one per migsched::Error code (error.hpp:10-19) ------- */
typedef enum msg_status {
    MSG_OK = 0,
    MSG_ERR_INVALID_PLACEMENT = 1, /* "InvalidPlacement" profiles.cpp:49-57 */
    MSG_ERR_SLICES_BUSY = 2,       /* "SlicesBusy"       gpu.cpp:74,107 */
    MSG_ERR_UNKNOWN_JOB = 3,       /* "UnknownJob"       gpu.cpp:122,133,143 */
    MSG_ERR_UNKNOWN_GPU = 4,       /* "UnknownGpu"       migration.cpp:14 */
    MSG_ERR_NOT_LAZY = 5,          /* "NotLazy"          migration.cpp:128 */
    MSG_ERR_UNKNOWN_PROFILE = 6,   /* "UnknownProfile"   scheduler.cpp:13, sim.cpp:101 */
    MSG_ERR_BAD_THRESHOLD = 7,     /* "BadThreshold"     gpu.cpp:174, sim.cpp:76 */
    MSG_ERR_BAD_CONFIG = 8,        /* "BadConfig"        sim.cpp:74-90 */
    MSG_ERR_BAD_SPEC = 9,          /* "BadSpec"          sim.cpp:107-111, workload.cpp:44-63 */
    MSG_ERR_TRACE_UNSORTED = 10,   /* "TraceUnsorted"    sim.cpp:104 */
    MSG_ERR_BAD_CONCURRENCY = 11,  /* "BadConcurrency"   sim.cpp:28 */
    MSG_ERR_JOBS_PENDING = 12,     /* "JobsPending"      sim.cpp:465 */
    MSG_ERR_PARSE_ERROR = 13,      /* "ParseError"       workload.cpp:153-191 */
    /* engine-specific (no reference counterpart) */
    MSG_ERR_CUDA = 100,            /* "CudaError": no device / launch failure */
    MSG_ERR_UNSUPPORTED = 101,     /* "Unsupported": outside this engine's envelope */
    MSG_ERR_INVALID_ARGUMENT = 102 /* "InvalidArgument": malformed ABI call */
} msg_status;

/* Stable code string, e.g. "SlicesBusy"; "Unknown" for out-of-range values. */
const char* msg_status_name(int status);

/* ---- MIG geometry (profiles.hpp:15-24, profiles.cpp:8-15) --------------- */
enum {
    MSG_P7G40GB = 0,
    MSG_P4G20GB = 1,
    MSG_P3G20GB = 2,
    MSG_P2G10GB = 3,
    MSG_P1G10GB = 4,
    MSG_P1G5GB = 5,
    MSG_PROFILE_COUNT = 6
};

/* ---- configuration: SimConfig (sim.hpp:88-95) + SchedulerConfig
 *      (scheduler.hpp:12-29).  The static layout is CSR-flattened. -------- */
typedef struct msg_config {
    double threshold;             /* SchedulerConfig::threshold          */
    double contention_alpha;      /* SimConfig::contention_alpha         */
    double migration_overlap_s;   /* SimConfig::migration_overlap_s      */
    double reconfig_latency_s;    /* SimConfig::reconfig_latency_s       */
    uint64_t seed;                /* SimConfig::seed (echoed only)       */
    int32_t gpu_count;            /* SimConfig::gpu_count                */
    uint8_t load_balancing;       /* FeatureFlags                        */
    uint8_t dynamic_partitioning;
    uint8_t migration;
    uint8_t has_static_layout;    /* optional<StaticLayout> engaged      */
    int32_t layout_gpus;          /* StaticLayout::size()                */
    int32_t reserved0;
    const int32_t* layout_offsets; /* layout_gpus + 1 offsets            */
    const int32_t* layout_profile; /* ProfileId per entry                */
    const int32_t* layout_start;   /* start index per entry              */
} msg_config;

/* ---- traces: std::vector<Job> (sim.hpp:13-18), batched, SoA + CSR ------ */
typedef struct msg_trace_batch {
    uint32_t n_traces;
    uint32_t reserved0;
    const uint64_t* offsets;      /* n_traces + 1 job offsets            */
    const int64_t* job_id;        /* Job::id                             */
    const double* arrival_s;      /* Job::arrival_s                      */
    const int32_t* profile;       /* Job::profile (ProfileId)            */
    const double* service_s;      /* Job::service_s                      */
    const uint32_t* config_index; /* per-trace index into cfgs; NULL = 0 */
} msg_trace_batch;

/* ---- results ------------------------------------------------------------ */

/* Event kinds: EventKind (sim.hpp:20-28), same numeric order. */
enum {
    MSG_EV_ARRIVAL = 0,
    MSG_EV_COMPLETION = 1,
    MSG_EV_MIGRATION_START = 2,
    MSG_EV_MIGRATION_END = 3,
    MSG_EV_RECONFIG = 4,
    MSG_EV_ENQUEUE = 5,
    MSG_EV_DEQUEUE = 6
};

/* Presence bits of the optional SimEvent fields (sim.hpp:33-52). */
enum {
    MSG_HAS_JOB = 1u << 0,
    MSG_HAS_GPU = 1u << 1,
    MSG_HAS_PROFILE = 1u << 2,
    MSG_HAS_START = 1u << 3,
    MSG_HAS_SIZE = 1u << 4,
    MSG_HAS_REUSED = 1u << 5,
    MSG_HAS_SCHEDULED = 1u << 6,
    MSG_HAS_ACTION = 1u << 7,
    MSG_HAS_FROM_GPU = 1u << 8,
    MSG_HAS_FROM_START = 1u << 9,
    MSG_HAS_TO_GPU = 1u << 10,
    MSG_HAS_TO_START = 1u << 11,
    MSG_HAS_MOVE_KIND = 1u << 12,
    MSG_HAS_OVERLAP = 1u << 13,
    MSG_HAS_COSTS = 1u << 14 /* the four from/to cost fields */
};

/* Decoded SimEvent.  Absent fields are zero; `present` says which are set.
 * profile: ProfileId; action: 0 create / 1 destroy; move_kind: 0 intra /
 * 1 inter.  No implicit padding (120 bytes). */
typedef struct msg_event {
    double time_s;
    double scheduled_s;
    double overlap_s;
    double from_cost_before;
    double from_cost_after;
    double to_cost_before;
    double to_cost_after;
    int64_t job;
    int32_t kind;
    uint32_t present;
    int32_t gpu;
    int32_t profile;
    int32_t start;
    int32_t size;
    int32_t reused;
    int32_t action;
    int32_t from_gpu;
    int32_t from_start;
    int32_t to_gpu;
    int32_t to_start;
    int32_t move_kind;
    int32_t reserved0;
} msg_event;

/* JobMetrics (sim.hpp:56-67); rows are in job-id order like metrics(). */
typedef struct msg_job_row {
    int64_t id;
    double arrival_s;
    double scheduled_s;
    double completed_s;
    double wait_s;
    double execution_s;
    double turnaround_s;
    int32_t profile;
    int32_t gpu;
    int32_t migrations;
    int32_t reserved0;
} msg_job_row;

/* One fragmentation-timeline sample (SimReport::frag_timeline, sim.hpp:85). */
typedef struct msg_timeline_point {
    double time_s;
    double mean_frag_cost;
} msg_timeline_point;

/* Per-trace aggregate: SimReport (sim.hpp:75-86) + ComplexityStats + the
 * engine's counters.  handler_events counts Arrival, valid Completion,
 * MigrationEnd and ServiceStart timer pops (sim.cpp:124-134) — the unit of
 * the "scheduling decisions/s" metric.  timeline_sum is the sequential double
 * sum of every timeline sample value (a digest available without
 * MSG_OUT_TIMELINE). */
typedef struct msg_trace_summary {
    int32_t status;
    int32_t gpu_count;
    uint64_t n_jobs;
    uint64_t handler_events;
    uint64_t n_events;
    uint64_t timeline_samples;
    int64_t migration_count;
    int64_t reconfig_op_count;
    int64_t enqueue_count;
    int64_t dequeue_count;
    int32_t max_arrival_frag_evals;
    int32_t max_intra_iter_frag_evals;
    int32_t max_inter_iter_frag_evals;
    int32_t reserved0;
    double mean_wait_s;
    double mean_execution_s;
    double mean_turnaround_s;
    double workload_makespan_s;
    double timeline_sum;
} msg_trace_summary;

/* Output selection for msg_run_batch / msg_stage. The summary is always
 * produced. */
enum {
    MSG_OUT_JOBS = 1u << 0,     /* per-job rows                          */
    MSG_OUT_EVENTS = 1u << 1,   /* full event log                        */
    MSG_OUT_TIMELINE = 1u << 2  /* every frag-timeline sample            */
};

typedef struct msg_engine msg_engine;
typedef struct msg_staged msg_staged;
typedef struct msg_batch_result msg_batch_result;

/* ---- engine lifecycle --------------------------------------------------- */
msg_status msg_engine_create(int device, msg_engine** out);
void msg_engine_destroy(msg_engine* engine);
const char* msg_engine_last_error(const msg_engine* engine);
/* Number of kernels this engine has launched so far. */
uint64_t msg_engine_launch_count(const msg_engine* engine);
/* Device name / SM count, for reports. */
msg_status msg_engine_device_info(const msg_engine* engine, char* name, size_t name_len,
                                  int32_t* sm_count);

/* ---- engine-level entry: replaces migsched::run (sim.hpp:114, sim.cpp:504)
 * for a batch of independent traces.  Each trace is validated exactly like
 * Engine::Engine (sim.cpp:73-116); a trace that fails validation gets its
 * status and the reference's message and no results.  (With page-locked
 * inputs the validation runs on host threads while the kernel already
 * simulates the batch; a failing trace's device results are discarded.)
 * JobsPending (sim.cpp:464-466) is reported per trace after the
 * simulation. -------------------------------------------------------------- */
msg_status msg_run_batch(msg_engine* engine, const msg_trace_batch* batch, const msg_config* cfgs,
                         uint32_t n_cfgs, uint32_t out_flags, msg_batch_result** out);

/* Page-locked host memory for input batches.  When a batch's arrival_s,
 * service_s and profile arrays live in such memory (this allocator, or any
 * cudaHostAlloc / cudaHostRegister(..., Mapped) range), msg_run_batch
 * launches the whole batch at once and the kernel reads the inputs in place
 * over PCIe as each trace's arrivals reach them (zero copy; no staging, the
 * checks run under the kernel), and job rows are decoded while it runs.
 * Any host memory works; this removes the staging and its latency.
 * msg_host_alloc returns mapped memory usable from every device of the
 * process.  The arrays must stay unchanged until msg_run_batch returns. */
msg_status msg_host_alloc(size_t bytes, void** out);
void msg_host_free(void* p);

/* The same call split in three for device-resident benchmarking and
 * pipelining: msg_stage validates and copies host inputs to HBM;
 * msg_launch enqueues the simulation on the engine stream (asynchronous);
 * msg_collect waits, copies results back and decodes them.  A staged batch
 * may be launched any number of times. */
msg_status msg_stage(msg_engine* engine, const msg_trace_batch* batch, const msg_config* cfgs,
                     uint32_t n_cfgs, uint32_t out_flags, msg_staged** out);
msg_status msg_launch(msg_engine* engine, msg_staged* staged);
msg_status msg_collect(msg_engine* engine, msg_staged* staged, msg_batch_result** out);
void msg_staged_free(msg_staged* staged);
/* Handler events of all valid traces of the last collected launch (0 before). */
uint64_t msg_staged_handler_events(const msg_staged* staged);

/* ---- timing helpers (CUDA events on the engine stream) ------------------ */
msg_status msg_engine_sync(msg_engine* engine);
/* Launch `staged` once between two events on the engine stream and return
 * the device time in milliseconds. */
msg_status msg_time_launch(msg_engine* engine, msg_staged* staged, float* ms);
/* Write a buffer larger than L2 (256 MiB) so the next launch starts cold. */
msg_status msg_engine_flush_l2(msg_engine* engine);
/* The same write enqueued on the engine stream without waiting for it: the
 * launch that follows is queued behind it, so a kernel timed next starts on
 * a busy device (its host launch latency is not inside the events). */
msg_status msg_engine_flush_l2_async(msg_engine* engine);

/* ---- multi-GPU: one large trace split over the B200s of one NVLink /
 * NVSwitch domain, one process per GPU (configuration C4) ------
 * Rank r owns a contiguous range of the simulated cluster's GPUs (split
 * further over the CTAs of one thread-block cluster); every decision is a
 * device-initiated all-reduce of packed (score, index) keys: each rank's
 * record is stored into every peer's inbox over NVLink with a release stamp
 * and read back with acquire loads — no host round trip, no NCCL call on
 * the path.  Setup: msg_peer_open on every rank; exchange the
 * msg_peer_handle_size()-byte blobs of msg_peer_export (an all-gather, e.g.
 * over torch.distributed); msg_peer_connect with all blobs in rank order.
 * Every rank then calls msg_run_peer with the same single-trace batch and
 * config (more than 512 GPUs, no event log); the result is returned on rank 0
 * only (*out stays NULL on the others).  Replaces migsched::run (sim.hpp:114)
 * for that trace; the fragmentation timeline follows the block engine's
 * integer-sum rule above 512 GPUs. */
typedef struct msg_peer msg_peer;
size_t msg_peer_handle_size(void);
msg_status msg_peer_open(msg_engine* engine, int32_t world, int32_t rank, uint64_t max_jobs, msg_peer** out);
msg_status msg_peer_export(msg_peer* peer, void* blob);
msg_status msg_peer_connect(msg_peer* peer, const void* blobs);
msg_status msg_run_peer(msg_engine* engine, msg_peer* peer, const msg_trace_batch* batch, const msg_config* cfg,
                        uint32_t out_flags, msg_batch_result** out);
void msg_peer_close(msg_peer* peer);

/* ---- result accessors --------------------------------------------------- */
uint32_t msg_result_n_traces(const msg_batch_result* result);
const msg_trace_summary* msg_result_summary(const msg_batch_result* result, uint32_t trace);
const msg_job_row* msg_result_jobs(const msg_batch_result* result, uint32_t trace, uint64_t* n);
const msg_event* msg_result_events(const msg_batch_result* result, uint32_t trace, uint64_t* n);
const msg_timeline_point* msg_result_timeline(const msg_batch_result* result, uint32_t trace,
                                              uint64_t* n);
const char* msg_result_message(const msg_batch_result* result, uint32_t trace);
/* Bulk views: every trace's summary (n_traces, contiguous), and every
 * trace's job rows concatenated in trace order with n_traces + 1 offsets
 * (NULL unless MSG_OUT_JOBS).  Traces that failed have no rows. */
const msg_trace_summary* msg_result_summaries(const msg_batch_result* result);
const msg_job_row* msg_result_all_jobs(const msg_batch_result* result, const uint64_t** offsets, uint64_t* n);
void msg_result_free(msg_batch_result* result);

/* ---- trace ingest: migsched::load_trace (workload.hpp:53,
 * workload.cpp:151-199).  Reads a JSONL trace file (one {"schema":1,
 * "job_id", "arrival_s", "profile", "service_s"} object per line; blank lines
 * skipped) in parallel, with the reference's validation and messages
 * ("line N: not valid JSON" / "expected an object" / "unsupported schema
 * version" / "missing or mistyped field" / "times must be non-negative" as
 * ParseError, unknown profile names as UnknownProfile; the first failing
 * line wins) and returns the jobs stable-sorted by arrival, ready for a
 * msg_trace_batch.  `msg` (optional) receives "<Code>: <message>". */
typedef struct msg_trace_file msg_trace_file;
msg_status msg_trace_load(const char* path, msg_trace_file** out, char* msg, size_t msg_len);
uint64_t msg_trace_file_jobs(const msg_trace_file* file);
const int64_t* msg_trace_file_ids(const msg_trace_file* file);
const double* msg_trace_file_arrival(const msg_trace_file* file);
const int32_t* msg_trace_file_profile(const msg_trace_file* file);
const double* msg_trace_file_service(const msg_trace_file* file);
void msg_trace_file_free(msg_trace_file* file);

/* ---- report emission: the reference's output files (reports.cpp:14-116)
 * byte for byte, formatted in parallel on the host — events.jsonl
 * (events_to_jsonl), report.json (report_to_json, needs the summary, the
 * config and the per-job rows), report.csv (report_to_csv) and
 * fragcost_timeline.csv (frag_timeline_to_csv), from the records of one
 * trace (msg_result_events / _jobs / _timeline / _summary).  The text is
 * library-allocated (NUL-terminated, *len bytes); free it with
 * msg_text_free. */
typedef enum msg_text_kind {
    MSG_TEXT_EVENTS_JSONL = 0,
    MSG_TEXT_REPORT_JSON = 1,
    MSG_TEXT_REPORT_CSV = 2,
    MSG_TEXT_TIMELINE_CSV = 3
} msg_text_kind;
msg_status msg_format_text(int32_t kind, const msg_trace_summary* summary, const msg_config* cfg,
                           const msg_event* events, uint64_t n_events, const msg_job_row* jobs, uint64_t n_jobs,
                           const msg_timeline_point* timeline, uint64_t n_timeline, char** text, size_t* len);
void msg_text_free(char* text);

/* ---- workload generation: migsched::generate (workload.hpp:45,
 * workload.cpp:98-127) with the same mt19937_64 inverse-transform sampler, so
 * a seed gives the same trace as the reference.  Host-side (trace staging). */
typedef struct msg_workload_spec {
    double mean_interarrival_s; /* WorkloadSpec (workload.hpp:32-39) */
    double profile_mix[4];      /* over {1g.5gb, 2g.10gb, 3g.20gb, 4g.20gb} */
    double median_s;            /* ServiceDist (workload.hpp:17-23)   */
    double sigma;
    double mean_s;
    double value_s;
    uint64_t seed;
    int32_t query_type;         /* 0 Normal, 1 Long                   */
    int32_t service_family;     /* 0 Lognormal, 1 Exponential, 2 Fixed */
    int32_t job_count;
    int32_t reserved0;
} msg_workload_spec;

/* Fill `spec` with the preset of that name (workload.cpp:129-147); returns
 * MSG_ERR_INVALID_ARGUMENT for an unknown name. */
msg_status msg_workload_preset(const char* name, msg_workload_spec* spec);
/* Writes spec->job_count jobs into the four caller-provided arrays. */
msg_status msg_generate(const msg_workload_spec* spec, int64_t* job_id, double* arrival_s,
                        int32_t* profile, double* service_s);
/* Generate `n_seeds` traces (seeds seed0, seed0+1, ...) into CSR arrays
 * sized n_seeds*job_count, using `threads` host threads (0 = all). */
msg_status msg_generate_many(const msg_workload_spec* spec, uint64_t seed0, uint32_t n_seeds,
                             int32_t threads, uint64_t* offsets, int64_t* job_id,
                             double* arrival_s, int32_t* profile, double* service_s);

/* ---- decision-level entries (scheduler.hpp:59-83, migration.hpp:46-63) --
 *
 * A cluster snapshot is gpu_count × 8 instance slots keyed by start index
 * (instances on one GPU are pairwise slice-disjoint, gpu.cpp:146-156, so a
 * start index identifies an instance).  `seq` orders instances of one GPU by
 * creation (the reference's vector order, gpu.cpp:88-111).  `job` is the
 * bound job (busy) or -1. */
enum { MSG_SLOT_EMPTY = 0, MSG_SLOT_IDLE = 1, MSG_SLOT_BUSY = 2, MSG_SLOT_DRAINING = 3 };

typedef struct msg_instance {
    int64_t job;
    uint32_t seq;
    int8_t profile;
    uint8_t state;
    uint16_t reserved0;
} msg_instance;

/* When placed == 0 every field except evaluated_candidates is zero. */
typedef struct msg_decision {
    int32_t placed;   /* 0 = queue the job                         */
    int32_t gpu;
    int32_t start;
    int32_t size;
    int32_t reused;
    int32_t evaluated_candidates;
} msg_decision;

enum { MSG_OP_SCHEDULE = 0, MSG_OP_FIRST_FIT = 1, MSG_OP_DISPATCH = 2 };

typedef struct msg_sched_config {
    double threshold;
    uint8_t load_balancing;
    uint8_t dynamic_partitioning;
    uint8_t reserved[6];
} msg_sched_config;

/* Batched schedule / first_fit_schedule / dispatch_schedule
 * (scheduler.cpp:47-104): n independent cluster snapshots of gpu_count GPUs
 * each (slots: n × gpu_count × 8), one job profile per snapshot. */
msg_status msg_schedule_batch(msg_engine* engine, int32_t op, uint32_t n, int32_t gpu_count,
                              const msg_instance* slots, const int32_t* profile,
                              const msg_sched_config* cfg, msg_decision* out);

/* Packed per-GPU state word used by the large-cluster scorer:
 * bits 0-6 busy compute, 8-15 busy memory, 16-23 blocked memory,
 * 24-41 idle-exact placements (one bit per legal placement, in the order of
 * the profile table).  msg_pack_gpu_word builds it from 8 slots. */
uint64_t msg_pack_gpu_word(const msg_instance* slots8);

/* frag_cost(gpu) (frag.hpp:40-51, frag.cpp:60-65) for n GPU snapshots of 8
 * slots each: the exact cost as a numerator over 25200 (every reachable cost
 * is k/25200) and as the reference's double (k / 25200.0 rounds
 * like its num/den).  Idle instances do not count; draining ones block
 * memory.  Either output may be NULL. */
msg_status msg_frag_cost_batch(msg_engine* engine, uint32_t n, const msg_instance* slots, int32_t* numer_25200,
                               double* cost);

/* Batched scorer over large clusters (SURVEY §8d roofline path): n
 * snapshots × gpu_count packed words (device pointers, resident in HBM), one
 * job profile per snapshot (device).  d_out (device) receives 2 u64 per
 * snapshot: d_out[2i] = argmin key
 *   schedule:   pass << 41 | cost rank << 36 | !reused << 35 | gpu << 3 | start
 *   first fit:  gpu << 3 | start
 * or UINT64_MAX when the job would queue; d_out[2i+1] = (candidates on Lazy
 * GPUs) << 32 | (candidates on Busy GPUs).  Asynchronous on the engine
 * stream. */
msg_status msg_score_device(msg_engine* engine, uint32_t n, int64_t gpu_count, const uint64_t* d_words,
                            const uint8_t* d_profile, const msg_sched_config* cfg, uint64_t* d_out);
/* Same launch bracketed by CUDA events on the engine stream; returns the
 * kernel's device time in milliseconds (synchronous). */
msg_status msg_time_score_device(msg_engine* engine, uint32_t n, int64_t gpu_count, const uint64_t* d_words,
                                 const uint8_t* d_profile, const msg_sched_config* cfg, uint64_t* d_out,
                                 float* ms);

/* try_dequeue (scheduler.cpp:106-121): strict FCFS over each snapshot's
 * queue (CSR: queue_offsets n+1, queue_job, queue_profile).  Slots are
 * updated in place; placed[queue_offsets[i] + k] receives the k-th dequeued
 * head of snapshot i, n_placed[i] how many were placed. */
typedef struct msg_dequeue_item {
    int64_t job;
    int32_t gpu;
    int32_t start;
    int32_t size;
    int32_t reused;
    int32_t evaluated_candidates;
    int32_t n_destroyed;
} msg_dequeue_item;

msg_status msg_try_dequeue_batch(msg_engine* engine, uint32_t n, int32_t gpu_count, msg_instance* slots,
                                 const uint64_t* queue_offsets, const int64_t* queue_job,
                                 const int32_t* queue_profile, const msg_sched_config* cfg,
                                 msg_dequeue_item* placed, uint32_t* n_placed);

/* Migration planning on snapshots: on_departure / plan_intra / plan_inter
 * (migration.cpp:71-220).  Slots are updated in place (moves are applied
 * during planning, like the reference).  Up to max_moves moves per snapshot
 * are written to `moves` (n × max_moves). */
enum { MSG_PLAN_ON_DEPARTURE = 0, MSG_PLAN_INTRA = 1, MSG_PLAN_INTER = 2 };

typedef struct msg_move {
    int64_t job;
    int32_t profile;
    int32_t from_gpu;
    int32_t from_start;
    int32_t to_gpu;
    int32_t to_start;
    int32_t move_kind;        /* 0 intra, 1 inter */
    int32_t reused;           /* destination reused an idle instance */
    int32_t n_destroyed;      /* destination destroy ops */
    double from_cost_before, from_cost_after, to_cost_before, to_cost_after;
} msg_move;

typedef struct msg_plan_summary {
    int32_t status;           /* per snapshot (NotLazy, UnknownGpu, ...) */
    int32_t kind;             /* -1 none, 0 intra, 1 inter */
    int32_t n_moves;          /* may exceed max_moves (then truncated) */
    int32_t n_iterations;
    int32_t max_evals;        /* max frag evaluations per iteration */
    int32_t reserved0;
} msg_plan_summary;

msg_status msg_plan_batch(msg_engine* engine, int32_t op, uint32_t n, int32_t gpu_count,
                          msg_instance* slots, const int32_t* gpu, double threshold,
                          int32_t enabled, double overlap_s, uint32_t max_moves,
                          msg_move* moves, msg_plan_summary* summaries);

#ifdef __cplusplus
}
#endif

#endif /* MIGSCHED_B200_H */
