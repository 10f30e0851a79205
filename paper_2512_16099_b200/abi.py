"""ctypes / numpy mirrors of the record types in include/migsched_b200.h.

Pure data layout — no logic.  Field order and sizes must match the C header
exactly; tests/test_abi.py checks the sizes against the compiled library.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

# ---- status codes (include/migsched_b200.h, reference error.hpp:10-19) ----
STATUS_NAMES = {
    0: "Ok",
    1: "InvalidPlacement",
    2: "SlicesBusy",
    3: "UnknownJob",
    4: "UnknownGpu",
    5: "NotLazy",
    6: "UnknownProfile",
    7: "BadThreshold",
    8: "BadConfig",
    9: "BadSpec",
    10: "TraceUnsorted",
    11: "BadConcurrency",
    12: "JobsPending",
    13: "ParseError",
    100: "CudaError",
    101: "Unsupported",
    102: "InvalidArgument",
}
STATUS_BY_NAME = {v: k for k, v in STATUS_NAMES.items()}

OUT_JOBS = 1
OUT_EVENTS = 2
OUT_TIMELINE = 4

SLOT_EMPTY, SLOT_IDLE, SLOT_BUSY, SLOT_DRAINING = 0, 1, 2, 3
OP_SCHEDULE, OP_FIRST_FIT, OP_DISPATCH = 0, 1, 2
PLAN_ON_DEPARTURE, PLAN_INTRA, PLAN_INTER = 0, 1, 2

HAS_JOB = 1 << 0
HAS_GPU = 1 << 1
HAS_PROFILE = 1 << 2
HAS_START = 1 << 3
HAS_SIZE = 1 << 4
HAS_REUSED = 1 << 5
HAS_SCHEDULED = 1 << 6
HAS_ACTION = 1 << 7
HAS_FROM_GPU = 1 << 8
HAS_FROM_START = 1 << 9
HAS_TO_GPU = 1 << 10
HAS_TO_START = 1 << 11
HAS_MOVE_KIND = 1 << 12
HAS_OVERLAP = 1 << 13
HAS_COSTS = 1 << 14


class MsgConfig(C.Structure):
    _fields_ = [
        ("threshold", C.c_double),
        ("contention_alpha", C.c_double),
        ("migration_overlap_s", C.c_double),
        ("reconfig_latency_s", C.c_double),
        ("seed", C.c_uint64),
        ("gpu_count", C.c_int32),
        ("load_balancing", C.c_uint8),
        ("dynamic_partitioning", C.c_uint8),
        ("migration", C.c_uint8),
        ("has_static_layout", C.c_uint8),
        ("layout_gpus", C.c_int32),
        ("reserved0", C.c_int32),
        ("layout_offsets", C.POINTER(C.c_int32)),
        ("layout_profile", C.POINTER(C.c_int32)),
        ("layout_start", C.POINTER(C.c_int32)),
    ]


class MsgTraceBatch(C.Structure):
    _fields_ = [
        ("n_traces", C.c_uint32),
        ("reserved0", C.c_uint32),
        ("offsets", C.POINTER(C.c_uint64)),
        ("job_id", C.POINTER(C.c_int64)),
        ("arrival_s", C.POINTER(C.c_double)),
        ("profile", C.POINTER(C.c_int32)),
        ("service_s", C.POINTER(C.c_double)),
        ("config_index", C.POINTER(C.c_uint32)),
    ]


class MsgWorkloadSpec(C.Structure):
    _fields_ = [
        ("mean_interarrival_s", C.c_double),
        ("profile_mix", C.c_double * 4),
        ("median_s", C.c_double),
        ("sigma", C.c_double),
        ("mean_s", C.c_double),
        ("value_s", C.c_double),
        ("seed", C.c_uint64),
        ("query_type", C.c_int32),
        ("service_family", C.c_int32),
        ("job_count", C.c_int32),
        ("reserved0", C.c_int32),
    ]


class MsgSchedConfig(C.Structure):
    _fields_ = [
        ("threshold", C.c_double),
        ("load_balancing", C.c_uint8),
        ("dynamic_partitioning", C.c_uint8),
        ("reserved", C.c_uint8 * 6),
    ]


EVENT_DTYPE = np.dtype(
    [
        ("time_s", "<f8"),
        ("scheduled_s", "<f8"),
        ("overlap_s", "<f8"),
        ("from_cost_before", "<f8"),
        ("from_cost_after", "<f8"),
        ("to_cost_before", "<f8"),
        ("to_cost_after", "<f8"),
        ("job", "<i8"),
        ("kind", "<i4"),
        ("present", "<u4"),
        ("gpu", "<i4"),
        ("profile", "<i4"),
        ("start", "<i4"),
        ("size", "<i4"),
        ("reused", "<i4"),
        ("action", "<i4"),
        ("from_gpu", "<i4"),
        ("from_start", "<i4"),
        ("to_gpu", "<i4"),
        ("to_start", "<i4"),
        ("move_kind", "<i4"),
        ("reserved0", "<i4"),
    ]
)
assert EVENT_DTYPE.itemsize == 120

JOB_DTYPE = np.dtype(
    [
        ("id", "<i8"),
        ("arrival_s", "<f8"),
        ("scheduled_s", "<f8"),
        ("completed_s", "<f8"),
        ("wait_s", "<f8"),
        ("execution_s", "<f8"),
        ("turnaround_s", "<f8"),
        ("profile", "<i4"),
        ("gpu", "<i4"),
        ("migrations", "<i4"),
        ("reserved0", "<i4"),
    ]
)
assert JOB_DTYPE.itemsize == 72

TIMELINE_DTYPE = np.dtype([("time_s", "<f8"), ("mean_frag_cost", "<f8")])

SUMMARY_DTYPE = np.dtype(
    [
        ("status", "<i4"),
        ("gpu_count", "<i4"),
        ("n_jobs", "<u8"),
        ("handler_events", "<u8"),
        ("n_events", "<u8"),
        ("timeline_samples", "<u8"),
        ("migration_count", "<i8"),
        ("reconfig_op_count", "<i8"),
        ("enqueue_count", "<i8"),
        ("dequeue_count", "<i8"),
        ("max_arrival_frag_evals", "<i4"),
        ("max_intra_iter_frag_evals", "<i4"),
        ("max_inter_iter_frag_evals", "<i4"),
        ("reserved0", "<i4"),
        ("mean_wait_s", "<f8"),
        ("mean_execution_s", "<f8"),
        ("mean_turnaround_s", "<f8"),
        ("workload_makespan_s", "<f8"),
        ("timeline_sum", "<f8"),
    ]
)
assert SUMMARY_DTYPE.itemsize == 128

INSTANCE_DTYPE = np.dtype(
    [("job", "<i8"), ("seq", "<u4"), ("profile", "i1"), ("state", "u1"), ("reserved0", "<u2")]
)
assert INSTANCE_DTYPE.itemsize == 16

DECISION_DTYPE = np.dtype(
    [
        ("placed", "<i4"),
        ("gpu", "<i4"),
        ("start", "<i4"),
        ("size", "<i4"),
        ("reused", "<i4"),
        ("evaluated_candidates", "<i4"),
    ]
)

MOVE_DTYPE = np.dtype(
    [
        ("job", "<i8"),
        ("profile", "<i4"),
        ("from_gpu", "<i4"),
        ("from_start", "<i4"),
        ("to_gpu", "<i4"),
        ("to_start", "<i4"),
        ("move_kind", "<i4"),
        ("reused", "<i4"),
        ("n_destroyed", "<i4"),
        ("from_cost_before", "<f8"),
        ("from_cost_after", "<f8"),
        ("to_cost_before", "<f8"),
        ("to_cost_after", "<f8"),
    ]
)
assert MOVE_DTYPE.itemsize == 72

PLAN_SUMMARY_DTYPE = np.dtype(
    [
        ("status", "<i4"),
        ("kind", "<i4"),
        ("n_moves", "<i4"),
        ("n_iterations", "<i4"),
        ("max_evals", "<i4"),
        ("reserved0", "<i4"),
    ]
)


def ptr(arr: np.ndarray, ctype):
    """ctypes pointer to a contiguous numpy array (or NULL for None)."""
    if arr is None:
        return C.POINTER(ctype)()
    assert arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data_as(C.POINTER(ctype))
