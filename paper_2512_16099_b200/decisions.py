"""Decision-level API: the reference's per-callback policy functions on
cluster snapshots, executed by the decision kernels (decide.cu, score.cu).

Reference signatures mirrored (proj/include/migsched/):
  schedule / first_fit_schedule / dispatch_schedule   scheduler.hpp:59-70
  try_dequeue                                          scheduler.hpp:81-83
  plan_intra / plan_inter / on_departure               migration.hpp:51-63

A `Cluster` is the snapshot form of std::vector<GpuState>: 8 slots per GPU
keyed by start index (instances are slice-disjoint, gpu.cpp:146-156), with a
creation sequence that stands for the instance-vector order.  Building a
snapshot is input preparation; every decision runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import abi
from .engine import _check, default_engine, lib
from .model import MEMORY_SLICES, START_INDEXES, MigschedError, SchedulerConfig


def _bind():
    L = lib()
    if getattr(L, "_decisions_bound", False):
        return L
    vp, u32, i32 = C.c_void_p, C.c_uint32, C.c_int32
    for name, res, args in (
        ("msg_schedule_batch", C.c_int, [vp, i32, u32, i32, vp, vp, vp, vp]),
        ("msg_plan_batch", C.c_int, [vp, i32, u32, i32, vp, vp, C.c_double, i32, C.c_double, u32, vp, vp]),
        ("msg_try_dequeue_batch", C.c_int, [vp, u32, i32, vp, vp, vp, vp, vp, vp, vp]),
        ("msg_pack_gpu_word", C.c_uint64, [vp]),
        ("msg_frag_cost_batch", C.c_int, [vp, u32, vp, vp, vp]),
        ("msg_score_device", C.c_int, [vp, u32, C.c_int64, vp, vp, vp, vp]),
        ("msg_time_score_device", C.c_int, [vp, u32, C.c_int64, vp, vp, vp, vp, C.POINTER(C.c_float)]),
    ):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    L._decisions_bound = True
    return L


def _sched_cfg(cfg: SchedulerConfig) -> abi.MsgSchedConfig:
    c = abi.MsgSchedConfig()
    c.threshold = cfg.threshold
    c.load_balancing = int(cfg.features.load_balancing)
    c.dynamic_partitioning = int(cfg.features.dynamic_partitioning)
    return c


class Cluster:
    """Snapshot of gpu_count GpuStates (gpu.hpp:47-97)."""

    def __init__(self, gpu_count: int):
        self.gpu_count = gpu_count
        self.slots = np.zeros(gpu_count * 8, abi.INSTANCE_DTYPE)
        self.slots["job"] = -1
        self.slots["profile"] = -1
        self._seq = 0

    def _put(self, gpu: int, profile: int, start: int, state: int, job: int = -1):
        if start not in START_INDEXES[profile]:
            raise MigschedError("InvalidPlacement", f"({start},{MEMORY_SLICES[profile]}) for profile {profile}")
        m = ((1 << MEMORY_SLICES[profile]) - 1) << start
        if m & self.memory_mask(gpu, include_idle=True):
            raise MigschedError("SlicesBusy", f"instance overlaps an existing one on GPU {gpu}")
        s = self.slots[gpu * 8 + start]
        s["job"], s["seq"], s["profile"], s["state"] = job, self._seq, profile, state
        self._seq += 1

    def add_busy(self, gpu, profile, start, job):
        self._put(gpu, profile, start, abi.SLOT_BUSY, job)
        return self

    def add_idle(self, gpu, profile, start):
        self._put(gpu, profile, start, abi.SLOT_IDLE)
        return self

    def add_draining(self, gpu, profile, start):
        self._put(gpu, profile, start, abi.SLOT_DRAINING)
        return self

    def instances(self, gpu):
        """(profile, start, state, job) in instance-vector (creation) order."""
        g = self.slots[gpu * 8:(gpu + 1) * 8]
        rows = [(int(g[s]["seq"]), int(g[s]["profile"]), s, int(g[s]["state"]), int(g[s]["job"]))
                for s in range(8) if g[s]["state"] != abi.SLOT_EMPTY]
        return [r[1:] for r in sorted(rows)]

    def memory_mask(self, gpu, include_idle=False, states=None):
        m = 0
        for p, s, st, _ in self.instances(gpu):
            if states is not None and st not in states:
                continue
            if st == abi.SLOT_IDLE and not include_idle:
                continue
            m |= ((1 << MEMORY_SLICES[p]) - 1) << s
        return m

    def find_job(self, job):
        hit = np.nonzero((self.slots["job"] == job) & (self.slots["state"] == abi.SLOT_BUSY))[0]
        if len(hit) == 0:
            return None
        k = int(hit[0])
        return k // 8, k % 8, int(self.slots[k]["profile"])

    def busy_count(self, gpu):
        return sum(1 for _, _, st, _ in self.instances(gpu) if st == abi.SLOT_BUSY)

    def utilization(self, gpu):
        from .model import COMPUTE_SLICES

        return sum(COMPUTE_SLICES[p] for p, _, st, _ in self.instances(gpu) if st == abi.SLOT_BUSY) / 7.0

    def copy(self):
        c = Cluster(self.gpu_count)
        c.slots = self.slots.copy()
        c._seq = self._seq
        return c


@dataclass
class Decision:
    placed: bool
    gpu: int = -1
    start: int = 0
    size: int = 0
    reused: bool = False
    evaluated_candidates: int = 0

    @property
    def queued(self):
        return not self.placed


def schedule_batch(op: int, slots: np.ndarray, profiles: Sequence[int], cfg: SchedulerConfig,
                   gpu_count: Optional[int] = None, engine=None) -> np.ndarray:
    """Batched schedule (op = abi.OP_SCHEDULE / OP_FIRST_FIT / OP_DISPATCH)
    over n snapshots: slots shape (n, gpu_count*8) INSTANCE_DTYPE."""
    L = _bind()
    eng = engine or default_engine()
    slots = np.ascontiguousarray(slots, abi.INSTANCE_DTYPE)
    n = len(profiles)
    G = gpu_count if gpu_count is not None else slots.size // max(n, 1) // 8
    prof = np.ascontiguousarray(profiles, np.int32)
    out = np.zeros(n, abi.DECISION_DTYPE)
    c = _sched_cfg(cfg)
    _check(L.msg_schedule_batch(eng._h, op, n, G, slots.ctypes.data, prof.ctypes.data, C.byref(c),
                                out.ctypes.data), eng)
    return out


def _one(op, profile, cluster: Cluster, cfg) -> Decision:
    d = schedule_batch(op, cluster.slots[None, :], [profile], cfg, cluster.gpu_count)[0]
    return Decision(bool(d["placed"]), int(d["gpu"]), int(d["start"]), int(d["size"]), bool(d["reused"]),
                    int(d["evaluated_candidates"]))


def schedule(profile: int, cluster: Cluster, cfg: SchedulerConfig) -> Decision:
    """scheduler.cpp:47-81"""
    return _one(abi.OP_SCHEDULE, profile, cluster, cfg)


def first_fit_schedule(profile: int, cluster: Cluster, cfg: SchedulerConfig) -> Decision:
    """scheduler.cpp:83-98"""
    return _one(abi.OP_FIRST_FIT, profile, cluster, cfg)


def dispatch_schedule(profile: int, cluster: Cluster, cfg: SchedulerConfig) -> Decision:
    """scheduler.cpp:100-104"""
    return _one(abi.OP_DISPATCH, profile, cluster, cfg)


@dataclass
class Move:
    job: int
    profile: int
    from_gpu: int
    from_start: int
    to_gpu: int
    to_start: int
    kind: str
    reused: bool
    n_destroyed: int
    from_cost_before: float
    from_cost_after: float
    to_cost_before: float
    to_cost_after: float


@dataclass
class Plan:
    kind: Optional[str]
    moves: List[Move] = field(default_factory=list)
    n_iterations: int = 0
    max_evals: int = 0

    def empty(self):
        return not self.moves


def plan_batch(op: int, slots: np.ndarray, gpus: Sequence[int], threshold=0.4, enabled=True, overlap_s=0.0,
               gpu_count: Optional[int] = None, max_moves: int = 64, engine=None):
    """Batched planners over n snapshots; slots (n, G*8) are updated in place.
    Returns (summaries PLAN_SUMMARY_DTYPE[n], moves MOVE_DTYPE[n, max_moves])."""
    L = _bind()
    eng = engine or default_engine()
    assert slots.dtype == abi.INSTANCE_DTYPE and slots.flags["C_CONTIGUOUS"]
    n = len(gpus)
    G = gpu_count if gpu_count is not None else slots.size // max(n, 1) // 8
    g = np.ascontiguousarray(gpus, np.int32)
    moves = np.zeros((n, max_moves), abi.MOVE_DTYPE)
    sums = np.zeros(n, abi.PLAN_SUMMARY_DTYPE)
    _check(L.msg_plan_batch(eng._h, op, n, G, slots.ctypes.data, g.ctypes.data, threshold, int(enabled), overlap_s,
                            max_moves, moves.ctypes.data, sums.ctypes.data), eng)
    return sums, moves


def _plan(op, cluster: Cluster, gpu, threshold, enabled, overlap_s) -> Plan:
    slots = cluster.slots[None, :].copy()
    sums, moves = plan_batch(op, slots, [gpu], threshold, enabled, overlap_s, cluster.gpu_count)
    s = sums[0]
    if s["status"] != 0:
        raise MigschedError(abi.STATUS_NAMES[int(s["status"])])
    cluster.slots = slots[0].copy()
    kind = {-1: None, 0: "intra", 1: "inter"}[int(s["kind"])]
    out = Plan(kind, [], int(s["n_iterations"]), int(s["max_evals"]))
    for m in moves[0][: int(s["n_moves"])]:
        out.moves.append(Move(int(m["job"]), int(m["profile"]), int(m["from_gpu"]), int(m["from_start"]),
                              int(m["to_gpu"]), int(m["to_start"]), "inter" if m["move_kind"] else "intra",
                              bool(m["reused"]), int(m["n_destroyed"]), float(m["from_cost_before"]),
                              float(m["from_cost_after"]), float(m["to_cost_before"]), float(m["to_cost_after"])))
    return out


def plan_intra(cluster: Cluster, gpu: int, overlap_s: float = 0.0) -> Plan:
    """migration.cpp:71-123 (mutates the cluster like the reference)."""
    return _plan(abi.PLAN_INTRA, cluster, gpu, 0.4, True, overlap_s)


def plan_inter(cluster: Cluster, lazy_gpu: int, threshold: float = 0.4, overlap_s: float = 0.0) -> Plan:
    """migration.cpp:125-210; raises NotLazy like the reference."""
    return _plan(abi.PLAN_INTER, cluster, lazy_gpu, threshold, True, overlap_s)


def on_departure(cluster: Cluster, departed_gpu: int, threshold: float = 0.4, enabled: bool = True,
                 overlap_s: float = 0.0) -> Plan:
    """migration.cpp:212-220"""
    return _plan(abi.PLAN_ON_DEPARTURE, cluster, departed_gpu, threshold, enabled, overlap_s)


DEQUEUE_DTYPE = np.dtype([("job", "<i8"), ("gpu", "<i4"), ("start", "<i4"), ("size", "<i4"), ("reused", "<i4"),
                          ("evaluated_candidates", "<i4"), ("n_destroyed", "<i4")])


def try_dequeue(queue: list, cluster: Cluster, cfg: SchedulerConfig) -> list:
    """scheduler.cpp:106-121: queue is a list of (job id, profile); placed
    heads are removed from it and applied to the cluster."""
    L = _bind()
    eng = default_engine()
    qoff = np.array([0, len(queue)], np.uint64)
    qjob = np.array([j for j, _ in queue] or [0], np.int64)
    qprof = np.array([p for _, p in queue] or [0], np.int32)
    placed = np.zeros(max(len(queue), 1), DEQUEUE_DTYPE)
    n_placed = np.zeros(1, np.uint32)
    slots = cluster.slots[None, :].copy()
    c = _sched_cfg(cfg)
    _check(L.msg_try_dequeue_batch(eng._h, 1, cluster.gpu_count, slots.ctypes.data, qoff.ctypes.data,
                                   qjob.ctypes.data, qprof.ctypes.data, C.byref(c), placed.ctypes.data,
                                   n_placed.ctypes.data), eng)
    cluster.slots = slots[0].copy()
    k = int(n_placed[0])
    del queue[:k]
    return [dict(zip(DEQUEUE_DTYPE.names, (x.item() for x in row))) for row in placed[:k]]


def frag_cost_batch(slots: np.ndarray, engine=None):
    """frag_cost(gpu) (frag.cpp:60-65) of n GPU snapshots (slots shape (n, 8)
    INSTANCE_DTYPE) on the device: (numerators over 25200, doubles)."""
    L = _bind()
    eng = engine or default_engine()
    slots = np.ascontiguousarray(slots, abi.INSTANCE_DTYPE).reshape(-1, 8)
    n = len(slots)
    num = np.zeros(n, np.int32)
    cost = np.zeros(n, np.float64)
    _check(L.msg_frag_cost_batch(eng._h, n, slots.ctypes.data, num.ctypes.data, cost.ctypes.data), eng)
    return num, cost


def frag_cost(cluster: Cluster, gpu: int) -> float:
    """migsched::frag_cost of one GPU of a cluster snapshot."""
    return float(frag_cost_batch(cluster.slots[8 * gpu:8 * gpu + 8])[1][0])


def pack_gpu_word(slots8: np.ndarray) -> int:
    L = _bind()
    s = np.ascontiguousarray(slots8, abi.INSTANCE_DTYPE)
    return int(L.msg_pack_gpu_word(s.ctypes.data))
