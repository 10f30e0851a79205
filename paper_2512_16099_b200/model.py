"""Reference-shaped value types and input packing for the C ABI.

Mirrors the reference's public value types so callers (and the parity tests)
read like the reference's own code:

* MIG geometry  — profiles.hpp:11-33, profiles.cpp:8-15
* Job           — sim.hpp:13-18
* FeatureFlags / SchedulerConfig / StaticLayout — scheduler.hpp:12-29
* SimConfig     — sim.hpp:88-95
* WorkloadSpec and presets — workload.hpp:13-39, workload.cpp:129-147
* static layout presets    — scheduler.cpp:123-155

No scheduling logic lives here: everything on the hot path executes in the
CUDA engine behind include/migsched_b200.h.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import abi

# ---- MIG geometry (profiles.cpp:8-15) ------------------------------------
PROFILE_NAMES = ("7g.40gb", "4g.20gb", "3g.20gb", "2g.10gb", "1g.10gb", "1g.5gb")
COMPUTE_SLICES = (7, 4, 3, 2, 1, 1)
MEMORY_SLICES = (8, 4, 4, 2, 2, 1)
START_INDEXES = ((0,), (0,), (0, 4), (0, 2, 4), (0, 2, 4, 6), (0, 1, 2, 3, 4, 5, 6))
P7G40GB, P4G20GB, P3G20GB, P2G10GB, P1G10GB, P1G5GB = range(6)
PROFILE_COUNT = 6
# Order of WorkloadSpec::profile_mix (workload.hpp:29-30).
WORKLOAD_PROFILES = (P1G5GB, P2G10GB, P3G20GB, P4G20GB)


def find_profile(name: str) -> Optional[int]:
    """profiles.cpp:23-29."""
    try:
        return PROFILE_NAMES.index(name)
    except ValueError:
        return None


class MigschedError(RuntimeError):
    """migsched::Error (error.hpp:10-19): carries the stable code string."""

    def __init__(self, code: str, message: str = ""):
        super().__init__(f"{code}: {message}" if message else code)
        self.code = code
        self.message = message

    @classmethod
    def from_library(cls, code: str, text: str) -> "MigschedError":
        """From a library message, which is the reference's what() text
        ("Code: message"; include/migsched_b200.h): str(e) == what()."""
        prefix = code + ": "
        return cls(code, text[len(prefix):] if text.startswith(prefix) else text)


@dataclass
class FeatureFlags:
    load_balancing: bool = True
    dynamic_partitioning: bool = True
    migration: bool = True


# StaticLayout = list (per GPU) of lists of (profile, start).
StaticLayout = list


@dataclass
class SchedulerConfig:
    threshold: float = 0.4
    features: FeatureFlags = field(default_factory=FeatureFlags)
    static_layout: Optional[StaticLayout] = None


@dataclass
class SimConfig:
    sched: SchedulerConfig = field(default_factory=SchedulerConfig)
    contention_alpha: float = 0.15
    migration_overlap_s: float = 0.0
    reconfig_latency_s: float = 0.0
    gpu_count: int = 4
    seed: int = 0


@dataclass
class Job:
    id: int
    arrival_s: float
    profile: int
    service_s: float


def static_layout_preset(name: str) -> Optional[StaticLayout]:
    """scheduler.cpp:123-155 (data only)."""
    P = (P7G40GB, P4G20GB, P3G20GB, P2G10GB, P1G10GB, P1G5GB)
    _, p4, p3, p2, _, p1 = P
    if name == "static-a":
        return [
            [(p4, 0), (p3, 4)],
            [(p4, 0), (p3, 4)],
            [(p2, 0), (p2, 2), (p2, 4), (p1, 6)],
            [(p1, 0), (p1, 1), (p1, 2), (p1, 3), (p2, 4), (p1, 6)],
        ]
    if name == "static-b":
        return [
            [(p4, 0), (p2, 4), (p1, 6)],
            [(p4, 0), (p2, 4), (p1, 6)],
            [(p3, 0), (p3, 4)],
            [(p3, 0), (p2, 4), (p1, 6)],
        ]
    if name == "static-c":
        return [
            [(p4, 0), (p3, 4)],
            [(p3, 0), (p3, 4)],
            [(p2, 0), (p2, 2), (p2, 4), (p1, 6)],
            [(p2, 0), (p2, 2), (p1, 4), (p1, 5), (p1, 6)],
        ]
    return None


def static_layout_preset_names():
    return ["static-a", "static-b", "static-c"]


# ---- workload specs (workload.hpp:13-39) ---------------------------------
NORMAL, LONG = 0, 1
LOGNORMAL, EXPONENTIAL, FIXED = 0, 1, 2


@dataclass
class WorkloadSpec:
    mean_interarrival_s: float = 25.0
    query_type: int = NORMAL
    profile_mix: tuple = (0.25, 0.25, 0.25, 0.25)
    family: int = LOGNORMAL
    median_s: float = 120.0
    sigma: float = 0.8
    mean_s: float = 150.0
    value_s: float = 100.0
    job_count: int = 200
    seed: int = 0

    def to_abi(self) -> abi.MsgWorkloadSpec:
        s = abi.MsgWorkloadSpec()
        s.mean_interarrival_s = self.mean_interarrival_s
        for i in range(4):
            s.profile_mix[i] = self.profile_mix[i]
        s.median_s, s.sigma, s.mean_s, s.value_s = self.median_s, self.sigma, self.mean_s, self.value_s
        s.seed = self.seed
        s.query_type = self.query_type
        s.service_family = self.family
        s.job_count = self.job_count
        return s


def preset(name: str) -> Optional[WorkloadSpec]:
    """workload.cpp:129-147."""
    table = {
        "normal25": (25.0, NORMAL),
        "long25": (25.0, LONG),
        "normal50": (50.0, NORMAL),
        "long50": (50.0, LONG),
    }
    if name not in table:
        return None
    ia, qt = table[name]
    return WorkloadSpec(mean_interarrival_s=ia, query_type=qt)


def preset_names():
    return ["normal25", "long25", "normal50", "long50"]


# ---- packing for the C ABI ------------------------------------------------
class TraceBatch:
    """SoA + CSR trace batch (msg_trace_batch); keeps the arrays alive."""

    def __init__(self, offsets, job_id, arrival_s, profile, service_s, config_index=None):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.job_id = np.ascontiguousarray(job_id, dtype=np.int64)
        self.arrival_s = np.ascontiguousarray(arrival_s, dtype=np.float64)
        self.profile = np.ascontiguousarray(profile, dtype=np.int32)
        self.service_s = np.ascontiguousarray(service_s, dtype=np.float64)
        self.config_index = (
            None if config_index is None else np.ascontiguousarray(config_index, dtype=np.uint32)
        )
        self.n_traces = len(self.offsets) - 1
        self._c = abi.MsgTraceBatch()
        self._c.n_traces = self.n_traces
        self._c.offsets = abi.ptr(self.offsets, C.c_uint64)
        self._c.job_id = abi.ptr(self.job_id, C.c_int64)
        self._c.arrival_s = abi.ptr(self.arrival_s, C.c_double)
        self._c.profile = abi.ptr(self.profile, C.c_int32)
        self._c.service_s = abi.ptr(self.service_s, C.c_double)
        self._c.config_index = abi.ptr(self.config_index, C.c_uint32)

    @property
    def c(self):
        return C.byref(self._c)

    @property
    def n_jobs(self) -> int:
        return int(self.offsets[-1])

    @classmethod
    def from_traces(cls, traces: Sequence[Sequence[Job]], config_index=None) -> "TraceBatch":
        offsets = np.zeros(len(traces) + 1, dtype=np.uint64)
        n = 0
        for i, t in enumerate(traces):
            n += len(t)
            offsets[i + 1] = n
        ids = np.empty(n, np.int64)
        arr = np.empty(n, np.float64)
        prof = np.empty(n, np.int32)
        svc = np.empty(n, np.float64)
        k = 0
        for t in traces:
            for j in t:
                ids[k], arr[k], prof[k], svc[k] = j.id, j.arrival_s, j.profile, j.service_s
                k += 1
        return cls(offsets, ids, arr, prof, svc, config_index)

    def trace(self, t: int) -> list:
        lo, hi = int(self.offsets[t]), int(self.offsets[t + 1])
        return [
            Job(int(self.job_id[i]), float(self.arrival_s[i]), int(self.profile[i]), float(self.service_s[i]))
            for i in range(lo, hi)
        ]

    @classmethod
    def concat(cls, batches: Sequence["TraceBatch"], config_index=None) -> "TraceBatch":
        """The traces of several batches, in order, as one batch."""
        offs = [np.zeros(1, np.uint64)]
        base = 0
        for b in batches:
            offs.append(b.offsets[1:] + np.uint64(base))
            base += b.n_jobs
        return cls(np.concatenate(offs), np.concatenate([b.job_id for b in batches]),
                   np.concatenate([b.arrival_s for b in batches]), np.concatenate([b.profile for b in batches]),
                   np.concatenate([b.service_s for b in batches]), config_index)

    def subset(self, traces: Sequence[int]) -> "TraceBatch":
        offs = [0]
        parts = []
        for t in traces:
            lo, hi = int(self.offsets[t]), int(self.offsets[t + 1])
            parts.append((lo, hi))
            offs.append(offs[-1] + hi - lo)
        idx = np.concatenate([np.arange(lo, hi) for lo, hi in parts]) if parts else np.zeros(0, np.int64)
        ci = None if self.config_index is None else self.config_index[list(traces)]
        return TraceBatch(np.array(offs, np.uint64), self.job_id[idx], self.arrival_s[idx],
                          self.profile[idx], self.service_s[idx], ci)


class ConfigPack:
    """Array of msg_config (one per SimConfig); keeps layout arrays alive."""

    def __init__(self, cfgs: Sequence[SimConfig]):
        self.cfgs = list(cfgs)
        self._arr = (abi.MsgConfig * max(1, len(self.cfgs)))()
        self._keep = []
        for i, cfg in enumerate(self.cfgs):
            c = self._arr[i]
            c.threshold = cfg.sched.threshold
            c.contention_alpha = cfg.contention_alpha
            c.migration_overlap_s = cfg.migration_overlap_s
            c.reconfig_latency_s = cfg.reconfig_latency_s
            c.seed = cfg.seed
            c.gpu_count = cfg.gpu_count
            c.load_balancing = int(cfg.sched.features.load_balancing)
            c.dynamic_partitioning = int(cfg.sched.features.dynamic_partitioning)
            c.migration = int(cfg.sched.features.migration)
            layout = cfg.sched.static_layout
            c.has_static_layout = 0 if layout is None else 1
            if layout is not None:
                offs = np.zeros(len(layout) + 1, np.int32)
                profs, starts = [], []
                for g, entries in enumerate(layout):
                    for p, s in entries:
                        profs.append(int(p))
                        starts.append(int(s))
                    offs[g + 1] = len(profs)
                profs_a = np.array(profs, np.int32)
                starts_a = np.array(starts, np.int32)
                self._keep += [offs, profs_a, starts_a]
                c.layout_gpus = len(layout)
                c.layout_offsets = abi.ptr(offs, C.c_int32)
                c.layout_profile = abi.ptr(profs_a, C.c_int32)
                c.layout_start = abi.ptr(starts_a, C.c_int32)

    @property
    def c(self):
        return self._arr

    def __len__(self):
        return len(self.cfgs)
