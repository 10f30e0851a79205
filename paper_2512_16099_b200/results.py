"""Result containers shaped like the reference's SimResult (sim.hpp:75-109).

A TraceResult holds numpy views of the decoded records (include/
migsched_b200.h): `summary` (SUMMARY_DTYPE record), `per_job` (JOB_DTYPE,
job-id order like metrics()), `events` (EVENT_DTYPE, the EventLog) and
`frag_timeline` (TIMELINE_DTYPE).  For results of the CUDA engine the arrays
are zero-copy, read-only views into the library-owned buffers of the whole
batch (engine.BatchResult): a kept TraceResult keeps those buffers alive;
call .copy() on an array for an independent, writable one.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import abi
from .model import PROFILE_NAMES, MigschedError

EVENT_KIND_NAMES = (
    "arrival",
    "completion",
    "migration_start",
    "migration_end",
    "reconfig",
    "enqueue",
    "dequeue",
)


@dataclass
class TraceResult:
    status: int
    message: str
    summary: np.void
    per_job: Optional[np.ndarray] = None
    events: Optional[np.ndarray] = None
    frag_timeline: Optional[np.ndarray] = None

    @property
    def ok(self) -> bool:
        return self.status == 0

    @property
    def code(self) -> str:
        return abi.STATUS_NAMES.get(self.status, "Unknown")

    def text(self, kind: str, cfg=None) -> str:
        """The reference CLI's output file for this result, byte for byte
        (reports.cpp:14-116): kind in {"events.jsonl", "report.json",
        "report.csv", "fragcost_timeline.csv"}; report.json needs the
        SimConfig.  Formatted natively and in parallel (msg_format_text)."""
        from .engine import format_text

        return format_text(kind, self, cfg)

    def raise_for_status(self) -> "TraceResult":
        if self.status != 0:
            raise MigschedError.from_library(self.code, self.message)
        return self

    # SimReport-style accessors (sim.hpp:75-86)
    @property
    def mean_wait_s(self) -> float:
        return float(self.summary["mean_wait_s"])

    @property
    def mean_execution_s(self) -> float:
        return float(self.summary["mean_execution_s"])

    @property
    def mean_turnaround_s(self) -> float:
        return float(self.summary["mean_turnaround_s"])

    @property
    def workload_makespan_s(self) -> float:
        return float(self.summary["workload_makespan_s"])

    @property
    def migration_count(self) -> int:
        return int(self.summary["migration_count"])

    @property
    def reconfig_op_count(self) -> int:
        return int(self.summary["reconfig_op_count"])

    @property
    def complexity(self) -> tuple:
        s = self.summary
        return (
            int(s["max_arrival_frag_evals"]),
            int(s["max_intra_iter_frag_evals"]),
            int(s["max_inter_iter_frag_evals"]),
        )


def event_to_dict(ev) -> dict:
    """One decoded event as the reference's SimEvent field set (sim.hpp:33-52),
    absent optionals omitted — the same keys event_to_json_line emits
    (reports.cpp:14-37)."""
    p = int(ev["present"])
    d = {"t": float(ev["time_s"]), "kind": EVENT_KIND_NAMES[int(ev["kind"])]}
    if p & abi.HAS_JOB:
        d["job"] = int(ev["job"])
    if p & abi.HAS_GPU:
        d["gpu"] = int(ev["gpu"])
    if p & abi.HAS_PROFILE:
        d["profile"] = PROFILE_NAMES[int(ev["profile"])]
    if p & abi.HAS_START:
        d["start"] = int(ev["start"])
    if p & abi.HAS_SIZE:
        d["size"] = int(ev["size"])
    if p & abi.HAS_REUSED:
        d["reused"] = bool(ev["reused"])
    if p & abi.HAS_SCHEDULED:
        d["scheduled_s"] = float(ev["scheduled_s"])
    if p & abi.HAS_ACTION:
        d["action"] = "destroy" if int(ev["action"]) else "create"
    if p & abi.HAS_FROM_GPU:
        d["from_gpu"] = int(ev["from_gpu"])
    if p & abi.HAS_FROM_START:
        d["from_start"] = int(ev["from_start"])
    if p & abi.HAS_TO_GPU:
        d["to_gpu"] = int(ev["to_gpu"])
    if p & abi.HAS_TO_START:
        d["to_start"] = int(ev["to_start"])
    if p & abi.HAS_MOVE_KIND:
        d["move_kind"] = "inter" if int(ev["move_kind"]) else "intra"
    if p & abi.HAS_OVERLAP:
        d["overlap_s"] = float(ev["overlap_s"])
    if p & abi.HAS_COSTS:
        d["from_cost_before"] = float(ev["from_cost_before"])
        d["from_cost_after"] = float(ev["from_cost_after"])
        d["to_cost_before"] = float(ev["to_cost_before"])
        d["to_cost_after"] = float(ev["to_cost_after"])
    return d
