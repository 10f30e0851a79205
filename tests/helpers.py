"""Shared test helpers: result diffing and the test-only emulation binding."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.model import ConfigPack

HERE = os.path.dirname(os.path.abspath(__file__))
EMU_SO = os.path.join(HERE, "emu", "_build", "libemu.so")
_emu = None

SUMMARY_COMPARE = [
    "status",
    "handler_events",
    "n_events",
    "timeline_samples",
    "migration_count",
    "reconfig_op_count",
    "enqueue_count",
    "dequeue_count",
    "max_arrival_frag_evals",
    "max_intra_iter_frag_evals",
    "max_inter_iter_frag_evals",
    "mean_wait_s",
    "mean_execution_s",
    "mean_turnaround_s",
    "workload_makespan_s",
    "timeline_sum",
]


def emu_lib():
    """The CPU emulation of the device code (tests/emu) — test-only."""
    global _emu
    if _emu is None:
        if not os.path.exists(EMU_SO):
            import subprocess

            subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "emu")])
        from oracle import refbind

        lib = C.CDLL(EMU_SO)
        refbind._bind_result_api(lib, "emu_")
        _emu = lib
    return _emu


def emu_run_batch_results(batch, cfgs):
    from oracle import refbind

    lib = emu_lib()
    pack = ConfigPack(cfgs)
    return [refbind._run(lib, "emu_", batch, pack, t) for t in range(batch.n_traces)]


def diff_results(a, b, check_text=False) -> str:
    """'' if the two TraceResults are bit-identical, else a description of
    the first difference."""
    if a.status != b.status:
        return f"status {a.status} vs {b.status} ({a.message} | {b.message})"
    if a.status != 0:
        return ""
    for f in SUMMARY_COMPARE:
        x, y = a.summary[f], b.summary[f]
        if isinstance(x, (np.floating, float)):
            if np.float64(x).tobytes() != np.float64(y).tobytes():
                return f"summary.{f}: {x!r} vs {y!r}"
        elif x != y:
            return f"summary.{f}: {x!r} vs {y!r}"
    for name in ("events", "per_job", "frag_timeline"):
        x, y = getattr(a, name), getattr(b, name)
        if x is None or y is None:
            continue
        if len(x) != len(y):
            n = min(len(x), len(y))
            first = next((i for i in range(n) if x[i].tobytes() != y[i].tobytes()), n)
            return f"{name}: length {len(x)} vs {len(y)}; first difference at {first}: " + (
                f"{x[first]} vs {y[first]}" if first < n else "")
        if x.tobytes() != y.tobytes():
            i = next(i for i in range(len(x)) if x[i].tobytes() != y[i].tobytes())
            return f"{name}[{i}]: {x[i]} vs {y[i]}"
    return ""
