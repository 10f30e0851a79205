"""ORACLE / TEST INFRASTRUCTURE: ctypes bindings to the reference library and
to the C restatement.  See oracle/__init__.py for the usage rules."""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.model import ConfigPack, SimConfig, TraceBatch, WorkloadSpec
from paper_2512_16099_b200.results import TraceResult

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmigsched_ref.so")
PORT_SO = os.path.join(HERE, "_port", "liboracle_port.so")

_ref = None
_port = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def port_available() -> bool:
    return os.path.exists(PORT_SO)


def _bind_result_api(lib, prefix):
    vp = C.c_void_p
    f = getattr(lib, prefix + "run")
    f.restype = vp
    f.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
    getattr(lib, prefix + "result_status").restype = C.c_int
    getattr(lib, prefix + "result_status").argtypes = [vp]
    getattr(lib, prefix + "result_message").restype = C.c_char_p
    getattr(lib, prefix + "result_message").argtypes = [vp]
    getattr(lib, prefix + "result_summary").restype = C.c_void_p
    getattr(lib, prefix + "result_summary").argtypes = [vp]
    for name in ("events", "jobs", "timeline"):
        g = getattr(lib, prefix + "result_" + name)
        g.restype = C.c_void_p
        g.argtypes = [vp, C.POINTER(C.c_uint64)]
    getattr(lib, prefix + "result_free").argtypes = [vp]


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference library not built: {REF_SO} (run make -C oracle)")
        lib = C.CDLL(REF_SO)
        _bind_result_api(lib, "ref_")
        lib.ref_result_text.restype = C.c_char_p
        lib.ref_result_text.argtypes = [C.c_void_p, C.c_int]
        lib.ref_run_batch.restype = C.c_double
        lib.ref_run_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_int32, C.c_void_p]
        lib.ref_hardware_threads.restype = C.c_int32
        lib.ref_generate.restype = C.c_int
        lib.ref_generate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_schedule.restype = C.c_int
        lib.ref_schedule.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        lib.ref_plan.restype = C.c_int
        lib.ref_plan.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_double, C.c_int32,
                                 C.c_double, C.c_uint32, C.c_void_p, C.c_void_p]
        lib.ref_try_dequeue.restype = C.c_int
        lib.ref_try_dequeue.argtypes = [C.c_int32, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
        lib.ref_frag_cost.argtypes = [C.c_uint8] * 4 + [C.POINTER(C.c_int64)] * 2
        lib.ref_oracle_run_all.restype = C.c_int
        lib.ref_enumerate_states.restype = C.c_int64
        lib.ref_enumerate_states.argtypes = [C.c_int, C.c_void_p, C.c_int64]
        lib.ref_load_trace.restype = C.c_void_p
        lib.ref_load_trace.argtypes = [C.c_char_p]
        for n in ("ref_trace_code", "ref_trace_message"):
            getattr(lib, n).restype = C.c_char_p
            getattr(lib, n).argtypes = [C.c_void_p]
        lib.ref_trace_jobs.restype = C.c_int64
        lib.ref_trace_jobs.argtypes = [C.c_void_p]
        lib.ref_trace_get.argtypes = [C.c_void_p] * 5
        lib.ref_trace_free.argtypes = [C.c_void_p]
        lib.ref_save_trace.restype = C.c_int
        lib.ref_save_trace.argtypes = [C.c_char_p, C.c_int64] + [C.c_void_p] * 4
        _ref = lib
    return _ref


def port_lib():
    global _port
    if _port is None:
        if not port_available():
            raise RuntimeError(f"oracle port not built: {PORT_SO} (run make -C oracle)")
        lib = C.CDLL(PORT_SO)
        _bind_result_api(lib, "port_")
        lib.port_frag_k.restype = C.c_int32
        lib.port_frag_k.argtypes = [C.c_uint8] * 4
        lib.port_run_batch.restype = C.c_double
        lib.port_run_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p]
        _port = lib
    return _port


def _collect(lib, prefix, h) -> TraceResult:
    status = getattr(lib, prefix + "result_status")(h)
    msg = getattr(lib, prefix + "result_message")(h).decode()
    sp = getattr(lib, prefix + "result_summary")(h)
    summary = np.frombuffer(C.string_at(sp, abi.SUMMARY_DTYPE.itemsize), abi.SUMMARY_DTYPE)[0].copy()

    def arr(name, dtype):
        n = C.c_uint64()
        p = getattr(lib, prefix + "result_" + name)(h, C.byref(n))
        if n.value == 0:
            return np.zeros(0, dtype)
        return np.frombuffer(C.string_at(p, n.value * dtype.itemsize), dtype).copy()

    return TraceResult(
        status,
        msg,
        summary,
        arr("jobs", abi.JOB_DTYPE),
        arr("events", abi.EVENT_DTYPE),
        arr("timeline", abi.TIMELINE_DTYPE),
    )


def _run(lib, prefix, batch: TraceBatch, cfgs: ConfigPack, trace: int) -> TraceResult:
    ci = 0 if batch.config_index is None else int(batch.config_index[trace])
    h = getattr(lib, prefix + "run")(C.addressof(batch._c), trace, C.addressof(cfgs.c[ci]))
    try:
        return _collect(lib, prefix, h)
    finally:
        getattr(lib, prefix + "result_free")(h)


def ref_run_batch_results(batch: TraceBatch, cfgs: Sequence[SimConfig], texts=False):
    """Full results of the reference run() for every trace of the batch."""
    lib = ref_lib()
    pack = ConfigPack(cfgs)
    out = []
    for t in range(batch.n_traces):
        ci = 0 if batch.config_index is None else int(batch.config_index[t])
        h = lib.ref_run(C.addressof(batch._c), t, C.addressof(pack.c[ci]))
        try:
            r = _collect(lib, "ref_", h)
            if texts and r.status == 0:
                r.texts = tuple(lib.ref_result_text(h, i).decode() for i in range(4))
        finally:
            lib.ref_result_free(h)
        out.append(r)
    return out


def port_run_batch_results(batch: TraceBatch, cfgs: Sequence[SimConfig]):
    lib = port_lib()
    pack = ConfigPack(cfgs)
    return [_run(lib, "port_", batch, pack, t) for t in range(batch.n_traces)]


def ref_run_batch_summaries(batch: TraceBatch, cfgs: Sequence[SimConfig], threads: int = 0):
    """Summaries only, on a std::thread pool; returns (summaries, seconds)."""
    lib = ref_lib()
    pack = ConfigPack(cfgs)
    out = np.zeros(batch.n_traces, abi.SUMMARY_DTYPE)
    secs = lib.ref_run_batch(C.addressof(batch._c), C.addressof(pack.c[0]), len(pack), threads,
                             out.ctypes.data)
    return out, secs


def port_run_batch_summaries(batch: TraceBatch, cfgs: Sequence[SimConfig]):
    lib = port_lib()
    pack = ConfigPack(cfgs)
    out = np.zeros(batch.n_traces, abi.SUMMARY_DTYPE)
    secs = lib.port_run_batch(C.addressof(batch._c), C.addressof(pack.c[0]), len(pack), out.ctypes.data)
    return out, secs


def hardware_threads() -> int:
    return int(ref_lib().ref_hardware_threads())


def ref_generate(spec: WorkloadSpec):
    lib = ref_lib()
    n = spec.job_count
    ids = np.zeros(n, np.int64)
    arr = np.zeros(n, np.float64)
    prof = np.zeros(n, np.int32)
    svc = np.zeros(n, np.float64)
    s = spec.to_abi()
    st = lib.ref_generate(C.byref(s), ids.ctypes.data, arr.ctypes.data, prof.ctypes.data, svc.ctypes.data)
    if st != 0:
        raise RuntimeError(abi.STATUS_NAMES.get(st, st))
    return ids, arr, prof, svc


def ref_generate_batch(spec: WorkloadSpec, seeds: Sequence[int]) -> TraceBatch:
    parts = []
    for sd in seeds:
        sp = WorkloadSpec(**{**spec.__dict__, "seed": int(sd)})
        parts.append(ref_generate(sp))
    n = spec.job_count
    offsets = np.arange(len(parts) + 1, dtype=np.uint64) * n
    return TraceBatch(
        offsets,
        np.concatenate([p[0] for p in parts]),
        np.concatenate([p[1] for p in parts]),
        np.concatenate([p[2] for p in parts]),
        np.concatenate([p[3] for p in parts]),
    )


def ref_schedule(op: int, slots: np.ndarray, profile: int, threshold=0.4, lb=True, dyn=True):
    """slots: INSTANCE_DTYPE array of gpu_count*8."""
    lib = ref_lib()
    cfg = abi.MsgSchedConfig()
    cfg.threshold = threshold
    cfg.load_balancing = int(lb)
    cfg.dynamic_partitioning = int(dyn)
    out = np.zeros(1, abi.DECISION_DTYPE)
    slots = np.ascontiguousarray(slots, abi.INSTANCE_DTYPE)
    st = lib.ref_schedule(op, len(slots) // 8, slots.ctypes.data, profile, C.byref(cfg), out.ctypes.data)
    return st, out[0]


def ref_plan(op: int, slots: np.ndarray, gpu: int, threshold=0.4, enabled=True, overlap_s=0.0,
             max_moves=64):
    lib = ref_lib()
    slots = np.ascontiguousarray(slots, abi.INSTANCE_DTYPE).copy()
    moves = np.zeros(max_moves, abi.MOVE_DTYPE)
    summ = np.zeros(1, abi.PLAN_SUMMARY_DTYPE)
    st = lib.ref_plan(op, len(slots) // 8, slots.ctypes.data, gpu, threshold, int(enabled), overlap_s,
                      max_moves, moves.ctypes.data, summ.ctypes.data)
    n = min(int(summ[0]["n_moves"]), max_moves)
    return st, summ[0], moves[:n], slots


def ref_frag_cost(bc, bm, kc, km):
    lib = ref_lib()
    num, den = C.c_int64(), C.c_int64()
    lib.ref_frag_cost(bc, bm, kc, km, C.byref(num), C.byref(den))
    return num.value, den.value


def ref_enumerate_states(depth: int):
    lib = ref_lib()
    cap = 1 << 22
    buf = np.zeros(cap, np.int32)
    n = lib.ref_enumerate_states(depth, buf.ctypes.data, cap)
    assert n >= 0
    states, i = [], 0
    while i < n:
        k = int(buf[i])
        states.append([(int(buf[i + 1 + 2 * j]), int(buf[i + 2 + 2 * j])) for j in range(k)])
        i += 1 + 2 * k
    return states


def ref_try_dequeue(slots: np.ndarray, queue, threshold=0.4, lb=True, dyn=True):
    """queue: list of (job, profile). Returns (status, placed list of dicts, slots)."""
    lib = ref_lib()
    cfg = abi.MsgSchedConfig()
    cfg.threshold = threshold
    cfg.load_balancing = int(lb)
    cfg.dynamic_partitioning = int(dyn)
    slots = np.ascontiguousarray(slots, abi.INSTANCE_DTYPE).copy()
    dt = np.dtype([("job", "<i8"), ("gpu", "<i4"), ("start", "<i4"), ("size", "<i4"), ("reused", "<i4"),
                   ("evaluated_candidates", "<i4"), ("n_destroyed", "<i4")])
    placed = np.zeros(max(len(queue), 1), dt)
    n = np.zeros(1, np.uint32)
    qj = np.array([j for j, _ in queue] or [0], np.int64)
    qp = np.array([p for _, p in queue] or [0], np.int32)
    st = lib.ref_try_dequeue(len(slots) // 8, slots.ctypes.data, len(queue), qj.ctypes.data, qp.ctypes.data,
                             C.byref(cfg), placed.ctypes.data, n.ctypes.data)
    return st, [dict(zip(dt.names, (x.item() for x in r))) for r in placed[: int(n[0])]], slots


def ref_load_trace(path: str):
    """migsched::load_trace -> (code, message, ids, arrival, profile, service);
    code '' on success."""
    import os

    lib = ref_lib()
    h = lib.ref_load_trace(os.fsencode(path))
    try:
        code = lib.ref_trace_code(h).decode()
        msg = lib.ref_trace_message(h).decode(errors="replace")
        n = int(lib.ref_trace_jobs(h))
        ids = np.zeros(n, np.int64)
        arr = np.zeros(n, np.float64)
        prof = np.zeros(n, np.int32)
        svc = np.zeros(n, np.float64)
        if n:
            lib.ref_trace_get(h, ids.ctypes.data, arr.ctypes.data, prof.ctypes.data, svc.ctypes.data)
    finally:
        lib.ref_trace_free(h)
    return code, msg, ids, arr, prof, svc


def ref_save_trace(path: str, ids, arrival, profile, service) -> None:
    """migsched::save_trace (workload.cpp:201-213)."""
    import os

    ids = np.ascontiguousarray(ids, np.int64)
    arrival = np.ascontiguousarray(arrival, np.float64)
    profile = np.ascontiguousarray(profile, np.int32)
    service = np.ascontiguousarray(service, np.float64)
    if ref_lib().ref_save_trace(os.fsencode(path), len(ids), ids.ctypes.data, arrival.ctypes.data,
                                profile.ctypes.data, service.ctypes.data):
        raise RuntimeError("save_trace failed")


def ref_ablation(batch: TraceBatch, cfg: SimConfig):
    """The reference CLI's ablate (tools/migsched.cpp:64-99) on the
    reference library: (ablation.json text, table text)."""
    lib = ref_lib()
    f = lib.ref_ablation
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t]
    pack = ConfigPack([cfg])
    js = C.create_string_buffer(1 << 16)
    tb = C.create_string_buffer(1 << 12)
    if f(C.addressof(batch._c), C.addressof(pack.c[0]), js, len(js), tb, len(tb)):
        raise RuntimeError("reference ablation failed")
    return js.value.decode(), tb.value.decode()


def ref_oracle_clusters(depth: int, clusters: np.ndarray, threads: int = 0):
    """Brute-force scheduler oracle (oracle.cpp:233-296) for clusters given as
    rows of state indices into enumerate_states(depth): expected (gpu, start)
    per cluster and profile, shape (n, 6) each; -1 when nothing fits."""
    lib = ref_lib()
    f = lib.ref_oracle_clusters
    f.restype = None
    f.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int]
    idx = np.ascontiguousarray(clusters, np.int32)
    n, G = idx.shape
    g = np.zeros((n, 6), np.int32)
    s = np.zeros((n, 6), np.int32)
    f(depth, G, idx.ctypes.data, n, g.ctypes.data, s.ctypes.data, threads)
    return g, s
