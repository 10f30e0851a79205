"""ctypes binding of libmigsched_b200.so (include/migsched_b200.h).

The product path: every call here executes the sm_100a kernels.  If the
shared library or a CUDA device is missing, the calls raise — there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from . import abi
from .model import ConfigPack, MigschedError, SimConfig, TraceBatch, WorkloadSpec
from .results import TraceResult

LIB_PATH = os.environ.get("MSG_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmigsched_b200.so")

_lib = None


def lib():
    """Load the CUDA engine library (fails loudly if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"CUDA engine library missing: {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32
    sig = {
        "msg_status_name": (C.c_char_p, [C.c_int]),
        "msg_engine_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "msg_engine_destroy": (None, [vp]),
        "msg_engine_last_error": (C.c_char_p, [vp]),
        "msg_engine_launch_count": (u64, [vp]),
        "msg_engine_device_info": (C.c_int, [vp, C.c_char_p, C.c_size_t, C.POINTER(i32)]),
        "msg_run_batch": (C.c_int, [vp, vp, vp, u32, u32, C.POINTER(vp)]),
        "msg_stage": (C.c_int, [vp, vp, vp, u32, u32, C.POINTER(vp)]),
        "msg_launch": (C.c_int, [vp, vp]),
        "msg_collect": (C.c_int, [vp, vp, C.POINTER(vp)]),
        "msg_staged_free": (None, [vp]),
        "msg_staged_handler_events": (u64, [vp]),
        "msg_engine_sync": (C.c_int, [vp]),
        "msg_time_launch": (C.c_int, [vp, vp, C.POINTER(C.c_float)]),
        "msg_engine_flush_l2": (C.c_int, [vp]),
        "msg_engine_flush_l2_async": (C.c_int, [vp]),
        "msg_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
        "msg_host_free": (None, [vp]),
        "msg_result_n_traces": (u32, [vp]),
        "msg_result_summary": (vp, [vp, u32]),
        "msg_result_jobs": (vp, [vp, u32, C.POINTER(u64)]),
        "msg_result_events": (vp, [vp, u32, C.POINTER(u64)]),
        "msg_result_timeline": (vp, [vp, u32, C.POINTER(u64)]),
        "msg_result_message": (C.c_char_p, [vp, u32]),
        "msg_result_free": (None, [vp]),
        "msg_result_summaries": (vp, [vp]),
        "msg_result_all_jobs": (vp, [vp, C.POINTER(C.POINTER(u64)), C.POINTER(u64)]),
        "msg_workload_preset": (C.c_int, [C.c_char_p, vp]),
        "msg_generate": (C.c_int, [vp, vp, vp, vp, vp]),
        "msg_generate_many": (C.c_int, [vp, u64, u32, i32, vp, vp, vp, vp, vp]),
        "msg_trace_load": (C.c_int, [C.c_char_p, C.POINTER(vp), C.c_char_p, C.c_size_t]),
        "msg_format_text": (C.c_int, [C.c_int32, vp, vp, vp, u64, vp, u64, vp, u64, C.POINTER(vp),
                                      C.POINTER(C.c_size_t)]),
        "msg_text_free": (None, [vp]),
        "msg_trace_file_jobs": (u64, [vp]),
        "msg_trace_file_ids": (vp, [vp]),
        "msg_trace_file_arrival": (vp, [vp]),
        "msg_trace_file_profile": (vp, [vp]),
        "msg_trace_file_service": (vp, [vp]),
        "msg_trace_file_free": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(st: int, eng=None):
    if st != 0:
        msg = ""
        if eng is not None and eng._h:
            msg = lib().msg_engine_last_error(eng._h).decode()
        raise MigschedError.from_library(abi.STATUS_NAMES.get(st, str(st)), msg)


class Staged:
    """A batch resident in HBM (msg_stage); launch/collect any number of times."""

    def __init__(self, engine: "Engine", handle, n_traces: int, keep, out_flags: int):
        self.engine = engine
        self.out_flags = out_flags
        self._h = handle
        self.n_traces = n_traces
        self._keep = keep

    def launch(self):
        _check(lib().msg_launch(self.engine._h, self._h), self.engine)

    def time_launch(self) -> float:
        ms = C.c_float()
        _check(lib().msg_time_launch(self.engine._h, self._h, C.byref(ms)), self.engine)
        return ms.value

    def collect(self) -> "BatchResult":
        r = C.c_void_p()
        _check(lib().msg_collect(self.engine._h, self._h, C.byref(r)), self.engine)
        return _decode(r, self.out_flags)

    @property
    def handler_events(self) -> int:
        return int(lib().msg_staged_handler_events(self._h))

    def free(self):
        if self._h:
            lib().msg_staged_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Engine:
    """One CUDA device + stream (msg_engine)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        st = lib().msg_engine_create(device, C.byref(h))
        if st != 0:
            raise MigschedError(abi.STATUS_NAMES.get(st, str(st)),
                                f"cannot create the CUDA engine on device {device}")
        self._h = h

    def close(self):
        if self._h:
            lib().msg_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self) -> int:
        return int(lib().msg_engine_launch_count(self._h))

    def device_info(self):
        buf = C.create_string_buffer(256)
        sm = C.c_int32()
        lib().msg_engine_device_info(self._h, buf, 256, C.byref(sm))
        return buf.value.decode(), sm.value

    def sync(self):
        _check(lib().msg_engine_sync(self._h), self)

    def flush_l2(self, sync: bool = True):
        """Write 256 MiB (more than L2) on the engine stream; sync=False
        leaves it queued so the next timed launch starts on a busy device."""
        _check((lib().msg_engine_flush_l2 if sync else lib().msg_engine_flush_l2_async)(self._h), self)

    def run_batch(self, batch: TraceBatch, cfgs: Sequence[SimConfig], out_flags: int = abi.OUT_JOBS) -> "BatchResult":
        """migsched::run over every trace of the batch (sim.cpp:504-507)."""
        pack = ConfigPack(cfgs)
        r = C.c_void_p()
        _check(lib().msg_run_batch(self._h, C.addressof(batch._c), C.addressof(pack.c[0]), len(pack),
                                   out_flags, C.byref(r)), self)
        return _decode(r, out_flags)

    def stage(self, batch: TraceBatch, cfgs: Sequence[SimConfig], out_flags: int = 0) -> Staged:
        pack = ConfigPack(cfgs)
        h = C.c_void_p()
        _check(lib().msg_stage(self._h, C.addressof(batch._c), C.addressof(pack.c[0]), len(pack), out_flags,
                               C.byref(h)), self)
        return Staged(self, h, batch.n_traces, (batch, pack), out_flags)


class _ResultHolder:
    """Owns a msg_batch_result; numpy views into it keep this object alive."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            if self.handle:
                lib().msg_result_free(self.handle)
        except Exception:
            pass


class _Mem:
    """Array-interface wrapper over library memory that pins its owner."""

    def __init__(self, ptr, nbytes, owner):
        self.__array_interface__ = {"data": (ptr, False), "shape": (nbytes,), "typestr": "|u1", "version": 3}
        self.owner = owner


def _view(ptr, n, dtype, owner):
    """Zero-copy, read-only numpy view of n records at ptr, keeping `owner`
    (the whole batch's result buffers) alive; .copy() for an independent,
    writable array."""
    if not ptr or n == 0:
        return np.zeros(0, dtype)
    v = np.asarray(_Mem(ptr, n * dtype.itemsize, owner)).view(dtype)
    v.flags.writeable = False
    return v


class _Pinned:
    """Page-locked host memory from msg_host_alloc, freed with its last view."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        _check(lib().msg_host_alloc(max(int(nbytes), 1), C.byref(p)))
        self.ptr = p.value

    def __del__(self):
        try:
            lib().msg_host_free(self.ptr)
        except Exception:
            pass


def pinned_empty(n: int, dtype) -> np.ndarray:
    """Writable numpy array of n elements in page-locked host memory."""
    dt = np.dtype(dtype)
    mem = _Pinned(n * dt.itemsize)
    if n == 0:
        return np.zeros(0, dt)
    return np.asarray(_Mem(mem.ptr, n * dt.itemsize, mem)).view(dt)


def pin_batch(batch: TraceBatch) -> TraceBatch:
    """A copy of `batch` whose job arrays live in page-locked host memory:
    msg_run_batch then copies them to the device in place (no host staging
    copy).  Results are identical either way."""
    arrs = {}
    for name in ("job_id", "arrival_s", "profile", "service_s"):
        src = getattr(batch, name)
        dst = pinned_empty(len(src), src.dtype)
        dst[:] = src
        arrs[name] = dst
    return TraceBatch(batch.offsets.copy(), arrs["job_id"], arrs["arrival_s"], arrs["profile"], arrs["service_s"],
                      None if batch.config_index is None else batch.config_index.copy())


class BatchResult:
    """Results of one batch (msg_batch_result), decoded lazily.

    `summaries` (SUMMARY_DTYPE[n]) and `jobs` (JOB_DTYPE, all traces,
    `job_offsets`) are zero-copy, read-only views into the library's
    buffers (any view keeps the whole batch's buffers alive); indexing
    or iterating yields per-trace TraceResult objects shaped like the
    reference's SimResult."""

    def __init__(self, handle, flags: int):
        L = lib()
        self._owner = _ResultHolder(handle)
        self._h = handle
        self.flags = flags
        self.n = int(L.msg_result_n_traces(handle))
        self.summaries = _view(L.msg_result_summaries(handle), self.n, abi.SUMMARY_DTYPE, self._owner)
        self._jobs = None  # (jobs view, job_offsets), built on first use

    def _job_views(self):
        if self._jobs is None:
            cnt = C.c_uint64()
            offp = C.POINTER(C.c_uint64)()
            jp = lib().msg_result_all_jobs(self._h, C.byref(offp), C.byref(cnt))
            if jp:
                self._jobs = (_view(jp, cnt.value, abi.JOB_DTYPE, self._owner),
                              np.ctypeslib.as_array(offp, shape=(self.n + 1,)).copy())
            else:
                self._jobs = (None, None)
        return self._jobs

    @property
    def jobs(self):
        """Every valid trace's job rows (JOB_DTYPE), trace-major; None without OUT_JOBS."""
        return self._job_views()[0]

    @property
    def job_offsets(self):
        """Row offsets per trace (n + 1), or None without OUT_JOBS."""
        return self._job_views()[1]

    def __len__(self):
        return self.n

    def __getitem__(self, t):
        if isinstance(t, slice):
            return [self[i] for i in range(*t.indices(self.n))]
        if t < 0:
            t += self.n
        if not 0 <= t < self.n:
            raise IndexError(t)
        L = lib()
        cnt = C.c_uint64()
        summ = self.summaries[t]
        st = int(summ["status"])
        msg = L.msg_result_message(self._h, t).decode() if st != 0 else ""
        jobs = self.jobs[self.job_offsets[t]:self.job_offsets[t + 1]] if self.jobs is not None else None
        res = TraceResult(st, msg, summ, jobs, None, None)
        if self.flags & abi.OUT_EVENTS:
            res.events = _view(L.msg_result_events(self._h, t, C.byref(cnt)), cnt.value, abi.EVENT_DTYPE, self._owner)
        if self.flags & abi.OUT_TIMELINE:
            res.frag_timeline = _view(L.msg_result_timeline(self._h, t, C.byref(cnt)), cnt.value,
                                      abi.TIMELINE_DTYPE, self._owner)
        return res

    def __iter__(self):
        for t in range(self.n):
            yield self[t]

    @property
    def handler_events(self) -> int:
        return int(self.summaries["handler_events"].sum())


def _decode(r, flags: int) -> BatchResult:
    return BatchResult(r, flags)


_default_engines: dict = {}


def default_engine(device: Optional[int] = None) -> Engine:
    """One cached Engine per CUDA device; `device` defaults to this
    process's device (torch's current device, else LOCAL_RANK, else 0)."""
    if device is None:
        from .ensemble import local_device

        device = local_device()
    eng = _default_engines.get(device)
    if eng is None:
        eng = _default_engines[device] = Engine(device)
    return eng


def run(trace, cfg: SimConfig, out_flags: int = abi.OUT_JOBS | abi.OUT_EVENTS | abi.OUT_TIMELINE) -> TraceResult:
    """Drop-in for migsched::run(trace, cfg) (sim.hpp:114): raises
    MigschedError with the reference's error code on failure."""
    batch = TraceBatch.from_traces([list(trace)])
    res = default_engine().run_batch(batch, [cfg], out_flags)[0]
    return res.raise_for_status()


def generate(spec: WorkloadSpec):
    """migsched::generate (workload.cpp:98-127) -> list of Job."""
    from .model import Job

    n = spec.job_count
    ids = np.zeros(max(n, 1), np.int64)
    arr = np.zeros(max(n, 1), np.float64)
    prof = np.zeros(max(n, 1), np.int32)
    svc = np.zeros(max(n, 1), np.float64)
    s = spec.to_abi()
    _check(lib().msg_generate(C.byref(s), ids.ctypes.data, arr.ctypes.data, prof.ctypes.data, svc.ctypes.data))
    return [Job(int(ids[i]), float(arr[i]), int(prof[i]), float(svc[i])) for i in range(n)]


TEXT_KINDS = {"events.jsonl": 0, "report.json": 1, "report.csv": 2, "fragcost_timeline.csv": 3}


def format_text(kind: str, res: TraceResult, cfg: Optional[SimConfig] = None) -> str:
    """reports.cpp serializers over one TraceResult (see TraceResult.text)."""
    L = lib()
    k = TEXT_KINDS[kind]

    def ptr(a):
        return (a.ctypes.data if a is not None and len(a) else None), (len(a) if a is not None else 0)

    ev, nev = ptr(res.events)
    jb, njb = ptr(res.per_job)
    tl, ntl = ptr(res.frag_timeline)
    summ = np.ascontiguousarray(np.array([res.summary], abi.SUMMARY_DTYPE))
    pack = ConfigPack([cfg]) if cfg is not None else None
    cptr = C.addressof(pack.c[0]) if pack is not None else None
    out, n = C.c_void_p(), C.c_size_t()
    _check(L.msg_format_text(k, summ.ctypes.data, cptr, ev, nev, jb, njb, tl, ntl, C.byref(out), C.byref(n)))
    try:
        return C.string_at(out, n.value).decode()
    finally:
        L.msg_text_free(out)


def load_trace(path: str) -> TraceBatch:
    """migsched::load_trace (workload.cpp:151-199): a JSONL trace file as a
    one-trace TraceBatch (jobs stable-sorted by arrival).  Raises
    MigschedError with the reference's code (ParseError, UnknownProfile) and
    message on a bad file."""
    L = lib()
    h = C.c_void_p()
    msg = C.create_string_buffer(512)
    st = L.msg_trace_load(os.fsencode(path), C.byref(h), msg, len(msg))
    if st != 0:
        text = msg.value.decode(errors="replace")
        raise MigschedError.from_library(abi.STATUS_NAMES.get(st, str(st)), text)
    try:
        n = int(L.msg_trace_file_jobs(h))

        def arr(ptr, dt):
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(dt)), shape=(n,)).copy() if n else np.zeros(0, dt)

        ids = arr(L.msg_trace_file_ids(h), C.c_int64)
        a = arr(L.msg_trace_file_arrival(h), C.c_double)
        p = arr(L.msg_trace_file_profile(h), C.c_int32)
        s = arr(L.msg_trace_file_service(h), C.c_double)
    finally:
        L.msg_trace_file_free(h)
    return TraceBatch(np.array([0, n], np.uint64), ids, a, p, s)


def generate_batch(spec: WorkloadSpec, seed0: int, n_seeds: int, threads: int = 0) -> TraceBatch:
    """n_seeds traces with seeds seed0.. as one TraceBatch (host threads)."""
    n = spec.job_count * n_seeds
    offsets = np.zeros(n_seeds + 1, np.uint64)
    ids = np.zeros(max(n, 1), np.int64)
    arr = np.zeros(max(n, 1), np.float64)
    prof = np.zeros(max(n, 1), np.int32)
    svc = np.zeros(max(n, 1), np.float64)
    s = spec.to_abi()
    _check(lib().msg_generate_many(C.byref(s), seed0, n_seeds, threads, offsets.ctypes.data, ids.ctypes.data,
                                   arr.ctypes.data, prof.ctypes.data, svc.ctypes.data))
    return TraceBatch(offsets, ids[:n], arr[:n], prof[:n], svc[:n])
