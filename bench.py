"""Benchmark: scheduling decisions/s of the GPU engine (BASELINE.json metric).

Headline workload (BASELINE.json configs[1], "C2"): the ensemble of 4096
seeded synthetic traces (preset normal25, 200 jobs each, seeds 0..4095, the
reference generator) on 8-GPU A100 MIG clusters with load balancing +
dynamic partitioning + migration; one warp simulates one trace.  A
"decision" is one handler event (Arrival, valid Completion, MigrationEnd,
ServiceStart timer pop) — 1,638,400 per C2 ensemble, identical on both
engines because results are bit-exact.

  value  device-timed: inputs resident in HBM, L2 flushed before every step,
         CUDA events on the engine stream, max over ranks
  e2e    the public C-ABI call msg_run_batch from host buffers (validation,
         staging, H2D, kernel, summaries + per-job rows to the host, decode)
         plus the per-trace summary gather to rank 0, every step

N>1 (torchrun): the named ensemble is split into N contiguous trace ranges
(strong scaling; no data-path collective, one final gather).
`weak` beside it: every rank simulates its own 4096 traces.  C3 and C5 are
split the same way; C4 (one 16384-GPU cluster) runs over all ranks' GPUs as
device groups exchanging packed keys through peer memory.

Other keys: `c1` (configs[0]: the reference's default run, one trace,
latency through the C ABI with the full event log), `configs` (C3, C5),
`c4` (configs[3] prefix, with the reference timed on the same prefix),
`roofline` (the event loop against its real bound, instruction issue; its
HBM fraction beside it), `scorer_sweep` (the HBM-bound scorer at thresholds
0.4 / 0.0 / 1.0), `cpu_baseline` (the reference library on the box's host
cores, T = all and T = 1, best of 3).

--impl reference: the unmodified reference library (oracle/_ref, compiled
from /root/reference/proj/src with its Release flags; traces from the
reference's own generator) on all host threads, the same 4096-trace C2
ensemble per step, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scheduling decisions/sec (traces×events) at 1/2/4/8 B200 vs host-CPU ref; makespan parity"
UNIT = "decisions/s"
TRACES = 4096
JOBS = 200
GPUS_PER_CLUSTER = 8
C4_GPUS = 16384


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--traces", type=int, default=TRACES)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-c1", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--c4-arrivals", type=int, default=20000)
    ap.add_argument("--c4-cpu-arrivals", type=int, default=2000,
                    help="prefix timed on both engines for the same-prefix CPU comparison")
    ap.add_argument("--c4-peer-arrivals", type=int, default=2000,
                    help="prefix split over all ranks' GPUs (device groups) at N>1")
    ap.add_argument("--one-gpu", action="store_true",
                    help="N>1 test mode: every rank on cuda:0, gloo for the host-side collectives "
                         "(exercises every N>1 leg on a one-GPU box; times are not scaling numbers)")
    return ap.parse_args()


ONE_GPU = False  # --one-gpu: all ranks share cuda:0, collectives over gloo on host tensors


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if ONE_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def coll_device():
    """Device of the tensors handed to torch.distributed collectives."""
    return "cpu" if ONE_GPU else "cuda"


def host_cpu():
    """The host the CPU numbers were taken on."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count() or 1
    return {"model": model, "logical_cpus": os.cpu_count(), "usable_cpus": usable}


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    (nvidia_ml_py) every ~2 ms when available, else nvidia-smi (~10/s)."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, [4 reason flags])
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._t = None

    def _nvml_handle(self):
        import pynvml

        pynvml.nvmlInit()
        try:  # the CUDA device's own board (CUDA_VISIBLE_DEVICES may renumber)
            import torch

            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            nv, h = self._nvml_handle()
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.source = "nvml"

            def sample():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                return float(sm), float(mx), [bool(r & b) for b in bits]
        except Exception:
            def sample():
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                return float(f[0]), float(f[1]), [x == "Active" for x in f[2:6]]

        def loop():
            while not self._stop.is_set():
                try:
                    self.rows.append(sample())
                except Exception:
                    pass
                self._stop.wait(0.002 if self.source == "nvml" else 0.1)

        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()

    def stop(self) -> dict:
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2][i]})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "sm_mhz_min": min(r[0] for r in self.rows), "reasons": reasons, "samples": len(self.rows),
                "source": self.source}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def ncu_summary(name):
    """A kernel's entry in the committed ncu summary (profiles/ncu_summary.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(name, {})
    except Exception:
        return {}


# ---------------------------------------------------------------- reference
def ref_best(batch, cfgs, threads, reps=3):
    """The reference library over a batch: one warm-up pass, then the best
    of `reps` (BASELINE.md §2 protocol).  Returns (summaries, best seconds,
    all seconds)."""
    from oracle import refbind

    refbind.ref_run_batch_summaries(batch, cfgs, threads=threads)
    times = []
    for _ in range(reps):
        s, secs = refbind.ref_run_batch_summaries(batch, cfgs, threads=threads)
        times.append(secs)
    return s, min(times), times


def cpu_baseline(batch, cfg):
    """The unmodified reference library (checker build, oracle/_ref) on the
    box's host cores over the same C2 traces: T = all host threads over the
    whole ensemble and T = 1 over a 512-trace slice, each best of 3 after a
    warm-up pass."""
    from oracle import refbind

    if not refbind.ref_available():
        sub = batch.subset(range(min(256, batch.n_traces)))
        s, secs = refbind.port_run_batch_summaries(sub, [cfg])
        return {"value": float(s["handler_events"].sum() / secs), "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"{sub.n_traces} traces x {JOBS} jobs (C2 subset), oracle C port, 1 thread",
                "host": host_cpu()}
    threads = refbind.hardware_threads()
    s, best, times = ref_best(batch, [cfg], threads)
    ev = int(s["handler_events"].sum())
    n1 = min(512, batch.n_traces)
    s1, best1, _ = ref_best(batch.subset(range(n1)), [cfg], 1)
    return {"value": ev / best, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"all {batch.n_traces} C2 traces x {JOBS} jobs per pass, reference library -O3 "
                      f"-ffp-contract=off on {threads} std::threads; best of 3 after a warm-up pass",
            "seconds_best": best, "seconds_all": times,
            "t1": {"value": float(s1["handler_events"].sum()) / best1, "cores": 1,
                   "sample": f"{n1} of the traces, best of 3"},
            "host": host_cpu()}


def run_reference_arm(args, rank, world):
    """The reference's own CPU implementation of the path (oracle/_ref: the
    unmodified library compiled from its sources), traces from its own
    generator, the same 4096-trace C2 ensemble per step, all host threads.
    Rank 0 only; nothing from the product library is loaded."""
    if rank != 0:
        return
    from oracle import refbind
    from paper_2512_16099_b200.model import SimConfig, preset

    if not refbind.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmigsched_ref.so not built"}))
        return
    cfg = SimConfig(gpu_count=GPUS_PER_CLUSTER)
    batch = refbind.ref_generate_batch(preset("normal25"), range(args.traces))
    threads = refbind.hardware_threads()
    for _ in range(args.warmup):
        refbind.ref_run_batch_summaries(batch, [cfg], threads=threads)
    step_s, tot_ev = [], 0
    for _ in range(args.steps):
        s, secs = refbind.ref_run_batch_summaries(batch, [cfg], threads=threads)
        tot_ev += int(s["handler_events"].sum())
        step_s.append(secs)
    v = tot_ev / sum(step_s)
    n1 = min(512, batch.n_traces)
    s1, best1, _ = ref_best(batch.subset(range(n1)), [cfg], 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(step_s) / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the reference's own generator, seeds 0..4095)",
        "config": {"workload": f"C2 ensemble: {batch.n_traces} traces x {JOBS} jobs normal25, {GPUS_PER_CLUSTER}-GPU "
                               "clusters, all techniques (per step)", "traces_per_step": batch.n_traces,
                   "jobs_per_trace": JOBS, "gpus_per_cluster": GPUS_PER_CLUSTER, "same_config": True},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"all {batch.n_traces} traces per step, {args.steps} steps after {args.warmup} "
                                   "warm-up steps", "best_step_value": tot_ev / args.steps / min(step_s),
                         "t1": {"value": float(s1["handler_events"].sum()) / best1, "cores": 1,
                                "sample": f"{n1} of the traces, best of 3"},
                         "host": host_cpu()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------- ours
def scorer_sweep(eng, peaks, peak_kind, threshold=0.4):
    """Batched arrival scorer over 4096 snapshots of a 16384-GPU cluster
    (512 MiB of packed state, above L2): the HBM-bound decision kernel
    (SURVEY §8d).  Algorithmic bytes = 8 B per GPU word + 16 B out per
    snapshot + 1 B profile.  threshold 0.4: ~77% of the random words are
    Busy; 1.0: every GPU with a free slice is Lazy (pass 1 scores ~all
    words); 0.0: no GPU is Lazy (every snapshot is decided by the Busy
    pass)."""
    import ctypes as C

    import torch

    from paper_2512_16099_b200 import abi, decisions
    from paper_2512_16099_b200.model import SchedulerConfig

    L = decisions._bind()
    B, G = 4096, C4_GPUS
    gen = torch.Generator(device="cuda").manual_seed(1)
    rnd = torch.randint(0, 1 << 30, (B, G), device="cuda", dtype=torch.int64, generator=gen)
    bm = rnd & 0x7F
    words = (bm | (bm << 8) | (bm << 16)).contiguous()
    del rnd, bm
    # two copies, used alternately: each timed launch reads 512 MiB (4x L2)
    # that the previous 512 MiB of reads did not touch, so nothing it reads
    # can still be in L2
    bufs = (words, words.clone())
    prof = torch.randint(0, 6, (B,), device="cuda", dtype=torch.uint8, generator=gen)
    out = torch.empty(B * 2, device="cuda", dtype=torch.int64)
    res = {}
    for thr in (threshold, 0.0, 1.0):
        cfg = decisions._sched_cfg(SchedulerConfig(threshold=thr))
        ms = C.c_float()
        times = {"alt": [], "flush": []}
        for i in range(20):
            # even samples: inputs larger than L2, the two copies alternated
            # (no flush); odd samples: after the 256 MiB L2-flush write, whose
            # dirty lines the scorer's reads then evict (write-backs inside
            # the timed launch), reported beside it
            mode = "flush" if i & 1 else "alt"
            if mode == "flush":
                eng.flush_l2()
            st = L.msg_time_score_device(eng._h, B, G, bufs[(i >> 1) & 1].data_ptr(), prof.data_ptr(),
                                         C.byref(cfg), out.data_ptr(), C.byref(ms))
            if st != 0:
                return {"error": abi.STATUS_NAMES.get(st, st)}
            if i >= 4:
                times[mode].append(ms.value)
        t = statistics.median(times["alt"]) * 1e-3
        achieved = (B * G * 8 + B * 17) / t / 1e9
        res[thr] = {"ms": t * 1e3, "achieved": achieved, "frac": achieved / peaks["hbm_gbs"],
                    "ms_after_l2_flush_write": statistics.median(times["flush"])}
    head = res[threshold]
    sc = ncu_summary("score_kernel")
    return {"kernel": "score_kernel", "bound": "hbm", "achieved": head["achieved"], "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": head["frac"], "peak_kind": peak_kind,
            "traffic": sc.get("dram_bytes_per_launch"), "traffic_source": sc.get("round"), "ms": head["ms"],
            "threshold": threshold,
            "by_threshold": {str(k): v for k, v in res.items()},
            "workload": f"{B} snapshots x {G} GPUs (8 B words), one arrival each; inputs 4x L2, two copies"
                        " read alternately (ms_after_l2_flush_write: after a 256 MiB L2-flush write instead)"}


def c1_line(eng):
    """BASELINE.json configs[0], the reference's default run (one trace,
    normal25 seed 0, 8 GPUs, all techniques): per-call latency of
    msg_run_batch with the full event log, job rows and timeline, against the
    reference's run() on one host thread (best of 5)."""
    from paper_2512_16099_b200 import abi
    from paper_2512_16099_b200.engine import generate_batch
    from paper_2512_16099_b200.model import SimConfig, preset

    ALL = abi.OUT_JOBS | abi.OUT_EVENTS | abi.OUT_TIMELINE
    b = generate_batch(preset("normal25"), 0, 1)
    cfg = SimConfig(gpu_count=GPUS_PER_CLUSTER)
    for _ in range(5):
        r = eng.run_batch(b, [cfg], ALL)
    ev = int(r[0].summary["handler_events"])
    lat = []
    for _ in range(50):
        t0 = time.perf_counter()
        r = eng.run_batch(b, [cfg], ALL)
        lat.append(time.perf_counter() - t0)
    st = eng.stage(b, [cfg], ALL)
    st.launch()
    eng.sync()
    dev = statistics.median(st.time_launch() for _ in range(20))
    med = statistics.median(lat)
    out = {"workload": "C1: one trace, normal25 seed 0, 200 jobs, 8 GPUs, all techniques; msg_run_batch with event "
                       "log + job rows + timeline, from host arrays", "handler_events": ev,
           "value": ev / med, "unit": UNIT, "latency_ms": med * 1e3, "latency_min_ms": min(lat) * 1e3,
           "kernel_ms": dev, "events": len(r[0].events)}
    try:
        from oracle import refbind

        if refbind.ref_available():
            s, best, _ = ref_best(b, [cfg], 1, reps=5)
            out["cpu_reference"] = {"value": float(s["handler_events"][0]) / best, "latency_ms": best * 1e3,
                                    "cores": 1, "sample": "the same trace, reference run(), best of 5"}
            out["speedup_vs_reference_latency"] = best / med
    except Exception as e:  # noqa: BLE001
        out["cpu_reference"] = f"unavailable: {e}"
    return out


def c4_spec(n):
    from paper_2512_16099_b200.model import preset

    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 2048
    sp.job_count = n
    return sp


def c4_golden(n):
    """The reference's own result and wall time on the n-arrival prefix,
    if frozen in tests/golden/c4_prefix.npz (make_c4_golden.py)."""
    try:
        import numpy as np

        with np.load(os.path.join(ROOT, "tests", "golden", "c4_prefix.npz")) as z:
            if f"n{n}/summary" not in z.files:
                return None
            return z[f"n{n}/summary"][0], float(z[f"n{n}/seconds"][0])
    except Exception:
        return None


def c4_line(eng, args, rank, world):
    """C4 (BASELINE.json configs[3]): one 16384-GPU cluster, normal25 at
    ia = 25/2048 s, seed 0 — bounded prefixes of the 1M-arrival trace.  N=1:
    the sharded block engine (one 16-CTA thread-block cluster) on the first
    c4_arrivals (20K) and c4_cpu_arrivals (2K) arrivals, the reference's
    run() on one host thread on the same 2K prefix.  N>1: the c4_peer_arrivals
    prefix split over all ranks' GPUs as device groups (packed-key exchanges
    through peer memory); wall time max over ranks."""
    import numpy as np
    import torch

    from paper_2512_16099_b200 import abi
    from paper_2512_16099_b200.engine import generate_batch
    from paper_2512_16099_b200.model import SimConfig

    cfg = SimConfig(gpu_count=C4_GPUS)
    out = {"workload": f"C4 prefixes: {C4_GPUS}-GPU cluster, normal25 at ia=25/2048 s, seed 0 (first n of 1M "
                       "arrivals)", "unit": UNIT}
    if world == 1:
        def gpu_prefix(n):
            b = generate_batch(c4_spec(n), 0, 1)
            st = eng.stage(b, [cfg], abi.OUT_JOBS)
            st.launch()
            eng.sync()
            ms = st.time_launch()
            res = st.collect()[0]
            ev = int(res.summary["handler_events"])
            g = c4_golden(n)
            pin = None
            if g is not None:
                want = g[0]
                pin = all(int(res.summary[f]) == int(want[f]) for f in ("handler_events", "migration_count",
                                                                        "reconfig_op_count", "dequeue_count")) and \
                    all(np.float64(res.summary[f]).tobytes() == np.float64(want[f]).tobytes()
                        for f in ("mean_turnaround_s", "workload_makespan_s", "mean_wait_s"))
            return b, {"arrivals": n, "value": ev / (ms * 1e-3), "kernel_s": ms * 1e-3, "handler_events": ev,
                       "status": res.code, "matches_reference_golden": pin}

        _, head = gpu_prefix(args.c4_arrivals)
        out.update(head)
        out.update({"gpus": 1, "engine": "sharded block engine, one thread-block cluster of 16 CTAs"})
        b2, small = gpu_prefix(args.c4_cpu_arrivals)
        out["same_prefix"] = small
        try:
            from oracle import refbind

            if refbind.ref_available():
                s, secs = refbind.ref_run_batch_summaries(b2, [cfg], threads=1)
                cpu = float(s["handler_events"][0]) / secs
                small["cpu_reference"] = {"value": cpu, "seconds": secs, "cores": 1,
                                          "sample": f"reference run() on the same {args.c4_cpu_arrivals}-arrival "
                                                    "prefix, one pass (one host thread: run() is sequential)"}
                small["speedup_vs_reference"] = small["value"] / cpu
        except Exception as e:  # noqa: BLE001
            small["cpu_reference"] = f"unavailable: {e}"
        g = c4_golden(args.c4_arrivals)
        if g is not None:
            out["reference_build_box"] = {
                "arrivals": args.c4_arrivals, "seconds": g[1],
                "value": float(g[0]["handler_events"]) / g[1],
                "note": "the reference's run() on this prefix when its golden was frozen "
                        "(tests/golden/make_c4_golden.py, build box, one thread) — not this host"}
        return out
    import torch.distributed as dist

    from paper_2512_16099_b200.peer import PeerGroup, torch_allgather

    n = args.c4_peer_arrivals
    batch = generate_batch(c4_spec(n), 0, 1)
    group = PeerGroup(eng, world, rank, n, torch_allgather())
    try:
        group.run(batch, cfg, 0)  # warm-up
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = group.run(batch, cfg, 0)
        secs = time.perf_counter() - t0
    finally:
        group.close()
    t = torch.tensor([secs], dtype=torch.float64, device=coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ev = int(res[0].summary["handler_events"])
        g = c4_golden(n)
        out.update({"arrivals": n, "value": ev / float(t.item()), "seconds": float(t.item()), "handler_events": ev,
                    "gpus": world, "status": res[0].code,
                    "engine": f"device groups over {world} GPUs (peer-memory exchange of packed keys)",
                    "matches_reference_golden": None if g is None else bool(
                        np.float64(res[0].summary["workload_makespan_s"]).tobytes()
                        == np.float64(g[0]["workload_makespan_s"]).tobytes())})
    return out


def split_batch(batch, rank, world):
    from paper_2512_16099_b200.ensemble import shard_range

    lo, hi = shard_range(rank, world, batch.n_traces)
    return batch.subset(range(lo, hi))


def other_configs(eng, rank, world, allreduce_max, allreduce_sum):
    """BASELINE.json configs[2] (C3: 4 technique combinations x 1024 seeds x
    5 arrival loads, 4-GPU clusters, one launch) and configs[4] (C5: 4096
    high-churn traces, overlap 0.5 s, reconfiguration latency 0.1 s, 8-GPU
    clusters): device-timed decisions/s with L2 flushed, each split into N
    contiguous trace ranges at N>1 (max over ranks); on rank 0 at N=1 the
    reference library on all host threads over 1024 of the traces."""
    from oracle import refbind
    from paper_2512_16099_b200.engine import generate_batch
    from paper_2512_16099_b200.model import (FeatureFlags, SchedulerConfig, SimConfig, TraceBatch, WorkloadSpec,
                                             preset, static_layout_preset)

    out = {}
    combos = [FeatureFlags(False, False, False), FeatureFlags(True, False, False), FeatureFlags(True, True, False),
              FeatureFlags(True, True, True)]
    cfgs = [SimConfig(gpu_count=4, sched=SchedulerConfig(
        features=f, static_layout=None if f.dynamic_partitioning else static_layout_preset("static-a")))
        for f in combos]
    parts, index = [], []
    for load in (10.0, 15.0, 25.0, 35.0, 50.0):
        sp = preset("normal25")
        sp.mean_interarrival_s = load
        b = generate_batch(sp, 0, 1024)
        for k in range(4):
            parts.append(b)
            index += [k] * b.n_traces
    c3 = TraceBatch.concat(parts, config_index=index)
    c5 = generate_batch(WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2,
                                     profile_mix=(0.5, 0.3, 0.2, 0.0)), 0, 4096)
    c5cfg = [SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                       reconfig_latency_s=0.1)]
    for name, whole, cs, desc in (
            ("c3", c3, cfgs, "4 technique combinations x 1024 seeds x 5 loads (ia 10/15/25/35/50 s), 4-GPU clusters"),
            ("c5", c5, c5cfg, "4096 high-churn traces (ia 0.4 s, median 4 s), overlap 0.5 s, latency 0.1 s, 8 GPUs")):
        batch = split_batch(whole, rank, world)
        st = eng.stage(batch, cs, 0)
        for _ in range(3):
            st.launch()
        eng.sync()
        res = st.collect()
        ok = all(r.ok for r in res)
        ms = []
        for _ in range(5):
            eng.flush_l2()
            ms.append(st.time_launch())
        t = allreduce_max(statistics.median(ms))
        ev = allreduce_sum(float(st.handler_events))
        line = {"workload": desc, "traces": whole.n_traces, "decisions_per_step": int(ev),
                "value": ev / (t * 1e-3), "unit": UNIT, "ms_per_step": t, "ok": ok,
                "parallelism": f"split into {world} contiguous trace range(s)"}
        if rank == 0 and world == 1 and refbind.ref_available():
            threads = refbind.hardware_threads()
            sub = batch.subset(range(0, batch.n_traces, max(1, batch.n_traces // 1024)))
            s_, best, _ = ref_best(sub, cs, threads)
            line["cpu_reference"] = {"value": float(s_["handler_events"].sum() / best), "cores": threads,
                                     "sample": f"{sub.n_traces} of the traces (every "
                                               f"{max(1, batch.n_traces // 1024)}th), reference library, best of 3"}
        out[name] = line
    return out


def main():
    global ONE_GPU
    args = parse()
    ONE_GPU = args.one_gpu
    rank, world, local = dist_env()
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        if ONE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
        return

    import gc

    import numpy as np
    import torch

    from paper_2512_16099_b200 import abi
    from paper_2512_16099_b200.engine import Engine, generate_batch
    from paper_2512_16099_b200.ensemble import gather_records, rank_seeds, shard_range
    from paper_2512_16099_b200.model import SimConfig, preset

    torch.cuda.set_device(local)
    eng = Engine(local)
    cfg = SimConfig(gpu_count=GPUS_PER_CLUSTER)
    spec = preset("normal25")
    spec.job_count = JOBS
    lo, hi = shard_range(rank, world, args.traces)
    batch = generate_batch(spec, lo, hi - lo)  # this rank's contiguous share of the named ensemble

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def allreduce(x, op):
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=coll_device())
        dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}[op])
        return float(t.item())

    def device_steps(staged, steps):
        """Max over ranks of the mean device time of `steps` launches, each
        after an L2 flush (inputs are 14 MB, well inside the 126 MB L2)."""
        barrier()
        ms = []
        for _ in range(steps):
            eng.flush_l2()
            ms.append(staged.time_launch())
        barrier()
        return allreduce(sum(ms) / len(ms), "max")

    staged = eng.stage(batch, [cfg], 0)
    for _ in range(max(args.warmup, 3)):
        staged.launch()
    eng.sync()
    res = staged.collect()
    bad = [r.code for r in res if not r.ok]
    if bad:
        raise SystemExit(f"simulation failed: {bad[:3]}")
    events_local = staged.handler_events

    clocks = ClockSampler(local)
    clocks.start()
    launches0 = eng.launch_count
    ms_step = device_steps(staged, args.steps)
    gpu_launches = eng.launch_count - launches0
    clk = clocks.stop()
    total_events = allreduce(float(events_local), "sum")
    value = total_events / (ms_step * 1e-3)

    # e2e: the public C-ABI call with the inputs in page-locked host memory
    # (msg_host_alloc: what the contract's "H2D from pinned host memory"
    # assumes) + the summary gather, every step.  The kernel reads the inputs
    # in place over PCIe (arrival f64, service f64, profile i32 per job, plus
    # the trace table) and publishes the job records (24 B) and summaries
    # into mapped host memory as it goes.
    from paper_2512_16099_b200.engine import pin_batch

    pbatch = pin_batch(batch)
    h2d = allreduce(float(batch.n_jobs * (8 + 8 + 4) + batch.n_traces * 56), "sum")  # + DevTrace (56 B)
    d2h = allreduce(float(batch.n_traces * (120 + 4 + 8) + batch.n_jobs * 24), "sum")  # DevSummary, flag, progress
    gdev = "cuda" if world > 1 and not ONE_GPU else None

    def e2e_step():
        out = eng.run_batch(pbatch, [cfg], abi.OUT_JOBS)
        return out, gather_records(np.ascontiguousarray(out.summaries), world, gdev)

    for _ in range(max(3, args.warmup)):  # as timed: the previous result is alive during the next call
        out, gathered = e2e_step()
    barrier()
    e2e_s = []
    gc.disable()  # as timeit does: no collector pauses inside the timed calls
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out, gathered = e2e_step()
        e2e_s.append(time.perf_counter() - t0)
    gc.enable()
    barrier()
    e2e_ms = allreduce(1e3 * sum(e2e_s) / len(e2e_s), "max")
    e2e_value = total_events / (e2e_ms * 1e-3)
    if rank == 0:
        assert len(gathered) == args.traces and int(gathered["handler_events"].sum()) == int(total_events)

    peaks, peak_kind = measured_peaks()
    # The event loop's bound is instruction issue (a serial dependent chain
    # per trace, all state on chip): warp instructions per launch (ncu,
    # profiles/ncu_summary.json) over the SMs' issue rate, 4 warp-instr per
    # SM per clock at the clock sampled during the timed region.
    sim = ncu_summary("sim_kernel")
    name, sms = eng.device_info()
    mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    instr = sim.get("instructions_executed", 0.0) * (batch.n_traces / sim.get("traces", TRACES))
    issue_peak = sms * 4 * mhz * 1e6 / 1e9  # G warp-instr/s
    achieved_issue = instr / (ms_step * 1e-3) / 1e9
    algo = batch.n_jobs * (8 + 8 + 1 + 24) + batch.n_traces * 128
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference generator: preset normal25, seeds 0..4095)",
        "config": {
            "workload": f"C2 ensemble: {args.traces} traces x {JOBS} jobs (seeds 0..{args.traces - 1}), "
                        f"{GPUS_PER_CLUSTER}-GPU A100 MIG clusters, load balancing + dynamic partitioning + "
                        "migration",
            "traces": args.traces, "jobs_per_trace": JOBS, "gpus_per_cluster": GPUS_PER_CLUSTER,
            "decisions_per_step": int(total_events),
            "parallelism": f"named ensemble split into {world} contiguous trace range(s), one per GPU",
            "l2": "flushed (256 MiB write) before every timed step",
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_ms,
                "ms_median": 1e3 * statistics.median(e2e_s), "ms_min": 1e3 * min(e2e_s), "ms_max": 1e3 * max(e2e_s),
                "ms_steps": [round(1e3 * x, 4) for x in e2e_s],
                "path": "msg_run_batch(page-locked host SoA traces) -> per-job rows + summaries, then the per-trace summary "
                        "gather to rank 0"},
        "gpu_launches": int(gpu_launches),
        "roofline": {"kernel": "sim_kernel", "bound": "issue", "achieved": achieved_issue, "peak": issue_peak,
                     "unit": "G warp-instr/s", "frac": achieved_issue / issue_peak,
                     "peak_kind": f"{sms} SMs x 4 issue slots x {mhz:.0f} MHz (sampled)",
                     "traffic": sim.get("dram_bytes_per_launch"),
                     "instructions_per_launch": instr, "instructions_source": sim.get("round"),
                     "hbm": {"achieved": algo / (ms_step * 1e-3) / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                             "frac": algo / (ms_step * 1e-3) / 1e9 / peaks["hbm_gbs"], "peak_kind": peak_kind,
                             "algorithmic_bytes": algo},
                     "ncu": {k: sim.get(k) for k in ("issue_slots_busy_pct", "achieved_occupancy_pct",
                                                     "warp_execution_efficiency_threads", "registers_per_thread")},
                     "note": "event loop: one warp per trace, a serial dependent chain of ~400 events with all "
                             "state in shared memory/registers — bounded by instruction issue, not HBM "
                             "(SURVEY 8d); the HBM-bound kernel is scorer_sweep"},
        "clocks": clk,
        "device": name,
    }
    if world > 1:  # weak scaling beside the named split: every rank its own 4096 traces
        s0, n = rank_seeds(rank, args.traces)
        wb = generate_batch(spec, s0, n)
        ws = eng.stage(wb, [cfg], 0)
        for _ in range(3):
            ws.launch()
        eng.sync()
        wms = device_steps(ws, args.steps)
        ws.collect()  # handler_events is counted from the collected summaries
        wev = allreduce(float(ws.handler_events), "sum")
        line["weak"] = {"value": wev / (wms * 1e-3), "unit": UNIT, "ms_per_step": wms,
                        "traces_per_gpu": args.traces, "scaling": "weak"}
        ws.free()
    staged.free()
    if rank == 0 and not args.no_sweep:
        line["scorer_sweep"] = scorer_sweep(eng, peaks, peak_kind)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(batch, cfg)
    if rank == 0 and not args.no_c1:
        try:
            line["c1"] = c1_line(eng)
        except Exception as e:  # noqa: BLE001
            line["c1"] = {"error": f"{type(e).__name__}: {e}"}
    if not args.no_configs:
        try:
            cf = other_configs(eng, rank, world, lambda x: allreduce(x, "max"), lambda x: allreduce(x, "sum"))
        except Exception as e:  # noqa: BLE001
            cf = {"error": f"{type(e).__name__}: {e}"}
        if rank == 0:
            line["configs"] = cf
    if not args.no_c4:
        try:
            c4 = c4_line(eng, args, rank, world)
        except Exception as e:  # noqa: BLE001 (reported, the headline line still prints)
            c4 = {"error": f"{type(e).__name__}: {e}"}
        if rank == 0:
            line["c4"] = c4
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as tdist

        tdist.barrier()
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
