"""GPU parity: the CUDA engine (through the C ABI) against the unmodified
reference library, bit for bit — event logs, per-job rows, timelines and
summaries (SURVEY §8c/§8d parity bar: placements, reconfigurations and
migration sequences exact; makespan/JCT/timeline here also exact)."""
import numpy as np
import pytest

from helpers import diff_results
from oracle import refbind as rb
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.model import (
    EXPONENTIAL,
    FIXED,
    FeatureFlags,
    Job,
    SchedulerConfig,
    SimConfig,
    TraceBatch,
    WorkloadSpec,
    preset,
    preset_names,
    static_layout_preset,
)

pytestmark = pytest.mark.gpu

ALL = abi.OUT_JOBS | abi.OUT_EVENTS | abi.OUT_TIMELINE


@pytest.fixture(scope="module")
def engine():
    from paper_2512_16099_b200.engine import Engine

    return Engine(0)


def _check(engine, batch, cfgs):
    ref = rb.ref_run_batch_results(batch, cfgs)
    gpu = engine.run_batch(batch, cfgs, ALL)
    bad = [(t, d) for t, (r, g) in enumerate(zip(ref, gpu)) if (d := diff_results(r, g))]
    assert not bad, bad[:3]
    return ref, gpu


def test_c1_default_run_8_and_4_gpus(engine):
    b = rb.ref_generate_batch(preset("normal25"), [0])
    for G in (8, 4):
        ref, gpu = _check(engine, b, [SimConfig(gpu_count=G)])
    # survey anchors: C1 at 8 GPUs
    r8 = engine.run_batch(b, [SimConfig(gpu_count=8)], ALL)[0]
    assert r8.workload_makespan_s == 5550.2306096587145
    assert r8.migration_count == 74 and r8.reconfig_op_count == 156 and len(r8.events) == 704


@pytest.mark.parametrize("name", preset_names())
def test_presets_many_seeds(engine, name):
    b = rb.ref_generate_batch(preset(name), range(64))
    _check(engine, b, [SimConfig(gpu_count=4)])
    _check(engine, b, [SimConfig(gpu_count=8)])


def test_c3_ablation_combos_in_one_launch(engine):
    combos = [FeatureFlags(False, False, False), FeatureFlags(True, False, False),
              FeatureFlags(True, True, False), FeatureFlags(True, True, True)]
    cfgs = [SimConfig(gpu_count=4, sched=SchedulerConfig(
        features=f, static_layout=None if f.dynamic_partitioning else static_layout_preset("static-a")))
        for f in combos]
    parts = []
    for ia in (10.0, 15.0, 25.0, 35.0, 50.0):
        sp = preset("normal25")
        sp.mean_interarrival_s = ia
        parts.append(rb.ref_generate_batch(sp, range(8)))
    traces = [p.trace(t) for p in parts for t in range(p.n_traces)]
    all_traces = [tr for tr in traces for _ in cfgs]
    ci = [c for _ in traces for c in range(len(cfgs))]
    batch = TraceBatch.from_traces(all_traces, config_index=ci)
    _check(engine, batch, cfgs)


def test_c5_high_churn(engine):
    sp = WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, profile_mix=(0.5, 0.3, 0.2, 0.0))
    cfg = SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                    reconfig_latency_s=0.1)
    _check(engine, rb.ref_generate_batch(sp, range(128)), [cfg])


@pytest.mark.parametrize("G", [1, 2, 3, 5, 16, 32])
def test_cluster_sizes_and_ties(engine, G):
    sp = WorkloadSpec(mean_interarrival_s=4.0, family=FIXED, value_s=20.0, job_count=150)
    _check(engine, rb.ref_generate_batch(sp, range(8)),
           [SimConfig(gpu_count=G, reconfig_latency_s=0.25, migration_overlap_s=1.0)])
    sp = WorkloadSpec(mean_interarrival_s=2.0, family=EXPONENTIAL, job_count=150)
    _check(engine, rb.ref_generate_batch(sp, range(8)), [SimConfig(gpu_count=G, sched=SchedulerConfig(threshold=0.6))])


def test_shuffled_ids_equal_times_and_errors(engine):
    traces = [
        [Job(7, 0.0, 5, 10.0), Job(3, 0.0, 3, 5.0), Job(5, 0.0, 5, 10.0), Job(1, 1.0, 2, 3.0)],
        [Job(0, 10.0, 5, 1.0), Job(1, 5.0, 5, 1.0)],          # TraceUnsorted
        [Job(0, 0.0, 9, 1.0)],                                 # UnknownProfile
        [Job(0, 0.0, 5, 0.0)],                                 # BadSpec
        [Job(4, 0.0, 5, 1.0), Job(4, 1.0, 5, 1.0)],            # duplicate id
        [Job(0, -0.5, 0, 5.0), Job(1, -0.5, 0, 5.0), Job(2, 0.0, 5, 1.0)],
        [],
    ]
    _check(engine, TraceBatch.from_traces(traces), [SimConfig(gpu_count=1)])
    _check(engine, TraceBatch.from_traces(traces), [SimConfig(gpu_count=2, migration_overlap_s=3.0)])


def test_jobs_pending_and_bad_configs(engine):
    tr = [[Job(0, 0.0, 0, 10.0)]]
    cfg = SimConfig(gpu_count=1, sched=SchedulerConfig(
        features=FeatureFlags(True, False, True), static_layout=[[(2, 0), (2, 4)]]))
    _check(engine, TraceBatch.from_traces(tr), [cfg])
    for bad in (SimConfig(gpu_count=0), SimConfig(sched=SchedulerConfig(threshold=1.5)),
                SimConfig(sched=SchedulerConfig(features=FeatureFlags(True, False, True)))):
        _check(engine, TraceBatch.from_traces(tr), [bad])


def test_c2_full_ensemble_summaries(engine):
    """BASELINE config C2 at full size: 4096 traces x 200 jobs, 8 GPUs."""
    from paper_2512_16099_b200.engine import generate_batch

    b = generate_batch(preset("normal25"), 0, 4096)
    cfg = SimConfig(gpu_count=8)
    gpu = engine.run_batch(b, [cfg], 0)
    ref, _ = rb.ref_run_batch_summaries(b, [cfg], threads=0)
    got = gpu.summaries
    for f in ("status", "handler_events", "migration_count", "reconfig_op_count", "dequeue_count",
              "mean_turnaround_s", "workload_makespan_s", "mean_wait_s", "timeline_sum",
              "max_arrival_frag_evals", "max_inter_iter_frag_evals", "max_intra_iter_frag_evals"):
        assert got[f].tobytes() == ref[f].tobytes(), f
    # SURVEY Appendix B aggregate anchors
    assert int(got["handler_events"].sum()) == 1638400
    assert int(got["migration_count"].sum()) == 311361
    assert int(got["reconfig_op_count"].sum()) == 728524


def _agg_spec_cfg(entry):
    import importlib.util
    import os

    from helpers import GOLDEN

    spec_mod = importlib.util.spec_from_file_location("make_golden", os.path.join(GOLDEN, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec_mod)
    spec_mod.loader.exec_module(mg)
    sp = WorkloadSpec(**entry["spec"])
    sp.profile_mix = tuple(sp.profile_mix)
    return sp, mg.cfg_from(entry["cfg"])


@pytest.mark.parametrize("name", ["c2_4096", "c5_4096", "c3_ia25_combo0", "c3_ia25_combo1", "c3_ia25_combo2",
                                  "c3_ia25_combo3"])
def test_full_size_aggregates_vs_reference_goldens(engine, name):
    """Full-size ensembles (BASELINE configs C2, C5, a C3 load level) against
    aggregates produced by the reference library (tests/golden/aggregates.json):
    counts exact, per-trace means/makespans/timeline digests via exact
    bit-pattern checksums."""
    import json
    import os

    from helpers import GOLDEN
    from paper_2512_16099_b200.engine import generate_batch

    entry = json.load(open(os.path.join(GOLDEN, "aggregates.json")))[name]
    sp, cfg = _agg_spec_cfg(entry)
    lo, hi = entry["seeds"]
    res = engine.run_batch(generate_batch(sp, lo, hi - lo + 1), [cfg], 0)
    s = res.summaries
    assert int(s["handler_events"].sum()) == entry["handler_events"]
    assert int(s["migration_count"].sum()) == entry["migrations"]
    assert int(s["reconfig_op_count"].sum()) == entry["reconfig_ops"]
    assert int(s["dequeue_count"].sum()) == entry["dequeues"]
    for key, field in (("checksum_turnaround", "mean_turnaround_s"), ("checksum_makespan", "workload_makespan_s"),
                       ("checksum_timeline", "timeline_sum")):
        assert int(np.ascontiguousarray(s[field]).view(np.uint64).sum(dtype=np.uint64)) == entry[key], key


def test_pipelined_batch_matches_reference_with_failures(engine, monkeypatch):
    """msg_run_batch on >= 512 traces with job-row output runs pipelined
    (four trace chunks on four streams); valid, invalid and JobsPending
    traces mixed in one batch give the reference's per-trace results and the
    same bytes as the unpipelined stage / launch / collect path."""
    from paper_2512_16099_b200.engine import generate_batch

    good = generate_batch(preset("normal25"), 0, 600)
    traces = []
    for t in range(good.n_traces):
        lo, hi = int(good.offsets[t]), int(good.offsets[t + 1])
        traces.append([Job(int(good.job_id[i]), float(good.arrival_s[i]), int(good.profile[i]),
                           float(good.service_s[i])) for i in range(lo, hi)])
    traces[5] = [Job(0, 10.0, 5, 1.0), Job(1, 5.0, 5, 1.0)]  # TraceUnsorted
    traces[300] = [Job(0, 0.0, 0, 10.0)]  # 1g.5gb on a static 2g-only layout, no repartitioning: JobsPending
    traces[599] = []
    traces[7] = [Job(5, 0.0, 5, 2.0), Job(3, 1.0, 4, 1.0), Job(4, 1.0, 5, 3.0), Job(-2, 1.0, 0, 0.5)]  # rank != order
    traces[400] = [Job(1, 0.0, 5, 1.0), Job(2, 1.0, 5, 1.0), Job(1, 2.0, 5, 1.0)]  # duplicate id
    traces[450] = [Job(1, 0.0, 5, 1.0), Job(2, 1.0, 5, 0.0)]  # non-positive service
    cfgs = [SimConfig(gpu_count=8),
            SimConfig(gpu_count=1, sched=SchedulerConfig(features=FeatureFlags(True, False, True),
                                                         static_layout=[[(2, 0), (2, 4)]]))]
    b = TraceBatch.from_traces(traces, config_index=[1 if t == 300 else 0 for t in range(len(traces))])
    ref = rb.ref_run_batch_results(b, cfgs)
    piped = engine.run_batch(b, cfgs, abi.OUT_JOBS)
    monkeypatch.setenv("MSG_NO_PIPELINE", "1")
    plain = engine.run_batch(b, cfgs, abi.OUT_JOBS)
    assert piped.summaries.tobytes() == plain.summaries.tobytes()
    assert piped.jobs.tobytes() == plain.jobs.tobytes()
    assert np.array_equal(piped.job_offsets, plain.job_offsets)
    from paper_2512_16099_b200.engine import pin_batch

    monkeypatch.delenv("MSG_NO_PIPELINE")
    pinned = engine.run_batch(pin_batch(b), cfgs, abi.OUT_JOBS)  # direct inputs (chunk 0 staged: trace 7)
    assert pinned.summaries.tobytes() == piped.summaries.tobytes()
    assert pinned.jobs.tobytes() == piped.jobs.tobytes()
    assert [pinned[t].message for t in range(len(traces))] == [piped[t].message for t in range(len(traces))]
    assert piped[300].code == "JobsPending" and piped[5].code == "TraceUnsorted"
    assert piped[400].code == "BadSpec" and piped[450].code == "BadSpec" and piped[7].ok
    # Every valid trace in id order: the zero-copy launch (the kernel reads
    # the page-locked inputs in place, checks run under it); the failing
    # traces run sanitized on the device and are reported from their checks.
    traces_zc = list(traces)
    traces_zc[7] = [Job(1, 0.0, 5, 2.0), Job(3, 1.0, 4, 1.0), Job(4, 1.0, 5, 3.0), Job(9, 1.0, 0, 0.5)]
    traces_zc[8] = [Job(0, 0.0, 9, 1.0), Job(1, 0.5, 2, 1.0)]  # UnknownProfile (clamped in-kernel)
    traces_zc[9] = [Job(0, 0.0, 2, float("nan"))]  # NaN service
    bz = TraceBatch.from_traces(traces_zc, config_index=[1 if t == 300 else 0 for t in range(len(traces))])
    zc = engine.run_batch(pin_batch(bz), cfgs, abi.OUT_JOBS)
    monkeypatch.setenv("MSG_NO_ZC", "1")
    nozc = engine.run_batch(pin_batch(bz), cfgs, abi.OUT_JOBS)
    monkeypatch.delenv("MSG_NO_ZC")
    plain_z = engine.run_batch(bz, cfgs, abi.OUT_JOBS)
    for other in (nozc, plain_z):
        assert zc.summaries.tobytes() == other.summaries.tobytes()
        assert zc.jobs.tobytes() == other.jobs.tobytes()
        assert [zc[t].message for t in range(len(traces))] == [other[t].message for t in range(len(traces))]
    assert zc[8].code == "UnknownProfile" and zc[9].code == "BadSpec" and zc[7].ok and zc[5].code == "TraceUnsorted"
    ref_z = rb.ref_run_batch_results(bz, cfgs)
    for t in (7, 8, 10):  # (9: the reference accepts NaN times, this engine rejects them: DESIGN §8)
        r = ref_z[t]
        r.events = r.frag_timeline = None
        assert not diff_results(r, zc[t]), t
    bad = []
    for t, (r, g) in enumerate(zip(ref, piped)):
        r.events = r.frag_timeline = None
        if d := diff_results(r, g):
            bad.append((t, d))
    assert not bad, bad[:3]


@pytest.mark.parametrize("env", [{"MSG_PIPE_POLL": "0"}, {"MSG_JOBS_D2H": "1"}, {"MSG_ROWS_NT": "0"},
                                 {"MSG_PIPE_W": "1,2,3,1,1,1,1,1"}, {"MSG_NO_PIPELINE": "1"}, {"PINNED": "1"},
                                 {"PINNED": "1", "MSG_PIPE_POLL": "0"}, {"PINNED": "1", "MSG_NO_ZC": "1"},
                                 {"PINNED": "1", "MSG_JOBS_D2H": "1"}, {"MSG_PIPE_PROG": "0"},
                                 {"PINNED": "1", "MSG_PIPE_PROG": "0"}, {"MSG_PIPE_PROG": "1"},
                                 {"PINNED": "1", "MSG_PROG_EVERY": "128"}])
def test_pipeline_variants_agree(engine, monkeypatch, env):
    """The pipelined msg_run_batch's variants — chunk-by-chunk decode after
    each chunk's event, job records by copy, plain row stores, other chunk
    weights, no pipeline — return the same bytes as the default (records
    and a completion flag published per trace in mapped host memory)."""
    from paper_2512_16099_b200.engine import generate_batch

    from paper_2512_16099_b200.engine import pin_batch

    b = generate_batch(preset("normal25"), 5, 700)
    cfg = [SimConfig(gpu_count=8)]
    want = engine.run_batch(b, cfg, abi.OUT_JOBS)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    if env.get("PINNED"):  # inputs in page-locked memory: copied to the device in place
        b = pin_batch(b)
    got = engine.run_batch(b, cfg, abi.OUT_JOBS)
    assert got.summaries.tobytes() == want.summaries.tobytes()
    assert got.jobs.tobytes() == want.jobs.tobytes()
    again = engine.run_batch(b, cfg, abi.OUT_JOBS)  # the next run's completion flags (new epoch)
    assert again.jobs.tobytes() == want.jobs.tobytes()


def test_report_files_from_gpu_results_match_reference(engine):
    """§8f row 1: the reference CLI's files (events.jsonl, report.json,
    report.csv, fragcost_timeline.csv) formatted natively from the GPU
    engine's results equal the reference serializers' bytes."""
    kinds = ("events.jsonl", "report.json", "report.csv", "fragcost_timeline.csv")
    for spec, cfg, seeds in ((preset("normal25"), SimConfig(gpu_count=8), [0, 7]),
                             (WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2,
                                           profile_mix=(0.5, 0.3, 0.2, 0.0)),
                              SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                                        reconfig_latency_s=0.1), [3])):
        b = rb.ref_generate_batch(spec, seeds)
        ref = rb.ref_run_batch_results(b, [cfg], texts=True)
        gpu = engine.run_batch(b, [cfg], ALL)
        for r, g in zip(ref, gpu):
            for kind, want in zip(kinds, r.texts):
                assert g.text(kind, cfg) == want, kind

def test_zero_copy_ragged_traces(engine, monkeypatch):
    """Zero copy over page-locked inputs with trace lengths around the fetch
    blocks (the first block holds 8 jobs, then 24, then 32 each) and 512+
    traces (pipelined): the same bytes as the staged path and as the plain
    stage / launch / collect path, and the reference's results."""
    from paper_2512_16099_b200.engine import generate_batch, pin_batch

    lens = [1, 7, 8, 9, 31, 32, 33, 40, 63, 64, 65, 200, 1000, 3000]
    traces = []
    for t in range(520):
        n = lens[t % len(lens)]
        sp = preset("normal25")
        sp.job_count = n
        b1 = generate_batch(sp, 1000 + t, 1)
        traces.append([Job(int(b1.job_id[i]), float(b1.arrival_s[i]), int(b1.profile[i]), float(b1.service_s[i]))
                       for i in range(n)])
    b = TraceBatch.from_traces(traces)
    cfg = [SimConfig(gpu_count=8)]
    zc = engine.run_batch(pin_batch(b), cfg, abi.OUT_JOBS)
    monkeypatch.setenv("MSG_NO_ZC", "1")
    staged = engine.run_batch(pin_batch(b), cfg, abi.OUT_JOBS)
    monkeypatch.delenv("MSG_NO_ZC")
    monkeypatch.setenv("MSG_NO_PIPELINE", "1")
    plain = engine.run_batch(b, cfg, abi.OUT_JOBS)
    monkeypatch.delenv("MSG_NO_PIPELINE")
    for other in (staged, plain):
        assert zc.summaries.tobytes() == other.summaries.tobytes()
        assert zc.jobs.tobytes() == other.jobs.tobytes()
    ref = rb.ref_run_batch_results(TraceBatch.from_traces(traces[:len(lens)]), cfg)
    for t, r in enumerate(ref):
        r.events = r.frag_timeline = None
        assert not diff_results(r, zc[t]), (t, lens[t])
