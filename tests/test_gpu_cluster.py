"""Block engine (clusters of more than 32 GPUs) on the B200 against the
unmodified reference library, up to the 16384-GPU C4 cluster (prefix of the
C4 trace: the full 1M-arrival trace takes the reference ~12 h)."""
import numpy as np
import pytest

from helpers import diff_results, diff_results_relaxed_timeline
from oracle import refbind as rb
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.model import SchedulerConfig, SimConfig, TraceBatch, WorkloadSpec, preset

pytestmark = pytest.mark.gpu
ALL = abi.OUT_JOBS | abi.OUT_EVENTS | abi.OUT_TIMELINE


@pytest.fixture(scope="module")
def engine():
    from paper_2512_16099_b200.engine import Engine

    return Engine(0)


def _check(engine, batch, cfgs, relaxed=False):
    ref = rb.ref_run_batch_results(batch, cfgs)
    got = engine.run_batch(batch, cfgs, ALL)
    diff = diff_results_relaxed_timeline if relaxed else diff_results
    bad = [(t, d) for t, (r, g) in enumerate(zip(ref, got)) if (d := diff(r, g))]
    assert not bad, bad[:2]


@pytest.mark.parametrize("G", [33, 64, 200, 512])
def test_large_clusters_bit_exact(engine, G):
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 * 8 / G
    sp.job_count = 500
    _check(engine, rb.ref_generate_batch(sp, [0, 1]), [SimConfig(gpu_count=G)])
    churn = WorkloadSpec(mean_interarrival_s=0.4 * 8 / G, median_s=4.0, sigma=1.2, job_count=500)
    _check(engine, rb.ref_generate_batch(churn, [2]),
           [SimConfig(gpu_count=G, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                      reconfig_latency_s=0.1)])


def test_mixed_small_and_large_traces_one_call(engine):
    sp = preset("normal25")
    sp.job_count = 150
    b = rb.ref_generate_batch(sp, range(6))
    traces = [b.trace(t) for t in range(6)]
    cfgs = [SimConfig(gpu_count=8), SimConfig(gpu_count=40), SimConfig(gpu_count=4)]
    batch = TraceBatch.from_traces(traces, config_index=[0, 1, 2, 1, 0, 2])
    _check(engine, batch, cfgs)


def test_c4_prefix_16384_gpus(engine):
    """C4 (BASELINE configs[3]): 16384 GPUs, normal25 at ia = 25/2048 s, seed
    0 — first 600 arrivals; timeline to 1e-9 relative (above 512 GPUs)."""
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 2048
    sp.job_count = 600
    _check(engine, rb.ref_generate_batch(sp, [0]), [SimConfig(gpu_count=16384)], relaxed=True)


def _no_events(results):
    for r in results:
        r.events = None
    return results


def test_c4_prefix_sharded_cluster_matches_reference(engine, monkeypatch):
    """Without the event log the 16384-GPU trace runs on a 16-CTA cluster
    (GPU-range shards exchanging packed keys over DSMEM): the reference's
    results on a prefix, and bit-identical to one CTA on a longer one."""
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 2048
    sp.job_count = 600
    b = rb.ref_generate_batch(sp, [0])
    cfg = [SimConfig(gpu_count=16384)]
    ref = _no_events(rb.ref_run_batch_results(b, cfg))
    got = engine.run_batch(b, cfg, abi.OUT_JOBS | abi.OUT_TIMELINE)
    bad = [d for r, g in zip(ref, got) if (d := diff_results_relaxed_timeline(r, g))]
    assert not bad, bad
    sp.job_count = 4000
    b = rb.ref_generate_batch(sp, [0])
    sharded = engine.run_batch(b, cfg, abi.OUT_JOBS | abi.OUT_TIMELINE)[0]
    monkeypatch.setenv("MSG_SHARDS", "1")
    one = engine.run_batch(b, cfg, abi.OUT_JOBS | abi.OUT_TIMELINE)[0]
    assert sharded.summary.tobytes() == one.summary.tobytes()
    assert sharded.per_job.tobytes() == one.per_job.tobytes()
    assert sharded.frag_timeline.tobytes() == one.frag_timeline.tobytes()


@pytest.mark.parametrize("shards,groups", [(4, 2), (2, 4), (8, 2)])
def test_device_groups_on_one_gpu(engine, monkeypatch, shards, groups):
    """The multi-GPU protocol (device groups exchanging stamped records
    through global-memory inboxes) with all groups as clusters of this GPU:
    the reference's results (timeline to 1e-9)."""
    monkeypatch.setenv("MSG_SHARDS", str(shards))
    monkeypatch.setenv("MSG_VDEV", str(groups))
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 256
    sp.job_count = 800
    churn = WorkloadSpec(mean_interarrival_s=0.4 / 256, median_s=4.0, sigma=1.2, job_count=800)
    for spec, cfg in ((sp, SimConfig(gpu_count=2048)),
                      (churn, SimConfig(gpu_count=2048, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                                        reconfig_latency_s=0.1))):
        b = rb.ref_generate_batch(spec, [3])
        ref = _no_events(rb.ref_run_batch_results(b, [cfg]))
        got = engine.run_batch(b, [cfg], abi.OUT_JOBS | abi.OUT_TIMELINE)
        bad = [d for r, g in zip(ref, got) if (d := diff_results_relaxed_timeline(r, g))]
        assert not bad, bad
