"""CPU-side check of the block engine for large clusters (cluster_core.cuh,
compiled for the host with the test-only block/warp emulation) against the
reference library: bit-exact (timeline exact up to 512 GPUs, 1e-9 relative
above)."""
import os

import pytest

from helpers import diff_results, diff_results_relaxed_timeline, emu_run_batch_results
from oracle import refbind as rb
from paper_2512_16099_b200.model import FeatureFlags, SchedulerConfig, SimConfig, WorkloadSpec, preset, static_layout_preset

pytestmark = pytest.mark.skipif(not rb.ref_available(), reason="reference library not built")


@pytest.fixture
def block_env(monkeypatch):
    def set_(force=False, threads=64, gpu_smem=True):
        monkeypatch.setenv("MSG_EMU_GPU_SMEM", "1" if gpu_smem else "0")
        if force:
            monkeypatch.setenv("MSG_EMU_FORCE_BLOCK", "1")
        else:
            monkeypatch.delenv("MSG_EMU_FORCE_BLOCK", raising=False)
        monkeypatch.setenv("MSG_EMU_BLOCK_THREADS", str(threads))
    return set_


def _check(spec, cfg, seeds, relaxed=False, no_events=False):
    b = rb.ref_generate_batch(spec, seeds)
    ref = rb.ref_run_batch_results(b, [cfg])
    got = emu_run_batch_results(b, [cfg])
    if no_events:  # the sharded engine writes no event log
        for r in got:
            r.events = None
    diff = diff_results_relaxed_timeline if relaxed else diff_results
    bad = [(s, d) for s, r, g in zip(seeds, ref, got) if (d := diff(r, g))]
    assert not bad, bad[:2]


@pytest.mark.parametrize("threads", [32, 64, 96])
def test_block_engine_on_small_clusters_matches(block_env, threads):
    block_env(force=True, threads=threads, gpu_smem=threads != 64)
    _check(preset("normal25"), SimConfig(gpu_count=8), [0, 1])
    c5 = WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, profile_mix=(0.5, 0.3, 0.2, 0.0))
    _check(c5, SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                         reconfig_latency_s=0.1), [2])
    for f in (FeatureFlags(False, False, False), FeatureFlags(True, False, False)):
        sp = preset("normal25")
        sp.mean_interarrival_s = 10.0
        _check(sp, SimConfig(gpu_count=4, sched=SchedulerConfig(features=f, static_layout=static_layout_preset("static-b"))),
               [3])


@pytest.mark.parametrize("gpu_smem", [True, False])
def test_block_engine_large_clusters(block_env, gpu_smem):
    block_env(force=False, threads=64, gpu_smem=gpu_smem)
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 12
    sp.job_count = 400
    _check(sp, SimConfig(gpu_count=96), [0])
    churn = WorkloadSpec(mean_interarrival_s=0.04, median_s=4.0, sigma=1.2, job_count=400)
    _check(churn, SimConfig(gpu_count=50, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                            reconfig_latency_s=0.1), [1])


def test_block_engine_relaxed_timeline_above_512_gpus(block_env):
    block_env(force=False, threads=64)
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 80
    sp.job_count = 600
    _check(sp, SimConfig(gpu_count=640), [4], relaxed=True)


@pytest.mark.parametrize("shards", [2, 3, 5])
def test_sharded_block_engine(block_env, monkeypatch, shards):
    """S CTAs of one thread-block cluster, each owning a GPU range and its
    active list, exchanging packed keys per decision: identical results to
    the reference (timeline to 1e-9 above 512 GPUs)."""
    block_env(force=False, threads=32, gpu_smem=shards != 3)
    monkeypatch.setenv("MSG_EMU_SHARDS", str(shards))
    monkeypatch.setenv("MSG_EMU_SLOT_SMEM", "0" if shards == 2 else "1")  # slots in global / shared memory
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 80
    sp.job_count = 500
    _check(sp, SimConfig(gpu_count=640), [4], relaxed=True, no_events=True)
    churn = WorkloadSpec(mean_interarrival_s=0.005, median_s=4.0, sigma=1.2, job_count=500)
    _check(churn, SimConfig(gpu_count=520, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                            reconfig_latency_s=0.1), [1], relaxed=True, no_events=True)
    sp2 = preset("long25")
    sp2.mean_interarrival_s = 25.0 / 100
    sp2.job_count = 400
    _check(sp2, SimConfig(gpu_count=700, sched=SchedulerConfig(features=FeatureFlags(True, True, False))), [7],
           relaxed=True, no_events=True)


@pytest.mark.parametrize("groups,shards", [(2, 1), (2, 2), (3, 2), (4, 1)])
def test_device_groups(block_env, monkeypatch, groups, shards):
    """The trace split over device groups (one cluster each; GPUs of a box):
    two-level exchange — DSMEM inside a group, stamped peer-memory inboxes
    across groups; each group keeps its own queue, job rows go to group 0."""
    block_env(force=False, threads=32, gpu_smem=True)
    monkeypatch.setenv("MSG_EMU_SHARDS", str(shards))
    monkeypatch.setenv("MSG_EMU_GROUPS", str(groups))
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 80
    sp.job_count = 400
    _check(sp, SimConfig(gpu_count=640), [5], relaxed=True, no_events=True)
    churn = WorkloadSpec(mean_interarrival_s=0.005, median_s=4.0, sigma=1.2, job_count=400)
    _check(churn, SimConfig(gpu_count=520, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                            reconfig_latency_s=0.1), [2], relaxed=True, no_events=True)
