"""CPU-side check of the DEVICE code's logic: engine_core.cuh compiled for
the host with a 32-thread warp emulation (tests/emu, test-only) must
reproduce the reference bit for bit.  This runs on the build box without a
GPU; tests/test_gpu_parity.py repeats the comparison on the B200 itself."""
import numpy as np
import pytest

from helpers import diff_results, emu_run_batch_results, golden_runs
from oracle import refbind as rb
from paper_2512_16099_b200.model import (
    EXPONENTIAL,
    FeatureFlags,
    SchedulerConfig,
    SimConfig,
    TraceBatch,
    WorkloadSpec,
    static_layout_preset,
)


@pytest.mark.parametrize("name", sorted(golden_runs().keys()))
def test_emulated_kernel_matches_golden(name):
    batch, cfg, ref, _ = golden_runs()[name]
    got = emu_run_batch_results(batch, [cfg])[0]
    assert diff_results(ref, got) == ""


@pytest.mark.skipif(not rb.port_available(), reason="oracle port not built")
def test_emulated_kernel_vs_port_randomized():
    from paper_2512_16099_b200.engine import generate

    rng = np.random.default_rng(11)
    for _ in range(10):
        G = int(rng.choice([1, 2, 4, 5, 8, 12]))
        dyn = bool(rng.integers(0, 2)) or G != 4
        feats = FeatureFlags(bool(rng.integers(0, 2)), dyn, bool(rng.integers(0, 2)))
        sp = WorkloadSpec(mean_interarrival_s=float(rng.choice([1.0, 5.0, 20.0])), job_count=60,
                          family=int(rng.choice([0, EXPONENTIAL])), seed=int(rng.integers(0, 1 << 30)))
        cfg = SimConfig(gpu_count=G, sched=SchedulerConfig(
            threshold=float(rng.choice([0.0, 0.3, 0.5, 1.0])), features=feats,
            static_layout=None if dyn else static_layout_preset("static-c")),
            migration_overlap_s=float(rng.choice([0.0, 2.0])), reconfig_latency_s=float(rng.choice([0.0, 0.3])))
        b = TraceBatch.from_traces([generate(sp)])
        want = rb.port_run_batch_results(b, [cfg])[0]
        got = emu_run_batch_results(b, [cfg])[0]
        assert diff_results(want, got) == "", (G, feats, cfg)


@pytest.mark.parametrize("name", sorted(golden_runs().keys()))
def test_emulated_io_kernel_matches_golden(name, monkeypatch):
    """The pipelined msg_run_batch's IO instantiation of the event loop
    (zero-copy input blocks read from the caller's arrays, job records
    published progressively into SoA host columns, completion flag) in the
    warp emulation: the same summary and job rows as the reference, and the
    host columns equal to the device records (checked inside the harness)."""
    batch, cfg, ref, _ = golden_runs()[name]
    if cfg.gpu_count > 32:
        pytest.skip("the IO kernel is the warp engine's (G <= 32)")
    monkeypatch.setenv("MSG_EMU_IO", "1")
    got = emu_run_batch_results(batch, [cfg])[0]
    ref.events = ref.frag_timeline = None  # summary + rows only in the IO kernel
    got.events = got.frag_timeline = None
    assert diff_results(ref, got) == ""


@pytest.mark.skipif(not rb.port_available(), reason="oracle port not built")
def test_emulated_io_kernel_long_traces(monkeypatch):
    """Traces long enough for several zero-copy blocks and row flushes."""
    from paper_2512_16099_b200.engine import generate

    monkeypatch.setenv("MSG_EMU_IO", "1")
    for n, G, seed in ((7, 8, 1), (33, 4, 2), (150, 8, 3), (400, 16, 4)):
        sp = WorkloadSpec(mean_interarrival_s=3.0, job_count=n, seed=seed)
        cfg = SimConfig(gpu_count=G, migration_overlap_s=1.0)
        b = TraceBatch.from_traces([generate(sp)])
        want = rb.port_run_batch_results(b, [cfg])[0]
        got = emu_run_batch_results(b, [cfg])[0]
        want.events = want.frag_timeline = None
        got.events = got.frag_timeline = None
        assert diff_results(want, got) == "", (n, G)


@pytest.mark.parametrize("name", sorted(golden_runs().keys()))
def test_emulated_no_delay_kernel_matches_golden(name, monkeypatch):
    """The no-delay instantiation (chosen when every config has reconfig
    latency +0 and no migration overlap: no slot is ever WaitingStart or
    Draining) reproduces the golden runs it applies to, event log included;
    the others run the general kernel."""
    batch, cfg, ref, _ = golden_runs()[name]
    monkeypatch.setenv("MSG_EMU_ND", "1")
    got = emu_run_batch_results(batch, [cfg])[0]
    assert diff_results(ref, got) == ""


@pytest.mark.skipif(not rb.port_available(), reason="oracle port not built")
def test_emulated_no_delay_kernel_vs_port(monkeypatch):
    from paper_2512_16099_b200.engine import generate

    monkeypatch.setenv("MSG_EMU_ND", "1")
    rng = np.random.default_rng(5)
    for _ in range(8):
        G = int(rng.choice([2, 4, 8, 16]))
        feats = FeatureFlags(bool(rng.integers(0, 2)), True, bool(rng.integers(0, 2)))
        sp = WorkloadSpec(mean_interarrival_s=float(rng.choice([0.5, 2.0, 10.0])), job_count=80,
                          seed=int(rng.integers(0, 1 << 30)))
        cfg = SimConfig(gpu_count=G, sched=SchedulerConfig(threshold=float(rng.choice([0.0, 0.4, 1.0])),
                                                           features=feats))
        b = TraceBatch.from_traces([generate(sp)])
        want = rb.port_run_batch_results(b, [cfg])[0]
        got = emu_run_batch_results(b, [cfg])[0]
        assert diff_results(want, got) == "", (G, feats)
