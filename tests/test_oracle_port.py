"""The oracle's C restatement (oracle/oracle_port.c) pinned against the
reference: golden runs produced by the unmodified reference library, the
reference test suite's known-answer values, and (when the reference library
is present) randomized differential runs."""
import numpy as np
import pytest

from helpers import diff_results, golden_runs
from oracle import refbind as rb
from paper_2512_16099_b200.model import (
    FeatureFlags,
    SchedulerConfig,
    SimConfig,
    TraceBatch,
    WorkloadSpec,
    preset,
    static_layout_preset,
)

pytestmark = pytest.mark.skipif(not rb.port_available(), reason="oracle port not built")


@pytest.mark.parametrize("name", sorted(golden_runs().keys()))
def test_port_matches_golden_reference_runs(name):
    batch, cfg, ref, _ = golden_runs()[name]
    got = rb.port_run_batch_results(batch, [cfg])[0]
    assert diff_results(ref, got) == ""


def k(bc, bm, kc=None, km=None):
    kc = bc if kc is None else kc
    km = bm if km is None else km
    return rb.port_lib().port_frag_k(bc, bm, kc, km)


def test_frag_cost_known_answers():
    # test_frag_metric.cpp:43-67, acceptance.cpp:61-76 (values x 25200)
    assert k(0, 0) == 0                       # empty GPU
    assert k(0x07, 0x0F) == round(0.35 * 25200)  # busy 3g@0 -> 0.35
    assert k(0x0C, 0x0C) == round(0.2 * 25200)   # busy 2g@2 -> 0.2
    assert k(0x30, 0x30) == 0                 # 2g@4 keeps every profile creatable
    assert k(0x7F, 0xFF) == 0                 # 4g@0 + 3g@4: full, not fragmented
    # idle instances never count: busy 2g@2 with idle 2g@4 and 1g@0 = 0.2
    assert k(0x0C, 0x0C, 0x0C, 0x0C) == round(0.2 * 25200)


def _acceptance_trace(name, seed):
    from paper_2512_16099_b200.engine import generate

    sp = preset(name)
    sp.job_count = 200
    sp.seed = seed
    return generate(sp)


def test_acceptance_criterion_6_goldens():
    """acceptance.cpp:150-155 mean-turnaround goldens (4 GPUs)."""
    goldens = {
        ("normal25", 1001): (992.734900172, 965.670431208, 313.438170646, 258.640679930),
        ("long25", 1002): (2091.812659312, 2077.661989828, 1109.716298357, 1059.817040414),
        ("normal50", 1003): (205.498577738, 202.196551418, 169.038014042, 166.612534759),
        ("long50", 1004): (1007.366664150, 960.220466415, 351.748120417, 344.619718160),
    }
    flags = [FeatureFlags(False, False, False), FeatureFlags(True, False, False),
             FeatureFlags(True, True, False), FeatureFlags(True, True, True)]
    for (name, seed), want in goldens.items():
        tr = _acceptance_trace(name, seed)
        for f, w in zip(flags, want):
            cfg = SimConfig(gpu_count=4, sched=SchedulerConfig(
                features=f, static_layout=None if f.dynamic_partitioning else static_layout_preset("static-a")))
            got = rb.port_run_batch_results(TraceBatch.from_traces([tr]), [cfg])[0]
            assert abs(got.mean_turnaround_s - w) <= 1e-9 * w, (name, f, got.mean_turnaround_s, w)


@pytest.mark.skipif(not rb.ref_available(), reason="reference library not built")
def test_port_vs_reference_randomized():
    rng = np.random.default_rng(5)
    for _ in range(12):
        G = int(rng.integers(1, 9))
        sp = WorkloadSpec(mean_interarrival_s=float(rng.choice([2.0, 10.0, 25.0])), job_count=80,
                          family=int(rng.integers(0, 3)))
        cfg = SimConfig(gpu_count=G, sched=SchedulerConfig(threshold=float(rng.choice([0.0, 0.3, 0.4, 0.7, 1.0]))),
                        migration_overlap_s=float(rng.choice([0.0, 1.5])),
                        reconfig_latency_s=float(rng.choice([0.0, 0.2])),
                        contention_alpha=float(rng.choice([0.0, 0.15, 0.5])))
        b = rb.ref_generate_batch(sp, [int(rng.integers(0, 1 << 30))])
        ref = rb.ref_run_batch_results(b, [cfg])[0]
        got = rb.port_run_batch_results(b, [cfg])[0]
        assert diff_results(ref, got) == "", (G, sp, cfg)
