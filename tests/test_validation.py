"""Input validation follows Engine::Engine (sim.cpp:73-116): same error code
as the reference for every malformed trace / config.  Exercised through the
product's shared staging code (staging.h) via the test harness build."""
import pytest

from helpers import emu_run_batch_results
from oracle import refbind as rb
from paper_2512_16099_b200.model import FeatureFlags, Job, SchedulerConfig, SimConfig, TraceBatch

CASES = [
    ("unsorted", [Job(0, 10.0, 5, 1.0), Job(1, 5.0, 5, 1.0)], SimConfig(gpu_count=1), "TraceUnsorted"),
    ("profile", [Job(0, 0.0, 42, 1.0)], SimConfig(gpu_count=1), "UnknownProfile"),
    ("negative profile", [Job(0, 0.0, -1, 1.0)], SimConfig(gpu_count=1), "UnknownProfile"),
    ("service", [Job(0, 0.0, 5, 0.0)], SimConfig(gpu_count=1), "BadSpec"),
    ("dup", [Job(3, 0.0, 5, 1.0), Job(3, 1.0, 5, 1.0)], SimConfig(gpu_count=1), "BadSpec"),
    ("dup shuffled", [Job(9, 0.0, 5, 1.0), Job(3, 1.0, 5, 1.0), Job(9, 2.0, 5, 1.0)], SimConfig(gpu_count=1),
     "BadSpec"),
    ("first error wins", [Job(0, 1.0, 5, 1.0), Job(1, 0.5, 5, 0.0)], SimConfig(gpu_count=1), "TraceUnsorted"),
    ("arrival below -1", [Job(0, -2.0, 5, 1.0)], SimConfig(gpu_count=1), "TraceUnsorted"),
    ("gpus", [Job(0, 0.0, 5, 1.0)], SimConfig(gpu_count=0), "BadConfig"),
    ("threshold", [Job(0, 0.0, 5, 1.0)], SimConfig(sched=SchedulerConfig(threshold=1.2)), "BadThreshold"),
    ("threshold<0", [Job(0, 0.0, 5, 1.0)], SimConfig(sched=SchedulerConfig(threshold=-0.1)), "BadThreshold"),
    ("no layout", [Job(0, 0.0, 5, 1.0)], SimConfig(sched=SchedulerConfig(features=FeatureFlags(True, False, True))),
     "BadConfig"),
    ("layout size", [Job(0, 0.0, 5, 1.0)],
     SimConfig(gpu_count=2, sched=SchedulerConfig(features=FeatureFlags(True, False, True),
                                                  static_layout=[[(5, 0)]])), "BadConfig"),
    ("layout start", [Job(0, 0.0, 5, 1.0)],
     SimConfig(gpu_count=1, sched=SchedulerConfig(features=FeatureFlags(True, False, True),
                                                  static_layout=[[(1, 4)]])), "InvalidPlacement"),
    ("layout overlap", [Job(0, 0.0, 5, 1.0)],
     SimConfig(gpu_count=1, sched=SchedulerConfig(features=FeatureFlags(True, False, True),
                                                  static_layout=[[(1, 0), (5, 2)]])), "SlicesBusy"),
    ("pending", [Job(0, 0.0, 0, 10.0)],
     SimConfig(gpu_count=1, sched=SchedulerConfig(features=FeatureFlags(True, False, True),
                                                  static_layout=[[(2, 0), (2, 4)]])), "JobsPending"),
]


@pytest.mark.parametrize("name,trace,cfg,code", CASES, ids=[c[0] for c in CASES])
def test_error_codes(name, trace, cfg, code):
    b = TraceBatch.from_traces([trace])
    got = emu_run_batch_results(b, [cfg])[0]
    assert got.code == code, (got.code, got.message)
    if rb.ref_available():
        assert rb.ref_run_batch_results(b, [cfg])[0].code == code
    if rb.port_available():
        assert rb.port_run_batch_results(b, [cfg])[0].code == code


@pytest.mark.skipif(not rb.ref_available(), reason="reference library not built")
@pytest.mark.parametrize("name,trace,cfg,code", CASES, ids=[c[0] for c in CASES])
def test_error_text_is_reference_what(name, trace, cfg, code):
    """str(MigschedError) raised for a failed trace equals the reference's
    Error::what() ("Code: message", error.hpp:10-19) — the code appears once."""
    from paper_2512_16099_b200.model import MigschedError

    b = TraceBatch.from_traces([trace])
    got = emu_run_batch_results(b, [cfg])[0]
    ref = rb.ref_run_batch_results(b, [cfg])[0]
    with pytest.raises(MigschedError) as e:
        got.raise_for_status()
    assert e.value.code == code
    assert str(e.value) == ref.message
