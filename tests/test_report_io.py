"""Report emission: msg_format_text writes the reference
CLI's files — events.jsonl, report.json, report.csv, fragcost_timeline.csv —
byte for byte, checked against the unmodified reference serializers
(reports.cpp:14-116) on the reference's own results (CPU; the GPU drop-in
test applies the same formatter to engine results)."""
import pytest

from oracle import refbind as rb
from paper_2512_16099_b200.model import (FeatureFlags, SchedulerConfig, SimConfig, WorkloadSpec, preset,
                                         static_layout_preset)

pytestmark = pytest.mark.skipif(not rb.ref_available(), reason="reference library not built")

KINDS = ("events.jsonl", "report.json", "report.csv", "fragcost_timeline.csv")

CASES = [
    (preset("normal25"), SimConfig(gpu_count=8), [0, 1]),
    (preset("long50"), SimConfig(gpu_count=4, sched=SchedulerConfig(threshold=0.6)), [3]),
    (WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, profile_mix=(0.5, 0.3, 0.2, 0.0), job_count=300),
     SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5, reconfig_latency_s=0.1,
               seed=42), [2]),
    (preset("normal50"), SimConfig(gpu_count=4, sched=SchedulerConfig(features=FeatureFlags(True, False, False),
                                                                       static_layout=static_layout_preset("static-b"))),
     [5]),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_texts_match_reference_serializers(case):
    spec, cfg, seeds = CASES[case]
    b = rb.ref_generate_batch(spec, seeds)
    for r in rb.ref_run_batch_results(b, [cfg], texts=True):
        assert r.status == 0
        for kind, want in zip(KINDS, r.texts):
            got = r.text(kind, cfg)
            assert got == want, (kind, next(i for i, (x, y) in enumerate(zip(got, want)) if x != y))


def test_empty_trace_texts():
    from paper_2512_16099_b200.model import TraceBatch

    b = TraceBatch.from_traces([[]])
    cfg = SimConfig(gpu_count=2)
    r = rb.ref_run_batch_results(b, [cfg], texts=True)[0]
    for kind, want in zip(KINDS, r.texts):
        assert r.text(kind, cfg) == want
