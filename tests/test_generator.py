"""Host trace generation (msg_generate) reproduces the reference generator
(workload.cpp:98-147) bit for bit."""
import numpy as np
import pytest

from helpers import golden_runs
from oracle import refbind as rb
from paper_2512_16099_b200.engine import generate, generate_batch
from paper_2512_16099_b200.model import EXPONENTIAL, FIXED, WorkloadSpec, preset, preset_names


@pytest.mark.parametrize("name", ["c1_g8_s0", "long25_g4_s7", "c5_s1", "ties_g3"])
def test_generator_matches_golden_traces(name):
    batch, _, _, meta = golden_runs()[name]
    spec = WorkloadSpec(**meta["spec"])
    spec.profile_mix = tuple(spec.profile_mix)
    spec.seed = meta["seed"]
    jobs = generate(spec)
    assert np.array([j.arrival_s for j in jobs]).tobytes() == batch.arrival_s.tobytes()
    assert np.array([j.service_s for j in jobs]).tobytes() == batch.service_s.tobytes()
    assert [j.profile for j in jobs] == list(batch.profile)
    assert [j.id for j in jobs] == list(batch.job_id)


def test_generate_batch_matches_single_generation():
    b = generate_batch(preset("long50"), 100, 9, threads=4)
    for t in range(9):
        sp = preset("long50")
        sp.seed = 100 + t
        jobs = generate(sp)
        assert np.array([j.service_s for j in jobs]).tobytes() == b.service_s[t * 200:(t + 1) * 200].tobytes()


@pytest.mark.skipif(not rb.ref_available(), reason="reference library not built")
def test_generator_vs_reference_many_specs():
    specs = [preset(n) for n in preset_names()] + [
        WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, profile_mix=(0.5, 0.3, 0.2, 0.0)),
        WorkloadSpec(family=EXPONENTIAL, query_type=1, job_count=300),
        WorkloadSpec(family=FIXED, value_s=3.0, job_count=50),
    ]
    for sp in specs:
        for seed in (0, 1, 12345, 2**40 + 7):
            sp.seed = seed
            ids, arr, prof, svc = rb.ref_generate(sp)
            jobs = generate(sp)
            assert np.array([j.arrival_s for j in jobs]).tobytes() == arr.tobytes()
            assert np.array([j.service_s for j in jobs]).tobytes() == svc.tobytes()
            assert np.array([j.profile for j in jobs], np.int32).tobytes() == prof.tobytes()


def test_generator_rejects_bad_specs():
    from paper_2512_16099_b200.model import MigschedError

    for bad in (WorkloadSpec(mean_interarrival_s=0.0), WorkloadSpec(profile_mix=(0.5, 0.5, 0.5, 0.0)),
                WorkloadSpec(sigma=0.0), WorkloadSpec(job_count=-1)):
        with pytest.raises(MigschedError) as e:
            generate(bad)
        assert e.value.code == "BadSpec"
