"""The scheduler oracle suites on the GPU: the batched
schedule kernel against the brute-force exact-fraction oracle — every 2-GPU
cluster of depth-7 states (723^2 = 522,729 clusters x 6 profiles = 3.1M
decisions; the reference's suite runs depth <= 3 on the CPU) and 200,000
sampled 3-GPU clusters (the reference samples 1,500)."""
import numpy as np
import pytest

from helpers import cluster_slots, states_to_slots
from oracle import refbind as rb
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.model import SchedulerConfig

pytestmark = pytest.mark.gpu


def _suite(depth, clusters, chunk=200_000):
    from paper_2512_16099_b200 import decisions

    states = rb.ref_enumerate_states(depth)
    one = states_to_slots(states)
    g_ref, s_ref = rb.ref_oracle_clusters(depth, clusters)
    G = clusters.shape[1]
    bad = 0
    for c0 in range(0, len(clusters), chunk):
        part = clusters[c0:c0 + chunk]
        slots = cluster_slots(one, part)
        for p in range(6):
            d = decisions.schedule_batch(abi.OP_SCHEDULE, slots, np.full(len(part), p), SchedulerConfig(), G)
            got_g = np.where(d["placed"] != 0, d["gpu"], -1)
            got_s = np.where(d["placed"] != 0, d["start"], -1)
            bad += int(np.sum((got_g != g_ref[c0:c0 + len(part), p]) | (got_s != s_ref[c0:c0 + len(part), p])))
    return bad


def test_all_two_gpu_clusters_depth7():
    n = len(rb.ref_enumerate_states(7))
    assert n == 723
    pairs = np.stack(np.meshgrid(np.arange(n), np.arange(n), indexing="ij"), -1).reshape(-1, 2)
    assert _suite(7, pairs) == 0


def test_sampled_three_gpu_clusters_depth7():
    rng = np.random.default_rng(2024)
    assert _suite(7, rng.integers(0, 723, (200_000, 3))) == 0
