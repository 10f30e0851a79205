"""The scheduler oracle suites (oracle.cpp:103-340), CPU
side: the brute-force multi-GPU oracle exported for the GPU suites
(ref_oracle_clusters: Lazy GPUs first, exact-fraction argmin, lower GPU /
start on ties) agrees with the reference's own schedule() on every 2-GPU
cluster at depth 2 and on sampled 3-GPU clusters — the same check the
reference's diff_multi_gpu_scheduler makes."""
import numpy as np
import pytest

from helpers import cluster_slots, states_to_slots
from oracle import refbind as rb
from paper_2512_16099_b200 import abi

pytestmark = pytest.mark.skipif(not rb.ref_available(), reason="reference library not built")


def _check(depth, clusters):
    states = rb.ref_enumerate_states(depth)
    slots = cluster_slots(states_to_slots(states), clusters)
    g, s = rb.ref_oracle_clusters(depth, clusters)
    for i in range(len(clusters)):
        for p in range(6):
            st, d = rb.ref_schedule(abi.OP_SCHEDULE, slots[i], p)
            assert st == 0
            want = (int(d["gpu"]), int(d["start"])) if d["placed"] else (-1, -1)
            assert (int(g[i, p]), int(s[i, p])) == want, (i, p)


def test_oracle_matches_reference_scheduler_on_all_pairs_depth2():
    n = len(rb.ref_enumerate_states(2))
    pairs = np.stack(np.meshgrid(np.arange(n), np.arange(n), indexing="ij"), -1).reshape(-1, 2)
    _check(2, pairs)


def test_oracle_matches_reference_scheduler_on_sampled_triples():
    rng = np.random.default_rng(2024)
    n = len(rb.ref_enumerate_states(3))
    _check(3, rng.integers(0, n, (300, 3)))
