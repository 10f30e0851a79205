"""Decision-level kernels (decide.cu, score.cu) against the reference's own
known answers (test_scheduler.cpp, test_migration.cpp, acceptance.cpp) and
differentially against the unmodified reference library."""
import numpy as np
import pytest

from helpers import normalize_slots, random_cluster, states_to_slots
from oracle import refbind as rb
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.model import (
    P1G5GB,
    P1G10GB,
    P2G10GB,
    P3G20GB,
    P4G20GB,
    P7G40GB,
    FeatureFlags,
    MigschedError,
    SchedulerConfig,
)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def d():
    from paper_2512_16099_b200 import decisions

    return decisions


# ---- known answers from the reference test suite --------------------------
def test_schedule_known_answers(d):
    cfg = SchedulerConfig()
    c = d.Cluster(2).add_busy(0, P3G20GB, 0, 1)  # test_scheduler.cpp:22-32
    r = d.schedule(P2G10GB, c, cfg)
    assert (r.placed, r.gpu, r.start, r.reused) == (True, 1, 4, False)
    r = d.schedule(P2G10GB, d.Cluster(1), cfg)  # :34-40, acceptance criterion 3
    assert (r.gpu, r.start) == (0, 4)
    c = d.Cluster(2).add_idle(1, P2G10GB, 4)  # reuse beats lower GPU id :42-54
    r = d.schedule(P2G10GB, c, cfg)
    assert (r.gpu, r.start, r.reused) == (1, 4, True)
    c = d.Cluster(3)
    for g in range(3):
        c.add_busy(g, P1G5GB, 6, g + 10)
    assert d.schedule(P7G40GB, c, cfg).queued  # :56-63
    c = d.Cluster(2).add_busy(0, P4G20GB, 0, 1).add_busy(1, P1G5GB, 0, 2)
    assert d.schedule(P4G20GB, c, cfg).queued  # :65-82
    c = d.Cluster(2).add_busy(0, P3G20GB, 0, 1)
    assert d.schedule(P1G5GB, c, cfg).gpu == 1
    with pytest.raises(MigschedError) as e:
        d.schedule(17, d.Cluster(1), cfg)
    assert e.value.code == "UnknownProfile"
    r = d.first_fit_schedule(P2G10GB, d.Cluster(2), cfg)  # :115-129
    assert (r.gpu, r.start, r.evaluated_candidates) == (0, 0, 0)
    r = d.first_fit_schedule(P1G5GB, d.Cluster(2).add_busy(0, P7G40GB, 0, 1), cfg)
    assert (r.gpu, r.start) == (1, 0)
    # static exact-match only (:131-149)
    nd = SchedulerConfig(features=FeatureFlags(True, False, True))
    c = d.Cluster(1).add_idle(0, P1G10GB, 0).add_idle(0, P1G10GB, 2).add_idle(0, P3G20GB, 4)
    assert d.first_fit_schedule(P2G10GB, c, nd).queued and d.schedule(P2G10GB, c, nd).queued
    r = d.first_fit_schedule(P3G20GB, c, nd)
    assert (r.start, r.reused) == (4, True)


def test_try_dequeue_strict_fcfs(d):
    cfg = SchedulerConfig()
    c = d.Cluster(1).add_busy(0, P4G20GB, 0, 50)  # test_scheduler.cpp:151-176
    q = [(1, P4G20GB), (2, P1G5GB)]
    assert d.try_dequeue(q, c, cfg) == [] and len(q) == 2
    c = d.Cluster(1)
    q = [(1, P1G5GB)]
    placed = d.try_dequeue(q, c, cfg)
    assert len(placed) == 1 and q == [] and c.find_job(1) is not None


def test_plan_intra_known_answers(d):
    c = d.Cluster(1).add_busy(0, P2G10GB, 2, 1)  # test_migration.cpp:28-39, acceptance criterion 4
    p = d.plan_intra(c, 0, 0.0)
    assert len(p.moves) == 1 and p.moves[0].job == 1 and p.moves[0].to_start == 4
    assert p.moves[0].from_cost_before == 0.2 and p.moves[0].from_cost_after == 0.0
    assert c.find_job(1)[:2] == (0, 4)
    c = d.Cluster(1).add_busy(0, P3G20GB, 0, 1)  # :41-56
    p = d.plan_intra(c, 0, 0.0)
    assert [m.to_start for m in p.moves] == [4] and p.moves[0].from_cost_before == 0.35
    assert d.plan_intra(c, 0, 0.0).moves == []
    assert d.plan_intra(d.Cluster(1), 0, 0.0).moves == []  # :58-61


def test_plan_intra_greedy_vs_two_move_optimum_is_76(d):
    """test_migration.cpp:77-135: frozen count of states where greedy stops
    short of the best <=2-move sequence, over enumerate_states(3)."""
    states = rb.ref_enumerate_states(3)
    slots = states_to_slots(states)
    sums, moves = d.plan_batch(abi.PLAN_INTRA, slots, [0] * len(states), gpu_count=1)
    port = rb.port_lib()
    from paper_2512_16099_b200.model import COMPUTE_SLICES, MEMORY_SLICES, START_INDEXES

    def cost(units):
        bc = bm = 0
        for p, s in units:
            bc |= ((1 << COMPUTE_SLICES[p]) - 1) << s
            bm |= ((1 << MEMORY_SLICES[p]) - 1) << s
        return port.port_frag_k(bc, bm, bc, bm)

    def moves_of(units):
        out = []
        for i, (p, s0) in enumerate(units):
            for s in START_INDEXES[p]:
                if s == s0:
                    continue
                rest = units[:i] + units[i + 1:]
                if any(s < t + MEMORY_SLICES[q] and t < s + MEMORY_SLICES[p] for q, t in rest):
                    continue
                out.append(rest + [(p, s)])
        return out

    disc = 0
    for i, st in enumerate(states):
        reached = [(int(x["profile"]), s) for s, x in enumerate(slots[i]) if x["state"] == abi.SLOT_BUSY]
        best = cost(st)
        for one in moves_of(st):
            best = min(best, cost(one))
            for two in moves_of(one):
                best = min(best, cost(two))
        if cost(reached) > best:
            disc += 1
    assert disc == 76


def test_plan_inter_known_answers(d):
    c = d.Cluster(2).add_busy(0, P3G20GB, 0, 1).add_busy(0, P1G5GB, 4, 2)  # test_migration.cpp:137-151
    p = d.plan_inter(c, 1, 0.4, 0.0)
    assert len(p.moves) == 1
    m = p.moves[0]
    assert (m.job, m.from_gpu, m.to_gpu, m.to_start, m.to_cost_after) == (2, 0, 1, 6, 0.0)
    assert d.plan_inter(d.Cluster(2).add_busy(0, P1G5GB, 0, 1), 1).moves == []  # :153-158
    assert d.plan_inter(d.Cluster(2).add_busy(0, P4G20GB, 0, 1), 1).moves == []  # :160-166
    with pytest.raises(MigschedError) as e:  # :168-173
        d.plan_inter(d.Cluster(2).add_busy(1, P4G20GB, 0, 1), 1)
    assert e.value.code == "NotLazy"


def test_plan_inter_never_rechecks_lazy(d):
    """SURVEY §7 hard part 5 known-answer case: 4 moves, the 4th onto a GPU
    that is already Busy; evals/iter 21, 19, 17, 10, 0."""
    c = d.Cluster(3)
    for s in range(7):
        c.add_busy(0, P1G5GB, s, 2 * s + 1)
        c.add_busy(2, P1G5GB, s, 2 * s + 2)
    p = d.plan_inter(c, 1, 0.4, 0.0)
    got = [(m.job, m.from_gpu, m.from_start, m.to_start) for m in p.moves]
    assert got == [(13, 0, 6, 6), (14, 2, 6, 4), (1, 0, 0, 5), (2, 2, 0, 0)]
    assert p.max_evals == 21 and p.n_iterations == 5
    assert [round(c.utilization(g) * 7) for g in range(3)] == [5, 4, 5]


def test_on_departure_dispatch(d):
    c = d.Cluster(2).add_busy(0, P3G20GB, 4, 1).add_busy(0, P1G5GB, 0, 2)  # test_migration.cpp:221-251
    assert d.on_departure(c, 0).kind == "intra"
    c = d.Cluster(2).add_busy(0, P2G10GB, 0, 1).add_busy(1, P4G20GB, 0, 2).add_busy(1, P1G5GB, 4, 3)
    p = d.on_departure(c, 0)
    assert p.kind == "inter" and [m.job for m in p.moves] == [3]
    assert d.on_departure(d.Cluster(1).add_busy(0, P3G20GB, 0, 1), 0, enabled=False).empty()
    with pytest.raises(MigschedError) as e:
        d.on_departure(d.Cluster(1), 5)
    assert e.value.code == "UnknownGpu"


def test_overlap_keeps_source_draining(d):
    c = d.Cluster(1).add_busy(0, P2G10GB, 2, 1)  # test_migration.cpp:253-272 via a planned move
    d.plan_intra(c, 0, 5.0)
    inst = c.instances(0)
    assert (P2G10GB, 2, abi.SLOT_DRAINING, -1) in inst and (P2G10GB, 4, abi.SLOT_BUSY, 1) in inst


# ---- differential against the reference library ----------------------------
def _ref_sched_all(op, snaps, profs, **kw):
    out = []
    for s, p in zip(snaps, profs):
        st, dec = rb.ref_schedule(op, s, int(p), **kw)
        assert st == 0
        out.append(dec)
    return np.array(out, abi.DECISION_DTYPE)


def test_schedule_exhaustive_single_gpu_depth7(d):
    states = rb.ref_enumerate_states(7)
    assert len(states) == 723
    slots = np.repeat(states_to_slots(states), 6, axis=0)
    profs = np.tile(np.arange(6), len(states))
    for op in (abi.OP_SCHEDULE, abi.OP_FIRST_FIT):
        got = d.schedule_batch(op, slots, profs, SchedulerConfig(), 1)
        want = _ref_sched_all(op, slots, profs)
        assert got.tobytes() == want.tobytes()


def test_schedule_exhaustive_two_gpus_depth2(d):
    one = states_to_slots(rb.ref_enumerate_states(2))
    pairs = np.concatenate([np.concatenate([a, b])[None] for a in one for b in one])
    pairs["job"] = np.where(pairs["state"] == abi.SLOT_BUSY, np.arange(16)[None, :] + 1, -1)
    slots = np.repeat(pairs, 6, axis=0)
    profs = np.tile(np.arange(6), len(pairs))
    got = d.schedule_batch(abi.OP_SCHEDULE, slots, profs, SchedulerConfig(), 2)
    want = _ref_sched_all(abi.OP_SCHEDULE, slots, profs)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("G", [1, 3, 8, 32, 33, 200, 1024, 2048, 4099])
def test_schedule_random_clusters(d, G):
    """G > 32 goes through the HBM scorer (score.cu): 1024/2048 are whole
    chunks, 4099 adds a ragged, odd-length tail (scalar loads)."""
    rng = np.random.default_rng(G)
    n = 150 if G <= 200 else 24
    snaps = np.stack([random_cluster(rng, G) for _ in range(n)])
    profs = rng.integers(0, 6, n)
    for op in (abi.OP_SCHEDULE, abi.OP_FIRST_FIT, abi.OP_DISPATCH):
        for thr, lb, dyn in ((0.4, True, True), (0.0, True, False), (1.0, False, True), (0.6, True, True)):
            cfg = SchedulerConfig(threshold=thr, features=FeatureFlags(lb, dyn, True))
            got = d.schedule_batch(op, snaps, profs, cfg, G)
            want = _ref_sched_all(op, snaps, profs, threshold=thr, lb=lb, dyn=dyn)
            assert got.tobytes() == want.tobytes(), (op, thr, lb, dyn)


@pytest.mark.parametrize("G", [9000, 16384, 16386])
def test_schedule_multi_item_snapshots(d, G):
    """Snapshots around one scorer item (4 chunks of 4096 GPUs): 9000 GPUs =
    one item with a ragged last chunk, 16384 = exactly one item (finished
    in the scoring grid, no merge kernel), 16386 = 2 items with a 2-GPU
    tail (merge kernel).  Configs alternate so consecutive launches
    exercise both pass-2 list counters, and the register path (an odd
    count, G + 1) runs between them."""
    rng = np.random.default_rng(G)
    n = 6
    snaps = np.stack([random_cluster(rng, G) for _ in range(n)])
    profs = rng.integers(0, 6, n)
    odd = np.stack([random_cluster(rng, G + 1) for _ in range(2)])
    for rep in range(2):
        for thr, lb, dyn in ((0.4, True, True), (0.0, True, False), (1.0, False, True), (0.0, True, True),
                             (0.6, True, True)):
            cfg = SchedulerConfig(threshold=thr, features=FeatureFlags(lb, dyn, True))
            got = d.schedule_batch(abi.OP_SCHEDULE, snaps, profs, cfg, G)
            want = _ref_sched_all(abi.OP_SCHEDULE, snaps, profs, threshold=thr, lb=lb, dyn=dyn)
            assert got.tobytes() == want.tobytes(), (rep, thr, lb, dyn)
            if rep == 1 and thr == 0.0:
                got = d.schedule_batch(abi.OP_SCHEDULE, odd, profs[:2], cfg, G + 1)
                want = _ref_sched_all(abi.OP_SCHEDULE, odd, profs[:2], threshold=thr, lb=lb, dyn=dyn)
                assert got.tobytes() == want.tobytes(), ("odd", thr, lb, dyn)


@pytest.mark.parametrize("G", [2, 3, 8, 17])
def test_planners_random_clusters(d, G):
    rng = np.random.default_rng(100 + G)
    n = 120
    snaps = np.stack([random_cluster(rng, G, fill=5) for _ in range(n)])
    gpus = rng.integers(0, G, n)
    for op in (abi.PLAN_ON_DEPARTURE, abi.PLAN_INTRA, abi.PLAN_INTER):
        for thr, ov in ((0.4, 0.0), (0.3, 2.0), (0.7, 0.0)):
            mine = snaps.copy()
            sums, moves = d.plan_batch(op, mine, gpus, thr, True, ov, G)
            for i in range(n):
                st, s, mv, after = rb.ref_plan(op, snaps[i], int(gpus[i]), thr, True, ov)
                assert sums[i]["status"] == st, (op, i)
                if st:
                    continue
                assert (sums[i]["kind"], sums[i]["n_moves"], sums[i]["n_iterations"], sums[i]["max_evals"]) == (
                    s["kind"], s["n_moves"], s["n_iterations"], s["max_evals"]), (op, thr, ov, i)
                assert moves[i][: len(mv)].tobytes() == mv.tobytes(), (op, thr, ov, i)
                assert normalize_slots(mine[i]) == normalize_slots(after), (op, thr, ov, i)


def test_try_dequeue_random(d):
    rng = np.random.default_rng(7)
    for _ in range(150):
        G = int(rng.integers(1, 6))
        snap = random_cluster(rng, G, fill=3, job0=1)
        q = [(1000 + k, int(rng.integers(0, 6))) for k in range(int(rng.integers(0, 6)))]
        thr, lb, dyn = float(rng.choice([0.3, 0.4, 0.8])), bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
        cfg = SchedulerConfig(threshold=thr, features=FeatureFlags(lb, dyn, True))
        c = d.Cluster(G)
        c.slots = snap.copy()
        mine_q = list(q)
        placed = d.try_dequeue(mine_q, c, cfg)
        st, ref_placed, ref_slots = rb.ref_try_dequeue(snap, q, thr, lb, dyn)
        assert st == 0
        assert placed == ref_placed
        assert normalize_slots(c.slots) == normalize_slots(ref_slots)


def test_frag_cost_known_answers_and_random_gpus(d):
    """frag_cost on the device (msg_frag_cost_batch) — the reference's
    known answers (test_frag_metric.cpp:43-93) and random GPUs with busy,
    idle and draining instances against frag_cost_masks."""
    from paper_2512_16099_b200.model import COMPUTE_SLICES, MEMORY_SLICES

    c = d.Cluster(1)
    assert d.frag_cost(c, 0) == 0.0                       # empty
    c.add_busy(0, 2, 0, 1)
    assert d.frag_cost(c, 0) == 0.35                      # 3g@0
    c = d.Cluster(1)
    c.add_busy(0, 3, 2, 1)
    c.add_idle(0, 3, 4)
    c.add_idle(0, 5, 0)
    assert d.frag_cost(c, 0) == 0.2                       # 2g@2 (+ idle instances: no effect)
    rng = np.random.default_rng(11)
    snaps = np.stack([random_cluster(rng, 1, fill=6) for _ in range(3000)])
    num, cost = d.frag_cost_batch(snaps)
    for i, s8 in enumerate(snaps):
        bc = bm = kc = km = 0
        for st in range(8):
            x = s8[st]
            if x["profile"] < 0 or x["state"] == abi.SLOT_IDLE or x["state"] == abi.SLOT_EMPTY:
                continue
            mc = ((1 << COMPUTE_SLICES[x["profile"]]) - 1) << st
            mm = ((1 << MEMORY_SLICES[x["profile"]]) - 1) << st
            kc |= mc
            km |= mm
            if x["state"] == abi.SLOT_BUSY:
                bc |= mc
                bm |= mm
        n_, den = rb.ref_frag_cost(bc, bm, kc, km)
        assert cost[i] == n_ / den and num[i] * den == n_ * 25200, i


def test_scorer_full_size_tma_vs_register_path(d):
    """bench.py's scorer sweep size (4096 snapshots x 16384 GPUs, 512 MiB),
    with idle-exact bits and a few draining words: the TMA kernel (key-only
    keys, merged in the grid) and the independent register-streaming kernel
    (odd G: the same snapshots less their last word, which is a full GPU
    with no candidate) agree bit for bit at every threshold.  Both are
    checked against the reference library at smaller sizes above."""
    import ctypes as C

    import torch

    L = d._bind()
    from paper_2512_16099_b200.engine import default_engine

    eng = default_engine(0)
    B, G = 4096, 16384
    gen = torch.Generator(device="cuda").manual_seed(7)
    rnd = torch.randint(0, 1 << 62, (B, G), device="cuda", dtype=torch.int64, generator=gen)
    bm = rnd & 0x7F
    idle = ((rnd >> 8) & 0x3FFFF) * (((rnd >> 30) & 3) == 0)
    drain = ((rnd >> 40) & 0x7F) * (((rnd >> 50) & 4095) == 0)
    words = bm | (bm << 8) | ((bm | drain) << 16) | (idle << 24)
    del rnd, bm, idle, drain
    words[:, G - 1] = 0xFFFF7F  # a full GPU: no candidate
    words = words.contiguous()
    odd = words[:, : G - 1].contiguous()
    prof = torch.randint(0, 6, (B,), device="cuda", dtype=torch.uint8, generator=gen)
    out_a = torch.empty(B * 2, device="cuda", dtype=torch.int64)
    out_b = torch.empty(B * 2, device="cuda", dtype=torch.int64)
    torch.cuda.synchronize()  # the engine launches on its own stream
    for thr in (0.4, 0.0, 1.0):
        cfg = d._sched_cfg(SchedulerConfig(threshold=thr))
        assert L.msg_score_device(eng._h, B, G, words.data_ptr(), prof.data_ptr(), C.byref(cfg),
                                  out_a.data_ptr()) == 0
        assert L.msg_score_device(eng._h, B, G - 1, odd.data_ptr(), prof.data_ptr(), C.byref(cfg),
                                  out_b.data_ptr()) == 0
        torch.cuda.synchronize()
        assert torch.equal(out_a, out_b), thr
        assert int((out_a[0::2] != -1).sum()) > B // 2  # most snapshots have a candidate
