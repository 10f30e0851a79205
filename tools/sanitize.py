"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): one case per kernel family, sized so the instrumented run takes
seconds.  Usage (GPU box):

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize.py sim

Cases:
  sim       sim_kernel: C1/C5-shaped batches (8 GPUs, events + timeline), the
            pipelined msg_run_batch (>= 512 traces, mapped-host completion
            flags polled by host threads), the zero-copy IO kernel on
            page-locked inputs (progressive rows), ties at 32 GPUs
  score     score_tma_kernel + merge + score_busy_kernel (bulk-async ring,
            mbarriers), thresholds 0.0 / 0.4 / 1.0
  snapshot  snapshot kernels: schedule / first fit / try_dequeue / planners
  cluster   cluster_kernel: 16384-GPU C4 prefix at S = 16 (DSMEM st.async
            exchange) and at MSG_VDEV=2 (two device groups: peer-stamp inboxes)
            plus 600 GPUs at S = 1
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def case_sim(eng):
    from paper_2512_16099_b200 import abi
    from paper_2512_16099_b200.engine import generate_batch
    from paper_2512_16099_b200.model import FIXED, SchedulerConfig, SimConfig, WorkloadSpec, preset

    ALL = abi.OUT_JOBS | abi.OUT_EVENTS | abi.OUT_TIMELINE
    b = generate_batch(preset("normal25"), 0, 8)
    r = eng.run_batch(b, [SimConfig(gpu_count=8)], ALL)
    assert all(x.ok for x in r)
    c5 = WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, profile_mix=(0.5, 0.3, 0.2, 0.0))
    r = eng.run_batch(generate_batch(c5, 0, 8), [SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3),
                                                          migration_overlap_s=0.5, reconfig_latency_s=0.1)], ALL)
    assert all(x.ok for x in r)
    ties = WorkloadSpec(mean_interarrival_s=4.0, family=FIXED, value_s=20.0, job_count=100)
    r = eng.run_batch(generate_batch(ties, 0, 4), [SimConfig(gpu_count=32, migration_overlap_s=1.0,
                                                            reconfig_latency_s=0.25)], ALL)
    assert all(x.ok for x in r)
    sp = preset("normal25")
    sp.job_count = 40
    r = eng.run_batch(generate_batch(sp, 0, 600), [SimConfig(gpu_count=8)], abi.OUT_JOBS)  # pipelined
    assert all(x.ok for x in r)
    from paper_2512_16099_b200.engine import pin_batch

    # page-locked inputs: the zero-copy IO kernel (inputs read over PCIe,
    # progressive SoA job rows + prefix words in mapped host memory)
    pb = pin_batch(generate_batch(sp, 0, 600))
    rz = eng.run_batch(pb, [SimConfig(gpu_count=8)], abi.OUT_JOBS)
    assert all(x.ok for x in rz) and rz.jobs.tobytes() == r.jobs.tobytes()
    print("sim ok")


def case_score(eng):
    import ctypes as C

    import torch

    from paper_2512_16099_b200 import decisions
    from paper_2512_16099_b200.model import SchedulerConfig

    L = decisions._bind()
    B, G = 64, 16384
    gen = torch.Generator(device="cuda").manual_seed(1)
    rnd = torch.randint(0, 1 << 30, (B, G), device="cuda", dtype=torch.int64, generator=gen)
    bm = rnd & 0x7F
    words = (bm | (bm << 8) | (bm << 16)).contiguous()
    prof = torch.randint(0, 6, (B,), device="cuda", dtype=torch.uint8, generator=gen)
    out = torch.empty(B * 2, device="cuda", dtype=torch.int64)
    for thr in (0.4, 0.0, 1.0):
        cfg = decisions._sched_cfg(SchedulerConfig(threshold=thr))
        assert L.msg_score_device(eng._h, B, G, words.data_ptr(), prof.data_ptr(), C.byref(cfg),
                                  out.data_ptr()) == 0
        torch.cuda.synchronize()
    print("score ok")


def case_snapshot(eng):
    from helpers import random_cluster

    from paper_2512_16099_b200 import abi, decisions
    from paper_2512_16099_b200.model import SchedulerConfig

    rng = np.random.default_rng(3)
    G, n = 8, 64
    slots = np.stack([random_cluster(rng, G) for _ in range(n)])
    prof = rng.integers(0, 6, n)
    for op in (abi.OP_SCHEDULE, abi.OP_FIRST_FIT, abi.OP_DISPATCH):
        decisions.schedule_batch(op, slots, prof, SchedulerConfig(), G, engine=eng)
    for op in (abi.PLAN_ON_DEPARTURE, abi.PLAN_INTRA, abi.PLAN_INTER):
        s = slots.copy()
        decisions.plan_batch(op, s, rng.integers(0, G, n), gpu_count=G, engine=eng)
    decisions.frag_cost_batch(slots.reshape(-1, 8), engine=eng)
    print("snapshot ok")


def case_cluster(eng):
    from paper_2512_16099_b200 import abi
    from paper_2512_16099_b200.engine import generate_batch
    from paper_2512_16099_b200.model import SimConfig, preset

    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 2048
    sp.job_count = 300
    b = generate_batch(sp, 0, 1)
    want = eng.run_batch(b, [SimConfig(gpu_count=16384)], abi.OUT_JOBS)[0]
    assert want.ok
    os.environ["MSG_VDEV"] = "2"
    got = eng.run_batch(b, [SimConfig(gpu_count=16384)], abi.OUT_JOBS)[0]
    del os.environ["MSG_VDEV"]
    assert got.per_job.tobytes() == want.per_job.tobytes()
    sp.mean_interarrival_s = 25.0 / 75
    sp.job_count = 200
    r = eng.run_batch(generate_batch(sp, 0, 1), [SimConfig(gpu_count=600)], abi.OUT_JOBS | abi.OUT_EVENTS)[0]
    assert r.ok
    print("cluster ok")


def main():
    from paper_2512_16099_b200.engine import Engine

    eng = Engine(0)
    cases = sys.argv[1:] or ["sim", "score", "snapshot", "cluster"]
    for c in cases:
        globals()["case_" + c](eng)


if __name__ == "__main__":
    main()
