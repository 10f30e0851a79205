"""Generate tests/golden/* from the UNMODIFIED reference library.

Run on the build box (needs oracle/_ref/libmigsched_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile):

    python tests/golden/make_golden.py

Fixtures (small, committed):
  runs.npz        per case: trace arrays, config, and the reference's event
                  log / per-job rows / timeline / summary in the ABI formats
  events_c1.jsonl the reference's own events_to_jsonl text for C1 (G=8)
  aggregates.json ensemble aggregates (C2 / C5 / C3 subsets) from the
                  reference, for full-size GPU checks
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refbind as rb  # noqa: E402
from paper_2512_16099_b200 import abi  # noqa: E402
from paper_2512_16099_b200.model import (  # noqa: E402
    FIXED,
    FeatureFlags,
    Job,
    SchedulerConfig,
    SimConfig,
    TraceBatch,
    WorkloadSpec,
    preset,
    static_layout_preset,
)


def cfg_dict(c: SimConfig) -> dict:
    return {
        "threshold": c.sched.threshold,
        "lb": c.sched.features.load_balancing,
        "dyn": c.sched.features.dynamic_partitioning,
        "mig": c.sched.features.migration,
        "layout": c.sched.static_layout,
        "alpha": c.contention_alpha,
        "overlap": c.migration_overlap_s,
        "latency": c.reconfig_latency_s,
        "gpus": c.gpu_count,
    }


def cfg_from(d: dict) -> SimConfig:
    return SimConfig(
        sched=SchedulerConfig(d["threshold"], FeatureFlags(d["lb"], d["dyn"], d["mig"]),
                              None if d["layout"] is None else [[tuple(e) for e in g] for g in d["layout"]]),
        contention_alpha=d["alpha"], migration_overlap_s=d["overlap"], reconfig_latency_s=d["latency"],
        gpu_count=d["gpus"])


def cases():
    c5 = WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, profile_mix=(0.5, 0.3, 0.2, 0.0))
    c5cfg = SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                      reconfig_latency_s=0.1)
    ties = WorkloadSpec(mean_interarrival_s=4.0, family=FIXED, value_s=20.0, job_count=120)
    yield "c1_g8_s0", preset("normal25"), 0, SimConfig(gpu_count=8)
    yield "c1_g4_s0", preset("normal25"), 0, SimConfig(gpu_count=4)
    yield "long25_g4_s7", preset("long25"), 7, SimConfig(gpu_count=4)
    for s in (0, 1):
        yield f"c5_s{s}", c5, s, c5cfg
    for i, f in enumerate([FeatureFlags(False, False, False), FeatureFlags(True, False, False),
                           FeatureFlags(True, True, False)]):
        sp = preset("normal25")
        sp.mean_interarrival_s = 10.0
        yield f"c3_combo{i}_ia10", sp, 3, SimConfig(gpu_count=4, sched=SchedulerConfig(
            features=f, static_layout=None if f.dynamic_partitioning else static_layout_preset("static-a")))
    yield "ties_g3", ties, 2, SimConfig(gpu_count=3, reconfig_latency_s=0.25, migration_overlap_s=1.0)


def aggregates(only=None):
    """Ensemble aggregates (full-size checks on the GPU box): C2 and C5 at
    4096 seeds and the whole C3 grid (4 combos x 5 loads
    x 1024 seeds, run_ablation's combos, tools/migsched.cpp:64-99).  `only`
    recomputes a subset of the tags and keeps the other stored entries."""
    path = os.path.join(HERE, "aggregates.json")
    agg = json.load(open(path)) if os.path.exists(path) else {}

    def aggregate(tag, spec, seeds, cfg):
        if only is not None and tag not in only:
            return
        b = rb.ref_generate_batch(spec, seeds) if spec is not None else None
        s, _ = rb.ref_run_batch_summaries(b, [cfg], threads=0)
        agg[tag] = {
            "seeds": [int(seeds[0]), int(seeds[-1])],
            "spec": spec.__dict__,
            "cfg": cfg_dict(cfg),
            "handler_events": int(s["handler_events"].sum()),
            "migrations": int(s["migration_count"].sum()),
            "reconfig_ops": int(s["reconfig_op_count"].sum()),
            "dequeues": int(s["dequeue_count"].sum()),
            "sum_mean_turnaround": float(np.add.reduce(s["mean_turnaround_s"])),
            "mean_turnaround_bits": s["mean_turnaround_s"].tobytes().hex()[:0],
            "checksum_turnaround": s["mean_turnaround_s"].view(np.uint64).sum(dtype=np.uint64).item(),
            "checksum_makespan": s["workload_makespan_s"].view(np.uint64).sum(dtype=np.uint64).item(),
            "checksum_timeline": s["timeline_sum"].view(np.uint64).sum(dtype=np.uint64).item(),
        }

    aggregate("c2_4096", preset("normal25"), list(range(4096)), SimConfig(gpu_count=8))
    c5 = WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, profile_mix=(0.5, 0.3, 0.2, 0.0))
    aggregate("c5_4096", c5, list(range(4096)), SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3),
                                                          migration_overlap_s=0.5, reconfig_latency_s=0.1))
    for ia in C3_LOADS:
        for i, f in enumerate(C3_COMBOS):
            sp = preset("normal25")
            sp.mean_interarrival_s = float(ia)
            aggregate(f"c3_ia{ia}_combo{i}", sp, list(range(1024)), SimConfig(gpu_count=4, sched=SchedulerConfig(
                features=f, static_layout=None if f.dynamic_partitioning else static_layout_preset("static-a"))))
    with open(path, "w") as f:
        json.dump(agg, f, indent=1)
    return agg


C3_LOADS = (10, 15, 25, 35, 50)
C3_COMBOS = (FeatureFlags(False, False, False), FeatureFlags(True, False, False),
             FeatureFlags(True, True, False), FeatureFlags(True, True, True))


def main():
    arrays = {}
    meta = {}
    for name, spec, seed, cfg in cases():
        b = rb.ref_generate_batch(spec, [seed])
        r = rb.ref_run_batch_results(b, [cfg], texts=(name == "c1_g8_s0"))[0]
        assert r.ok, (name, r.message)
        arrays[f"{name}/id"] = b.job_id
        arrays[f"{name}/arrival"] = b.arrival_s
        arrays[f"{name}/profile"] = b.profile
        arrays[f"{name}/service"] = b.service_s
        arrays[f"{name}/events"] = r.events
        arrays[f"{name}/jobs"] = r.per_job
        arrays[f"{name}/timeline"] = r.frag_timeline
        arrays[f"{name}/summary"] = np.array([r.summary], abi.SUMMARY_DTYPE)
        meta[name] = {"seed": seed, "spec": spec.__dict__, "cfg": cfg_dict(cfg)}
        if name == "c1_g8_s0":
            with open(os.path.join(HERE, "events_c1.jsonl"), "w") as f:
                f.write(r.texts[0])
    # Hand-built traces with shuffled ids, equal times and a negative arrival.
    hand = [Job(7, 0.0, 5, 10.0), Job(3, 0.0, 3, 5.0), Job(5, 0.0, 5, 10.0), Job(1, 1.0, 2, 3.0),
            Job(9, -0.5, 0, 4.0), Job(2, 1.0, 4, 2.0)]
    hand.sort(key=lambda j: j.arrival_s)
    b = TraceBatch.from_traces([hand])
    for G in (1, 2):
        cfg = SimConfig(gpu_count=G, migration_overlap_s=3.0)
        r = rb.ref_run_batch_results(b, [cfg])[0]
        name = f"hand_g{G}"
        for k, v in (("id", b.job_id), ("arrival", b.arrival_s), ("profile", b.profile), ("service", b.service_s),
                     ("events", r.events), ("jobs", r.per_job), ("timeline", r.frag_timeline),
                     ("summary", np.array([r.summary], abi.SUMMARY_DTYPE))):
            arrays[f"{name}/{k}"] = v
        meta[name] = {"seed": None, "spec": None, "cfg": cfg_dict(cfg)}
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **arrays)
    with open(os.path.join(HERE, "runs.json"), "w") as f:
        json.dump(meta, f, indent=1)

    agg = aggregates()
    print("wrote", len(meta), "runs and", len(agg), "aggregates")


if __name__ == "__main__":
    if sys.argv[1:] == ["aggregates"]:
        print("aggregates:", len(aggregates()))
    elif sys.argv[1:2] == ["aggregates"]:
        print("aggregates:", len(aggregates(only=set(sys.argv[2:]))))
    else:
        main()
