"""Reference goldens for the C4 prefixes that bench.py times (BASELINE.json
configs[3]): one 16384-GPU cluster, preset normal25 at ia = 25/2048 s, seed 0
(SURVEY §8d), first 2,000 and 20,000 arrivals.

The UNMODIFIED reference library (oracle/_ref, built by oracle/Makefile from
/root/reference/proj/src) runs each prefix once, single-threaded, through
`migsched::run` (sim.cpp:504-507) — about 15 minutes for the 20K prefix on
the build box.  Run here (needs /root/reference):

    python tests/golden/make_c4_golden.py

Writes tests/golden/c4_prefix.npz: per prefix the reference's per-job rows
(scheduled, completed, gpu, migrations in job-id order), its summary (counts,
makespan, mean turnaround, timeline_sum), the wall seconds it took, and a
checksum of the timeline sample bits.  The trace itself is regenerated on the
GPU box by the product generator (bit-identical to the reference generator,
tests/test_generator.py) and checked against the stored arrival checksum.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refbind as rb  # noqa: E402
from paper_2512_16099_b200 import abi  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

PREFIXES = (2000, 20000)


def c4_spec(n):
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 2048
    sp.job_count = n
    return sp


def main(prefixes=PREFIXES):
    out = {}
    path = os.path.join(HERE, "c4_prefix.npz")
    if os.path.exists(path):
        with np.load(path) as z:
            out = {k: z[k] for k in z.files}
    cfg = SimConfig(gpu_count=16384)
    for n in prefixes:
        b = rb.ref_generate_batch(c4_spec(n), [0])
        t0 = time.perf_counter()
        r = rb.ref_run_batch_results(b, [cfg])[0]
        secs = time.perf_counter() - t0
        assert r.ok, r.message
        j = r.per_job
        out[f"n{n}/scheduled"] = j["scheduled_s"]
        out[f"n{n}/completed"] = j["completed_s"]
        out[f"n{n}/gpu"] = j["gpu"]
        out[f"n{n}/migrations"] = j["migrations"]
        out[f"n{n}/summary"] = np.array([r.summary], abi.SUMMARY_DTYPE)
        out[f"n{n}/seconds"] = np.array([secs])
        out[f"n{n}/arrival_checksum"] = np.array([b.arrival_s.view(np.uint64).sum(dtype=np.uint64)])
        tl = r.frag_timeline
        out[f"n{n}/timeline_checksum"] = np.array([tl["mean_frag_cost"].view(np.uint64).sum(dtype=np.uint64)])
        out[f"n{n}/timeline_len"] = np.array([len(tl)])
        print(f"C4 prefix {n}: {secs:.1f} s, {int(r.summary['handler_events'])} handler events, "
              f"makespan {float(r.summary['workload_makespan_s'])!r}", flush=True)
        np.savez_compressed(path, **out)


if __name__ == "__main__":
    main(tuple(int(a) for a in sys.argv[1:]) or PREFIXES)
