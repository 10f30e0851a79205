"""C4 on one B200 with the sharded block engine: the same trace at S CTAs
per cluster (MSG_SHARDS) x D device groups (MSG_VDEV; "SxD"), results
compared field by field (summary, per-job rows, timeline) against the first
configuration, kernel time per configuration.
usage: python tools/c4_shards.py [arrivals] [S | SxD ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2512_16099_b200 import abi  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

jobs = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
shards = sys.argv[2:] or ["1", "2", "4", "8", "16"]
sp = preset("normal25")
sp.mean_interarrival_s = 25.0 / 2048
sp.job_count = jobs
eng = Engine(0)
batch = generate_batch(sp, 0, 1)
cfg = SimConfig(gpu_count=16384)
base = None
for spec in shards:
    S, D = (spec.split("x") + ["1"])[:2]
    os.environ["MSG_SHARDS"] = S
    os.environ["MSG_VDEV"] = D
    st = eng.stage(batch, [cfg], abi.OUT_JOBS | abi.OUT_TIMELINE)
    ms = st.time_launch()
    res = st.collect()[0]
    out = {"arrivals": jobs, "shards": int(S), "groups": int(D), "status": res.code, "kernel_s": ms / 1e3,
           "decisions_per_s": int(res.summary["handler_events"]) / (ms / 1e3),
           "migrations": int(res.summary["migration_count"]), "makespan_s": res.workload_makespan_s,
           "timeline_sum": float(res.summary["timeline_sum"])}
    if base is None:
        base = res
    else:
        diffs = []
        for f in res.summary.dtype.names:
            if np.asarray(res.summary[f]).tobytes() != np.asarray(base.summary[f]).tobytes():
                diffs.append(f)
        if res.per_job.tobytes() != base.per_job.tobytes():
            diffs.append("per_job")
        if res.frag_timeline.tobytes() != base.frag_timeline.tobytes():
            diffs.append("timeline")
        out["identical_to_first"] = not diffs
        out["diffs"] = diffs
    print(json.dumps(out), flush=True)
