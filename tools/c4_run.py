"""C4 (BASELINE.json configs[3]): one 16384-GPU cluster, 1M arrivals
(normal25 at ia = 25/2048 s, seed 0), all techniques — simulated by the block
engine on one B200.  Prints decisions/s; the reference needs ~12 h for it
(SURVEY §6), so its rate is measured on a prefix."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200.engine import Engine, generate_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

jobs = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ref_prefix = int(sys.argv[2]) if len(sys.argv) > 2 else 400
sp = preset("normal25")
sp.mean_interarrival_s = 25.0 / 2048
sp.job_count = jobs
eng = Engine(0)
batch = generate_batch(sp, 0, 1)
cfg = SimConfig(gpu_count=16384)
st = eng.stage(batch, [cfg], 0)
ms = st.time_launch()
res = st.collect()[0]
out = {"config": "C4: 16384 GPUs, %d arrivals, normal25 ia=25/2048 s, seed 0" % jobs, "status": res.code,
       "kernel_s": ms / 1e3, "handler_events": int(res.summary["handler_events"]),
       "decisions_per_s": int(res.summary["handler_events"]) / (ms / 1e3),
       "migrations": int(res.summary["migration_count"]), "makespan_s": res.workload_makespan_s,
       "mean_turnaround_s": res.mean_turnaround_s}
try:
    from oracle import refbind as rb

    if rb.ref_available() and ref_prefix:
        sp.job_count = ref_prefix
        b2 = generate_batch(sp, 0, 1)
        s, secs = rb.ref_run_batch_summaries(b2, [cfg], threads=1)
        g = eng.run_batch(b2, [cfg], 0)[0]
        out["reference_prefix"] = {"arrivals": ref_prefix, "seconds": secs,
                                   "decisions_per_s": float(s["handler_events"][0]) / secs,
                                   "gpu_makespan_equal": g.workload_makespan_s == float(s["workload_makespan_s"][0])}
except Exception as e:  # noqa: BLE001
    out["reference_prefix"] = str(e)
print(json.dumps(out))
