"""Time the event-loop kernel of each build/hv/lib_*.so variant on C2 (8
GPUs), C3-shaped (4 GPUs), C5 and 32-GPU traces, and check every summary
against the product library's (development aid; run on the GPU box)."""
import glob, json, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json, hashlib; sys.path.insert(0, %r)
import numpy as np
from paper_2512_16099_b200.engine import Engine, generate_batch
from paper_2512_16099_b200.model import SimConfig, SchedulerConfig, WorkloadSpec, preset
eng = Engine(0)
c5 = WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, profile_mix=(0.5, 0.3, 0.2, 0.0))
cases = [("c2", preset("normal25"), SimConfig(gpu_count=8), 4096),
         ("g4", preset("normal25"), SimConfig(gpu_count=4), 4096),
         ("c5", c5, SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3), migration_overlap_s=0.5,
                             reconfig_latency_s=0.1), 4096),
         ("g32", preset("normal25"), SimConfig(gpu_count=32), 1024)]
out = {}
for name, spec, cfg, T in cases:
    b = generate_batch(spec, 0, T)
    st = eng.stage(b, [cfg], 0)
    for _ in range(3): st.launch()
    eng.sync()
    res = st.collect()
    h = hashlib.sha1()
    for r in res: h.update(np.ascontiguousarray(r.summary).tobytes()); h.update(np.ascontiguousarray(r.jobs).tobytes() if getattr(r, "jobs", None) is not None else b"")
    ts = []
    for _ in range(7):
        eng.flush_l2(); ts.append(st.time_launch())
    ts.sort()
    out[name] = {"ms": ts[len(ts)//2], "min": ts[0], "hash": h.hexdigest()[:12]}
    st.free()
print(json.dumps(out))
''' % root
libs = sorted(glob.glob(os.path.join(root, "build/hv/lib_*.so")))  # lib_v0_* (the committed kernels) first: the parity base
if os.environ.get("HV_LIBS"):
    libs = [os.path.join(root, x) for x in os.environ["HV_LIBS"].split(",")]
envs = [dict(kv.split("=", 1) for kv in e.split("+") if kv) for e in os.environ.get("HV_ENVS", "").split(";")]
base = None
for rep in range(int(os.environ.get("HV_REPS", "2"))):
    for lib in libs:
        for ev in envs:
            env = dict(os.environ, MSG_B200_LIB=lib, **ev)
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception:
                print(os.path.basename(lib), ev, "FAILED", r.stderr[-600:]); continue
            if base is None: base = d
            same = all(d[k]["hash"] == base[k]["hash"] for k in d)
            tag = os.path.basename(lib) + (" " + ",".join(f"{k}={v}" for k, v in ev.items()) if ev else "")
            print(f"{tag:40s} " + " ".join(f"{k} {v['ms']:.4f}/{v['min']:.4f}" for k, v in d.items()) + f"  parity={'OK' if same else 'DIFF'}", flush=True)
