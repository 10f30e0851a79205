"""C2 msg_run_batch with job rows (page-locked inputs) under host-side
environment settings, each in its own process (development aid)."""
import os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import gc, sys, time; sys.path.insert(0, %r)
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.engine import Engine, generate_batch, pin_batch
from paper_2512_16099_b200.model import SimConfig, preset
eng = Engine(0)
b = pin_batch(generate_batch(preset("normal25"), 0, 4096))
cfg = [SimConfig(gpu_count=8)]
out = []
for flags, name in ((abi.OUT_JOBS, "rows"), (0, "summaries")):
    for _ in range(3):
        r = eng.run_batch(b, cfg, flags); del r
    ts = []
    gc.disable()
    for _ in range(20):
        t0 = time.perf_counter(); r = eng.run_batch(b, cfg, flags); ts.append(time.perf_counter() - t0); del r
    gc.enable()
    ts.sort()
    out.append("%%s median %%.3f min %%.3f ms" %% (name, 1e3 * ts[10], 1e3 * ts[0]))
print(" | ".join(out))
''' % root
for env in ({}, {"MSG_HOST_THREADS": "8"}, {"MSG_HOST_THREADS": "4"}, {"MSG_ROWS_NT": "0"}, {}):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
    print(env, r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
