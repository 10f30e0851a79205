import os, sys, time, gc
sys.path.insert(0, "/root/repo")
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.engine import Engine, generate_batch
from paper_2512_16099_b200.model import SimConfig, preset
eng = Engine(0)
b = generate_batch(preset("normal25"), 0, 4096)
cfg = [SimConfig(gpu_count=8)]
for mode in ("hold", "drop", "hold", "drop"):
    for _ in range(3): out = eng.run_batch(b, cfg, abi.OUT_JOBS)
    ts = []
    for _ in range(15):
        t0 = time.perf_counter()
        if mode == "hold":
            out = eng.run_batch(b, cfg, abi.OUT_JOBS)
        else:
            eng.run_batch(b, cfg, abi.OUT_JOBS)
        ts.append(time.perf_counter() - t0)
    out = None
    s = sorted(ts)
    print(mode, "mean %.3f median %.3f min %.3f max %.3f" % (1e3*sum(ts)/len(ts), 1e3*s[7], 1e3*s[0], 1e3*s[-1]))
