import glob, os, subprocess, sys
root = "/root/repo"
code = r'''
import os, sys, time
os.environ["MSG_PROFILE"] = "1"
sys.path.insert(0, "/root/repo")
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.engine import Engine, generate_batch, pin_batch
from paper_2512_16099_b200.model import SimConfig, preset
eng = Engine(0)
b = pin_batch(generate_batch(preset("normal25"), 0, 4096))
cfg = [SimConfig(gpu_count=8)]
for flags in (abi.OUT_JOBS, 0, abi.OUT_JOBS, 0):
    for i in range(6):
        r = eng.run_batch(b, cfg, flags); del r
'''
runs = [(lib, {"MSG_PROG_EVERY": v}) for lib in sorted(glob.glob(os.path.join(root, "build/variants/lib_*.so")))
        for v in sys.argv[1:] or ["64"]]
runs += [(os.path.join(root, "paper_2512_16099_b200/libmigsched_b200.so"), {"MSG_PROG_EVERY": v})
         for v in sys.argv[1:] or ["32"]]
for lib, extra in runs:
    env = dict(os.environ, MSG_B200_LIB=lib, **extra)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    ks = [l.split()[3] for l in r.stderr.splitlines() if "zero-copy kernel" in l]
    runs = [l.split()[3] for l in r.stderr.splitlines() if "pipelined run" in l]
    print(os.path.basename(lib), extra, "rows kernel", ks[2:6], ks[14:18], "| summaries kernel", ks[8:12], "| run", runs[2:6], runs[8:12])
