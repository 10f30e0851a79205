"""e2e msg_run_batch time vs pipeline chunk weights (MSG_PIPE_W; development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.engine import Engine, generate_batch
from paper_2512_16099_b200.model import SimConfig, preset
eng = Engine(0)
b = generate_batch(preset("normal25"), 0, 4096)
cfg = [SimConfig(gpu_count=8)]
shapes = sys.argv[1:] or ["1,1,1,1", "1,1", "1,1,1,1,1,1,1,1", "1,2,2,3", "1,2,3,2", "2,3,3,2", "1,1,1,1,1,1", "3,3,2,1"]
for rep in range(2):
    for w in shapes:
        os.environ["MSG_PIPE_W"] = w
        for _ in range(3):
            eng.run_batch(b, cfg, abi.OUT_JOBS)
        ts = []
        for _ in range(15):
            t0 = time.perf_counter()
            eng.run_batch(b, cfg, abi.OUT_JOBS)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        print(f"W={w:18s} median {1e3*ts[len(ts)//2]:.3f} ms  min {1e3*ts[0]:.3f} ms")
