"""Host phases (MSG_PROFILE) of the C2 msg_run_batch with rows and with summaries only (development aid)."""
import os, sys, time
os.environ["MSG_PROFILE"] = "1"
sys.path.insert(0, os.getcwd())
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.engine import Engine, generate_batch, pin_batch
from paper_2512_16099_b200.model import SimConfig, preset
eng = Engine(0)
b = pin_batch(generate_batch(preset("normal25"), 0, 4096))
cfg = [SimConfig(gpu_count=8)]
for flags, name in ((abi.OUT_JOBS, "rows"), (0, "summaries")):
    for i in range(6):
        print(f"--- {name} {i}", file=sys.stderr, flush=True)
        t0 = time.perf_counter(); r = eng.run_batch(b, cfg, flags); t1 = time.perf_counter()
        print(f"{name} {i}: {1e3*(t1-t0):.3f} ms", file=sys.stderr, flush=True)
        del r
