"""Host-side breakdown of the e2e path (development aid)."""
import os, sys, time
os.environ["MSG_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.engine import Engine, generate_batch
from paper_2512_16099_b200.model import SimConfig, preset
eng = Engine(0)
b = generate_batch(preset("normal25"), 0, 4096)
for i in range(3):
    t0 = time.perf_counter()
    r = eng.run_batch(b, [SimConfig(gpu_count=8)], abi.OUT_JOBS)
    print(f"python total {1e3*(time.perf_counter()-t0):.2f} ms", file=sys.stderr)
