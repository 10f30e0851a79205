"""Cold vs warm msg_run_batch on the C2 ensemble (development aid): a fresh
engine, then the first calls timed one by one, host phases on stderr
(MSG_PROFILE=1)."""
import os
import sys
import time

os.environ.setdefault("MSG_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200 import abi  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

t0 = time.perf_counter()
eng = Engine(0)
print(f"engine create {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
b = generate_batch(preset("normal25"), 0, 4096)
for i in range(6):
    print(f"--- call {i}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    r = eng.run_batch(b, [SimConfig(gpu_count=8)], abi.OUT_JOBS)
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
    del r
