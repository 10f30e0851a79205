"""bench.py's e2e loop on the C2 ensemble, with per-step times (development
aid): previous result kept alive during the next call (as bench.py did) vs
released first."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2512_16099_b200 import abi  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch, pin_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

if os.environ.get("WITH_TORCH"):  # as bench.py: torch's CUDA context first
    import torch
    torch.cuda.set_device(0)
eng = Engine(0)
b = pin_batch(generate_batch(preset("normal25"), 0, 4096))
cfg = [SimConfig(gpu_count=8)]
for keep in (True, False, True, False):
    out = None
    for _ in range(3):
        out = eng.run_batch(b, cfg, abi.OUT_JOBS)
    ts = []
    gc.disable()
    for _ in range(20):
        if not keep:
            out = None
        t0 = time.perf_counter()
        out = eng.run_batch(b, cfg, abi.OUT_JOBS)
        s = np.ascontiguousarray(out.summaries)
        ts.append(time.perf_counter() - t0)
    gc.enable()
    ts = sorted(1e3 * t for t in ts)
    print(f"keep previous={keep}: mean {sum(ts)/len(ts):.3f} median {ts[10]:.3f} min {ts[0]:.3f} max {ts[-1]:.3f} ms")
