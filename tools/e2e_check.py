"""e2e msg_run_batch timing in isolation (development aid): result held vs
dropped, with and without torch's CUDA runtime initialised first."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "torch" in sys.argv[1:]:
    import torch
    torch.cuda.set_device(0)
    x = torch.ones(1 << 20, device="cuda")
    torch.cuda.synchronize()
from paper_2512_16099_b200 import abi
from paper_2512_16099_b200.engine import Engine, generate_batch
from paper_2512_16099_b200.model import SimConfig, preset
eng = Engine(0)
b = generate_batch(preset("normal25"), 0, 4096)
cfg = [SimConfig(gpu_count=8)]
if "staged" in sys.argv[1:]:  # what bench.py does first: a staged copy, timed launches with L2 flushes
    st = eng.stage(b, cfg, 0)
    for _ in range(13):
        eng.flush_l2()
        st.time_launch()
if "nvml" in sys.argv[1:]:  # bench.py's clock sampler around a short region
    import bench
    c = bench.ClockSampler(0)
    c.start()
    time.sleep(0.05)
    c.stop()
if "bench" in sys.argv[1:]:  # bench.py's own workload object
    import bench
    bench.TRACES_RUN = 4096
    b, cfg0 = bench.workload(0)
    cfg = [cfg0]
for mode in ("hold", "drop", "hold", "drop"):
    for _ in range(3):
        out = eng.run_batch(b, cfg, abi.OUT_JOBS)
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
    print(sys.argv[1:], mode, "mean %.3f median %.3f min %.3f max %.3f" % (1e3 * sum(ts) / len(ts), 1e3 * s[7],
                                                                          1e3 * s[0], 1e3 * s[-1]))
