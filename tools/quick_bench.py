"""Quick device timing of the C2 ensemble (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200.engine import Engine, generate_batch
from paper_2512_16099_b200.model import SimConfig, preset
from paper_2512_16099_b200 import abi
eng = Engine(0)
print(eng.device_info())
for T, G in ((4096, 8), (16384, 8), (4096, 4)):
    b = generate_batch(preset("normal25"), 0, T)
    st = eng.stage(b, [SimConfig(gpu_count=G)], 0)
    for _ in range(3): st.launch()
    eng.sync()
    ts = []
    for _ in range(5):
        eng.flush_l2()
        ts.append(st.time_launch())
    res = st.collect()
    ev = st.handler_events
    ms = min(ts)
    print(f"T={T} G={G}: kernel {ms:.3f} ms (all {['%.3f'%x for x in ts]}), handler events {ev}, {ev/ms*1e3:.3e} ev/s")
    t0 = time.perf_counter()
    for _ in range(3): r = eng.run_batch(b, [SimConfig(gpu_count=G)], abi.OUT_JOBS)
    dt = (time.perf_counter() - t0) / 3
    print(f"   e2e run_batch (jobs out) {dt*1e3:.2f} ms -> {ev/dt:.3e} ev/s")
