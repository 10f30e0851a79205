"""Where the event-loop kernel's tail comes from (development aid; needs a
-DMSG_TRACE_TIMES library in MSG_B200_LIB): (1) C2 as is, per-trace
durations saved with each trace's summary counters to
gpurun_out/trace_spread.npz; (2) one trace replicated 4096 times, so the
spread left is placement / contention, not content."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200 import abi  # noqa: E402
from paper_2512_16099_b200 import engine as E  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, TraceBatch, preset  # noqa: E402

eng = Engine(0)
lib = E.lib()
buf = (ctypes.c_ulonglong * (4 * 65536))()
cfg = [SimConfig(gpu_count=8)]


def run(b):
    st = eng.stage(b, cfg, abi.OUT_JOBS)
    for _ in range(2):
        st.launch()
    eng.sync()
    lib.msg_debug_trace_times(buf, 65536)
    eng.flush_l2()
    ms = st.time_launch()
    n = lib.msg_debug_trace_times(buf, 65536)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4)[:n].astype(np.int64)
    a = a[np.argsort(a[:, 3], kind="stable")]
    res = st.collect()
    st.free()
    return ms, a, res


b = generate_batch(preset("normal25"), 0, 4096)
ms, a, res = run(b)
d = (a[:, 1] - a[:, 0]) / 1e3
summ = np.array([r.summary for r in res])
np.savez(os.path.join("gpurun_out", "trace_spread.npz"), dur_us=d, sm=a[:, 2], start=a[:, 0], end=a[:, 1], summary=summ)
print(f"C2: kernel {ms*1e3:.0f} us; dur p0 {d.min():.0f} p50 {np.median(d):.0f} p99 {np.percentile(d, 99):.0f} max {d.max():.0f}")
for seed in (0, 17):
    one = generate_batch(preset("normal25"), seed, 1)
    rep = TraceBatch.concat([one] * 4096)
    ms, a, _ = run(rep)
    d = (a[:, 1] - a[:, 0]) / 1e3
    print(f"seed {seed} x4096: kernel {ms*1e3:.0f} us; dur p0 {d.min():.0f} p50 {np.median(d):.0f} p99 {np.percentile(d, 99):.0f} max {d.max():.0f}")
