"""Per-trace start/end times of the event-loop kernel (development aid).
Needs a library built with -DMSG_TRACE_TIMES (tools/hv_build.sh, FLAGS file),
selected with MSG_B200_LIB.  Modes: the device-timed C2 launch, and the
pipelined msg_run_batch (pageable and pinned inputs), where it shows when
each chunk's traces start and finish."""
import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200 import abi  # noqa: E402
from paper_2512_16099_b200 import engine as E  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch, pin_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

eng = Engine(0)
lib = E.lib()
T = 4096
b = generate_batch(preset("normal25"), 0, T)
cfg = [SimConfig(gpu_count=8)]
buf = (ctypes.c_ulonglong * (4 * 65536))()


def read():
    n = lib.msg_debug_trace_times(buf, 65536)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4)[:n].astype(np.int64)
    return a[np.argsort(a[:, 3])]


def report(tag, a, host_t0_ns=None):
    t0 = a[:, 0].min()
    s, e = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
    d = e - s
    print(f"{tag}: span {e.max():.0f} us; durations p0 {d.min():.0f} p50 {np.median(d):.0f} max {d.max():.0f}")
    for k in range(8):
        sl = slice(k * T // 8, (k + 1) * T // 8)
        print(f"   chunk {k}: start {s[sl].min():7.1f}..{s[sl].max():7.1f}  end p50 {np.median(e[sl]):7.1f} max {e[sl].max():7.1f}")


st = eng.stage(b, cfg, 0)
for _ in range(3):
    st.launch()
eng.sync()
read()
eng.flush_l2()
ms = st.time_launch()
report(f"staged launch ({ms*1e3:.0f} us)", read())
st.free()
for name, batch in (("run_batch pageable", b), ("run_batch pinned", pin_batch(b))):
    for _ in range(3):
        eng.run_batch(batch, cfg, abi.OUT_JOBS)
    read()
    t0 = time.perf_counter()
    r = eng.run_batch(batch, cfg, abi.OUT_JOBS)
    dt = time.perf_counter() - t0
    report(f"{name} ({dt*1e3:.3f} ms wall)", read())
