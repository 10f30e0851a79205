"""C2 msg_run_batch timing under host-side variants (development aid): per-job
rows vs summaries only, non-temporal row stores on/off, pipeline chunk
weights, host thread counts; plus a host-memory bandwidth reference (numpy
copy of 64 MiB)."""
import faulthandler, os, sys, time
faulthandler.dump_traceback_later(150, exit=True)  # a hang prints every thread's stack
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200 import abi  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch, pin_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

eng = Engine(0)
b = generate_batch(preset("normal25"), 0, 4096)
cfg = [SimConfig(gpu_count=8)]
x = np.ones(8 << 20)
y = np.empty_like(x)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); np.copyto(y, x); ts.append(time.perf_counter() - t0)
print(f"host copy 64 MiB: {min(ts)*1e3:.2f} ms = {2*x.nbytes/min(ts)/1e9:.1f} GB/s (read+write)")
st = eng.stage(b, cfg, 0)
for _ in range(3):
    st.launch()
eng.sync()
k = []
for _ in range(5):
    eng.flush_l2(); k.append(st.time_launch())
print(f"kernel {min(k):.3f} ms")
st.free()


bp = pin_batch(b)
r0 = eng.run_batch(b, cfg, abi.OUT_JOBS)
r1 = eng.run_batch(bp, cfg, abi.OUT_JOBS)
print("pinned == pageable results:", r0.summaries.tobytes() == r1.summaries.tobytes() and r0.jobs.tobytes() == r1.jobs.tobytes())
del r0, r1


def timeit(flags, n=15, batch=None):
    batch = b if batch is None else batch
    for _ in range(3):
        out = eng.run_batch(batch, cfg, flags)
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        out = eng.run_batch(batch, cfg, flags)
        ts.append(time.perf_counter() - t0)
        del out
    ts.sort()
    return f"median {1e3*ts[n//2]:.3f} min {1e3*ts[0]:.3f} ms"


modes = [("jobs", {}, abi.OUT_JOBS), ("PINNED jobs (zero copy)", {}, abi.OUT_JOBS),
         ("PINNED jobs zc, no progressive rows", {"MSG_PIPE_PROG": "0"}, abi.OUT_JOBS),
         ("PINNED jobs staged chunks", {"MSG_NO_ZC": "1"}, abi.OUT_JOBS),
         ("PINNED jobs staged chunks, no prog", {"MSG_NO_ZC": "1", "MSG_PIPE_PROG": "0"}, abi.OUT_JOBS),
         ("PINNED summaries", {}, 0), ("summaries only", {}, 0),
         ("jobs, no progressive rows", {"MSG_PIPE_PROG": "0"}, abi.OUT_JOBS),
         ("PINNED jobs (zero copy)", {}, abi.OUT_JOBS), ("jobs", {}, abi.OUT_JOBS)]
for name, env, flags in modes:
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    print(f"{name:40s} {timeit(flags, batch=bp if name.startswith('PINNED') else None)}", flush=True)
    for k2, v in old.items():
        if v is None:
            del os.environ[k2]
        else:
            os.environ[k2] = v
