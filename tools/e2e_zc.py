"""Zero-copy / progressive-row variants of the C2 msg_run_batch with host
phases and the zero-copy kernel's device time (development aid)."""
import os, sys, time
os.environ["MSG_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200 import abi  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch, pin_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

eng = Engine(0)
b = pin_batch(generate_batch(preset("normal25"), 0, 4096))
cfg = [SimConfig(gpu_count=8)]
for name, env, flags in (("zc + prog rows", {}, abi.OUT_JOBS), ("zc summaries", {}, 0),
                         ("zc + prog rows, backoff 0", {"MSG_POLL_BACKOFF": "0"}, abi.OUT_JOBS),
                         ("zc + prog rows, backoff 128", {"MSG_POLL_BACKOFF": "128"}, abi.OUT_JOBS),
                         ("zc + prog rows /64", {"MSG_PROG_EVERY": "64"}, abi.OUT_JOBS),
                         ("zc rows, no prog", {"MSG_PIPE_PROG": "0"}, abi.OUT_JOBS),
                         ("staged no prog", {"MSG_NO_ZC": "1", "MSG_PIPE_PROG": "0"}, abi.OUT_JOBS),
                         ("zc + prog rows", {}, abi.OUT_JOBS)):
    os.environ.update(env)
    for i in range(8):
        print(f"--- {name} call {i}", file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        r = eng.run_batch(b, cfg, flags)
        print(f"{name} call {i}: {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
        del r
    for k in env:
        del os.environ[k]
