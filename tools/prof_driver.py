"""Short driver for ncu captures: C2 event-loop launches + scorer sweeps."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_16099_b200 import decisions  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch  # noqa: E402
from paper_2512_16099_b200.model import SchedulerConfig, SimConfig, preset  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "both"
eng = Engine(0)
if what in ("sim", "both"):
    b = generate_batch(preset("normal25"), 0, 4096)
    st = eng.stage(b, [SimConfig(gpu_count=8)], 0)
    for _ in range(2):
        st.launch()
    eng.sync()
if what in ("score", "both"):
    L = decisions._bind()
    B, G = 4096, 16384
    g = torch.Generator(device="cuda").manual_seed(1)
    rnd = torch.randint(0, 1 << 30, (B, G), device="cuda", dtype=torch.int64, generator=g)
    bm = rnd & 0x7F
    words = (bm | (bm << 8) | (bm << 16)).contiguous()
    prof = torch.randint(0, 6, (B,), device="cuda", dtype=torch.uint8, generator=g)
    out = torch.empty(B * 2, device="cuda", dtype=torch.int64)
    cfg = decisions._sched_cfg(SchedulerConfig())
    for _ in range(2):
        L.msg_score_device(eng._h, B, G, words.data_ptr(), prof.data_ptr(), C.byref(cfg), out.data_ptr())
    eng.sync()
print("done")
