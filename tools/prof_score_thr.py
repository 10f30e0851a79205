"""One scorer launch (msg_score_device) at a given threshold, for ncu captures (development aid).
usage: python tools/prof_score_thr.py [threshold]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_16099_b200 import decisions  # noqa: E402
from paper_2512_16099_b200.engine import Engine  # noqa: E402
from paper_2512_16099_b200.model import SchedulerConfig  # noqa: E402

thr = float(sys.argv[1]) if len(sys.argv) > 1 else 0.4
eng = Engine(0)
L = decisions._bind()
B, G = 4096, 16384
g = torch.Generator(device="cuda").manual_seed(1)
rnd = torch.randint(0, 1 << 30, (B, G), device="cuda", dtype=torch.int64, generator=g)
bm = rnd & 0x7F
words = (bm | (bm << 8) | (bm << 16)).contiguous()
del rnd, bm
prof = torch.randint(0, 6, (B,), device="cuda", dtype=torch.uint8, generator=g)
out = torch.empty(B * 2, device="cuda", dtype=torch.int64)
cfg = decisions._sched_cfg(SchedulerConfig(threshold=thr))
for _ in range(2):
    L.msg_score_device(eng._h, B, G, words.data_ptr(), prof.data_ptr(), C.byref(cfg), out.data_ptr())
eng.sync()
print("done", thr)
