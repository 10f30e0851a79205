"""Scorer sweep variants (development aid): bench.py's scorer_sweep at
thresholds 0.4 / 0.0 / 1.0, plus the same words carrying random idle-exact
bits (the reuse path) and a few draining words (the per-start path)."""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402

from paper_2512_16099_b200 import decisions  # noqa: E402
from paper_2512_16099_b200.engine import Engine  # noqa: E402
from paper_2512_16099_b200.model import SchedulerConfig  # noqa: E402

eng = Engine(0)
peaks, kind = bench.measured_peaks()
print(json.dumps(bench.scorer_sweep(eng, peaks, kind)["by_threshold"]))
torch.cuda.empty_cache()
L = decisions._bind()
B, G = 4096, 16384
gen = torch.Generator(device="cuda").manual_seed(2)
rnd = torch.randint(0, 1 << 62, (B, G), device="cuda", dtype=torch.int64, generator=gen)
bm = rnd & 0x7F
idle = ((rnd >> 8) & 0x3FFFF) * ((rnd >> 30) & 3 == 0)  # a quarter of the words carry idle-exact bits
drain = ((rnd >> 40) & 0x7F) * ((rnd >> 50) & 1023 == 0)  # ~0.1% of the words have a draining instance
drain1 = ((rnd >> 40) & 0x7F) * ((rnd >> 50) & 127 == 0)  # ~0.8%
for name, w in (("idle_exact", bm | (bm << 8) | (bm << 16) | (idle << 24)),
                ("draining_0.1pct", bm | (bm << 8) | ((bm | drain) << 16)),
                ("draining_1pct", bm | (bm << 8) | ((bm | drain1) << 16))):
    bufs = (w.contiguous(), w.contiguous().clone())  # read alternately, as bench.py does (4x L2 each)
    del w
    prof = torch.randint(0, 6, (B,), device="cuda", dtype=torch.uint8, generator=gen)
    out = torch.empty(B * 2, device="cuda", dtype=torch.int64)
    cfg = decisions._sched_cfg(SchedulerConfig())
    ms = C.c_float()
    t = []
    for i in range(12):
        assert L.msg_time_score_device(eng._h, B, G, bufs[i & 1].data_ptr(), prof.data_ptr(), C.byref(cfg),
                                       out.data_ptr(), C.byref(ms)) == 0
        if i >= 4:
            t.append(ms.value)
    del bufs
    m = statistics.median(t)
    gbs = (B * G * 8 + B * 17) / (m * 1e-3) / 1e9
    print(json.dumps({"variant": name, "ms": m, "GBs": gbs, "frac": gbs / peaks["hbm_gbs"]}))
