"""Scorer sweep at several load-balancing thresholds (development aid):
threshold 0 sends every snapshot through pass 2."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_16099_b200 import decisions  # noqa: E402
from paper_2512_16099_b200.engine import Engine  # noqa: E402
from paper_2512_16099_b200.model import SchedulerConfig  # noqa: E402
eng = Engine(0)
peaks, kind = bench.measured_peaks()
orig = decisions._sched_cfg
for thr in (0.4, 0.0, 1.0):
    decisions._sched_cfg = lambda cfg, t=thr: orig(SchedulerConfig(threshold=t))
    d = bench.scorer_sweep(eng, peaks, kind)
    print(thr, round(d["ms"] * 1e3, 1), "us", round(d["frac"], 3))
