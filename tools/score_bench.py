"""Scorer sweep alone (development aid): bench.py's scorer_sweep on cuda:0."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_16099_b200.engine import Engine  # noqa: E402
eng = Engine(0)
peaks, kind = bench.measured_peaks()
print(json.dumps(bench.scorer_sweep(eng, peaks, kind)))
