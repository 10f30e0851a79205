"""bench.py's scorer sweep (thresholds 0.4 / 0.0 / 1.0) for each library
variant under build/variants/ and the in-tree library, same box (development aid)."""
import glob, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import json, sys; sys.path.insert(0, %r)
import bench
from paper_2512_16099_b200.engine import Engine
eng = Engine(0)
peaks, kind = bench.measured_peaks()
d = bench.scorer_sweep(eng, peaks, kind)
print(" | ".join("thr %%s %%.1f us %%.3f" %% (k, v["ms"] * 1e3, v["frac"]) for k, v in d["by_threshold"].items()))
''' % root
for lib in sorted(glob.glob(os.path.join(root, "build/variants/lib_*.so"))) + [os.path.join(root, "paper_2512_16099_b200/libmigsched_b200.so")]:
    env = dict(os.environ, MSG_B200_LIB=lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
