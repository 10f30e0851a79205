"""Time a C4 prefix (16384 GPUs, normal25 at ia 25/2048 s, seed 0) with each
library variant under build/variants/ and the in-tree library, same box
(development aid).  usage: python tools/c4_variant_bench.py [arrivals]"""
import glob, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
code = r'''
import sys; sys.path.insert(0, %r)
from paper_2512_16099_b200.engine import Engine, generate_batch
from paper_2512_16099_b200.model import SimConfig, preset
sp = preset("normal25"); sp.mean_interarrival_s = 25.0 / 2048; sp.job_count = %d
eng = Engine(0)
st = eng.stage(generate_batch(sp, 0, 1), [SimConfig(gpu_count=16384)], 0)
ts = [st.time_launch() for _ in range(3)]
r = st.collect()[0]
print("%%.4f s (runs %%s) %%s makespan %%r turn %%r" %% (min(ts) / 1e3, ["%%.4f" %% (t / 1e3) for t in ts], r.code,
      r.workload_makespan_s, r.mean_turnaround_s))
''' % (root, n)
for lib in sorted(glob.glob(os.path.join(root, "build/variants/lib_*.so"))) + [os.path.join(root, "paper_2512_16099_b200/libmigsched_b200.so")]:
    env = dict(os.environ, MSG_B200_LIB=lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
