"""Time the C2 event-loop kernel for each library variant (development aid)."""
import glob, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys; sys.path.insert(0, %r)
from paper_2512_16099_b200.engine import Engine, generate_batch
from paper_2512_16099_b200.model import SimConfig, preset
eng = Engine(0)
out = []
for G, T in ((8, 4096), (4, 4096), (8, 16384)):
    b = generate_batch(preset("normal25"), 0, T)
    st = eng.stage(b, [SimConfig(gpu_count=G)], 0)
    for _ in range(3): st.launch()
    eng.sync(); st.collect()
    ts = []
    for _ in range(5):
        eng.flush_l2(); ts.append(st.time_launch())
    out.append("G%%d T%%d %%.3f ms %%.3e ev/s" %% (G, T, min(ts), st.handler_events / min(ts) * 1e3))
print(" | ".join(out))
''' % root
for lib in sorted(glob.glob(os.path.join(root, "build/variants/lib_*.so"))) + [os.path.join(root, "paper_2512_16099_b200/libmigsched_b200.so")]:
    env = dict(os.environ, MSG_B200_LIB=lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip() or r.stderr.strip()[-300:])
