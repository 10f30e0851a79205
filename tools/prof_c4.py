"""C4 prefix for ncu captures of the (sharded) block engine (development aid).
usage: MSG_SHARDS=S python tools/prof_c4.py [arrivals]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200.engine import Engine, generate_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

jobs = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
sp = preset("normal25")
sp.mean_interarrival_s = 25.0 / 2048
sp.job_count = jobs
eng = Engine(0)
st = eng.stage(generate_batch(sp, 0, 1), [SimConfig(gpu_count=16384)], 0)
ms = st.time_launch()
print(f"{jobs} arrivals: {ms:.1f} ms, {st.collect()[0].code}")
