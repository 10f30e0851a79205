"""Per-phase cycle split of the block engine on a C4 prefix (development
aid; needs build/variants/libphase.so from tools/c4_phases.sh)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("MSG_B200_LIB", os.path.join(ROOT, "build/variants/libphase.so"))
sys.path.insert(0, ROOT)
from paper_2512_16099_b200 import engine as E  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, preset  # noqa: E402

jobs = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
sp = preset("normal25")
sp.mean_interarrival_s = 25.0 / 2048
sp.job_count = jobs
eng = Engine(0)
lib = C.CDLL(os.environ["MSG_B200_LIB"])
f = lib.msg_debug_phase
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int, C.c_int]
buf = (C.c_ulonglong * 16)()
b = generate_batch(sp, 0, 1)
st = eng.stage(b, [SimConfig(gpu_count=16384)], 0)
st.launch()
eng.sync()
f(buf, 16, 1)
ms = st.time_launch()
f(buf, 16, 0)
names = ["timer scan", "spec placement search", "exchanges", "advance", "arrival", "departure", "service start",
         "reschedule+sample"]
tot = sum(buf[i] for i in range(8))
ev, xc = buf[9], buf[8]
print(f"kernel {ms:.1f} ms, events {ev}, exchanges {xc} ({xc / max(ev, 1):.2f}/event), "
      f"{ms * 1e3 / max(ev, 1):.2f} us/event")
for i, n in enumerate(names):
    print(f"  {n:24s} {100 * buf[i] / tot:5.1f}%  {buf[i] / max(ev, 1) / 1965:7.3f} us/event")
