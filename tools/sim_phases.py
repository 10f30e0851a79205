"""Cycles per event-loop phase (development aid): needs a library built with
-DMSG_SIM_PHASES (tools/hv_build.sh FLAGS), selected with MSG_B200_LIB.
Runs C1 (one trace alone: the latency floor) and C2 (4096 traces)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16099_b200 import engine as E  # noqa: E402
from paper_2512_16099_b200.engine import Engine, generate_batch  # noqa: E402
from paper_2512_16099_b200.model import SimConfig, WorkloadSpec, SchedulerConfig, preset  # noqa: E402

eng = Engine(0)
lib = E.lib()
buf = (ctypes.c_ulonglong * 8)()
names = ["timer scan+advance", "arrival", "service start", "departure", "sample"]
c5 = WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, profile_mix=(0.5, 0.3, 0.2, 0.0))
for name, spec, cfg, T in (("C1", preset("normal25"), SimConfig(gpu_count=8), 1),
                           ("C2", preset("normal25"), SimConfig(gpu_count=8), 4096),
                           ("C5", c5, SimConfig(gpu_count=8, sched=SchedulerConfig(threshold=0.3),
                                                migration_overlap_s=0.5, reconfig_latency_s=0.1), 4096)):
    b = generate_batch(spec, 0, T)
    st = eng.stage(b, [cfg], 0)
    st.launch(); eng.sync(); st.collect()
    lib.msg_debug_sim_phases(buf, 1)
    ms = st.time_launch()
    lib.msg_debug_sim_phases(buf, 1)
    ev = st.handler_events
    tot = sum(buf[:5])
    print(f"{name}: kernel {ms*1e3:.0f} us, {ev} events, {tot/ev:.0f} cycles/event per warp: " +
          ", ".join(f"{n} {buf[k]/ev:.0f} ({100*buf[k]/tot:.0f}%)" for k, n in enumerate(names)))
