for v in ph_head ph_cur; do echo "== $v"; MSG_B200_LIB=build/hv/lib_$v.so timeout 120 python tools/sim_phases.py; done > gpurun_out/ph1.log 2>&1
timeout 300 python tools/e2e_modes.py >> gpurun_out/ph1.log 2>&1
HV_REPS=2 HV_LIBS=build/hv/lib_v0_head.so,build/hv/lib_v2_compact.so,paper_2512_16099_b200/libmigsched_b200.so timeout 300 python tools/hv_bench.py >> gpurun_out/ph1.log 2>&1
cat gpurun_out/ph1.log
