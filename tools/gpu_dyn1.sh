HV_REPS=1 HV_LIBS=build/hv/lib_v0_head.so,paper_2512_16099_b200/libmigsched_b200.so HV_ENVS=";MSG_SIM_DYN=28;MSG_SIM_DYN=24;MSG_SIM_DYN=20;MSG_SIM_DYN=16;MSG_SIM_DYN=14" timeout 600 python tools/hv_bench.py > gpurun_out/dyn1.log 2>&1
for d in "" 28 20 14; do echo "== DYN=$d"; MSG_SIM_DYN=$d MSG_B200_LIB=build/hv/lib_tt_v4_dyn.so timeout 120 python tools/trace_times.py 2>&1 | grep -v Warn; done >> gpurun_out/dyn1.log
cat gpurun_out/dyn1.log
