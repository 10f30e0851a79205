HV_REPS=2 timeout 500 python tools/hv_bench.py > gpurun_out/hv2.log 2>&1
cat gpurun_out/hv2.log
