# scorer v2 (table + pass bit) and fused advance: correctness + timing + ncu of both kernels
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_decisions.py tests/test_gpu_oracle_suite.py tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_gpu_goldens.py -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r02c_tests.log
timeout 300 python tools/score_sweep.py > gpurun_out/r02c_sweep.log 2>&1
timeout 300 python tools/quick_bench.py > gpurun_out/r02c_qb.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:score_tma_kernel -c 1 -o gpurun_out/prof_score_r02c python tools/score_bench.py > gpurun_out/r02c_ncu_score.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:sim_kernel -s 1 -c 1 -o gpurun_out/prof_sim_r02c python tools/prof_driver.py sim > gpurun_out/r02c_ncu_sim.log 2>&1
tail -5 gpurun_out/r02c_tests.log; cat gpurun_out/r02c_sweep.log gpurun_out/r02c_qb.log; tail -3 gpurun_out/r02c_ncu_score.log gpurun_out/r02c_ncu_sim.log
