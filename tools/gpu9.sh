set -x
python -m pytest tests/test_gpu_decisions.py -q -x 2>&1 | tail -3
python tools/score_bench.py 2>&1 | tail -1
python tools/e2e_profile.py 2>&1 | tail -12
ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 1 -c 1 -o gpurun_out/prof_score_v3 python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -1 gpurun_out/ncu_score.log
