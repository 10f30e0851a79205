set -x
python -m pytest tests/test_gpu_decisions.py -q -x 2>&1 | tail -2
python tools/score_bench.py 2>&1 | tail -1 | cut -c1-250
MSG_SCORE_REG=1 python tools/score_bench.py 2>&1 | tail -1 | cut -c1-250
ncu --set full --clock-control none --import-source on -k regex:score_tma -s 1 -c 1 -o gpurun_out/prof_score_v7 python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -1 gpurun_out/ncu_score.log
