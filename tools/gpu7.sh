set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python tools/c4_run.py 20000 300 2>&1 | tail -2
timeout 900 python tools/c4_run.py 1000000 0 2>&1 | tail -2
python bench.py 2>&1 | tail -1 > gpurun_out/bench_v5.json; cat gpurun_out/bench_v5.json
python tools/prof_driver.py score && ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 1 -c 1 -o gpurun_out/prof_score python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -1 gpurun_out/ncu_score.log
