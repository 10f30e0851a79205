set -x
python -m pytest tests/test_gpu_decisions.py -q -x 2>&1 | tail -2
python tools/score_bench.py 2>&1 | tail -1 | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:score python tools/prof_driver.py score 2>&1 | grep -E "score_|gpu__time" | head -12
ncu --set full --clock-control none --import-source on -k regex:score_tma -s 1 -c 1 -o gpurun_out/prof_score_v10 python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -1 gpurun_out/ncu_score.log
python bench.py 2>gpurun_out/bench.err | tail -1 > gpurun_out/bench_r01_v7.json; cat gpurun_out/bench_r01_v7.json; tail -3 gpurun_out/bench.err
