set -x
python -m pytest tests/test_gpu_decisions.py -q -x 2>&1 | tail -2
python tools/score_bench.py 2>&1 | tail -1 | cut -c1-250
ncu --set full --clock-control none --import-source on -k regex:score_tma -s 1 -c 1 -o gpurun_out/prof_score_v11 python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -1 gpurun_out/ncu_score.log
python tools/e2e_profile.py 2>&1 | tail -14
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v7.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; wc -l gpurun_out/launches_v7.csv
MSG_SHARDS=16 timeout 600 python tools/c4_run.py 1000000 0 2>&1 | tail -1
