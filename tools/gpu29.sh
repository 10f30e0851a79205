set -x
python -m pytest tests/test_gpu_decisions.py -q -x 2>&1 | tail -2
for i in 1 2 3; do python tools/score_bench.py 2>&1 | tail -1 | cut -c1-200; done
MSG_SCORE_REG=1 python tools/score_bench.py 2>&1 | tail -1 | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:score python tools/prof_driver.py score 2>&1 | grep -E "score_|gpu__time" | head -6
