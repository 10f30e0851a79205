set -x
python -m pytest tests/test_gpu_decisions.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
python tools/score_bench.py 2>&1 | tail -1 | cut -c1-250
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:score python tools/prof_driver.py score 2>&1 | grep -E "score_|gpu__time" | head -6
python tools/e2e_profile.py 2>&1 | tail -12
