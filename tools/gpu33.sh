set -x
python -m pytest tests/test_gpu_oracle_suite.py tests/test_gpu_parity.py -q -x --durations=3 2>&1 | tail -8
python tools/quick_bench.py 2>&1 | tail -7
