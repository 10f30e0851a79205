set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_decisions.py -q -x 2>&1 | tail -2
python tools/quick_bench.py 2>&1 | grep kernel
