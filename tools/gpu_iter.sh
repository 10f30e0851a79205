# iteration check: GPU parity tests + device timing of the C2 event loop
TAG=${1:-iter}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; tail -3 gpurun_out/${TAG}_tests.log
timeout 300 python tools/quick_bench.py > gpurun_out/${TAG}_qb.log 2>&1; cat gpurun_out/${TAG}_qb.log
