set -x
python -m pytest tests/test_gpu_decisions.py tests/test_gpu_cluster.py -q -x 2>&1 | tail -2
python tools/score_bench.py 2>&1 | tail -1 | cut -c1-200
timeout 600 python tools/c4_shards.py 5000 1 16 8x2 4x4 16x2 2x4 1x4 2>&1 | tail -7
timeout 600 python tools/c4_shards.py 20000 16 16x2 8x4 2>&1 | tail -3
