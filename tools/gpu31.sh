set -x
python -m pytest tests/test_gpu_cluster.py -q -x 2>&1 | tail -2
timeout 300 python tools/c4_shards.py 20000 1 16 8x2 2>&1 | tail -3 | cut -c1-300
