set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/hbm_read.py 2>&1 | tail -6
timeout 900 python tools/c4_shards.py 20000 1 2 4 8 16 2>&1 | tail -6
timeout 600 python tools/c4_run.py 20000 300 2>&1 | tail -1
