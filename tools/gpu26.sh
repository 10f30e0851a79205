set -x
python -m pytest tests/test_gpu_decisions.py -q -x 2>&1 | tail -2
python tools/score_bench.py 2>&1 | tail -1 | cut -c1-250
python tools/score_bench.py 2>&1 | tail -1 | cut -c1-250
python tools/e2e_profile.py 2>&1 | tail -3
for l in build/variants/libcluster_*.so paper_2512_16099_b200/libmigsched_b200.so; do echo $l; MSG_B200_LIB=$l timeout 300 python tools/c4_shards.py 20000 16 8 2>&1 | tail -2 | cut -c1-160; done
