set -x
python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 900 python tools/c4_shards.py 20000 1 4 8 16 2>&1 | tail -4
MSG_SHARDS=16 ncu --set full --clock-control none --import-source on -k regex:cluster_kernel -c 1 -o gpurun_out/prof_c4_s16b python tools/prof_c4.py 3000 > gpurun_out/ncu_c4.log 2>&1; tail -1 gpurun_out/ncu_c4.log
python tools/e2e_profile.py 2>&1 | tail -6
