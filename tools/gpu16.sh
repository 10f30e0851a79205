set -x
python -m pytest tests/test_gpu_decisions.py tests/test_gpu_cluster.py -q -x 2>&1 | tail -2
for l in build/variants/libscore_*.so; do echo $l; MSG_B200_LIB=$l python tools/score_bench.py 2>&1 | tail -1 | cut -c1-200; done
MSG_SCORE_REG=1 python tools/score_bench.py 2>&1 | tail -1 | cut -c1-200
timeout 900 python tools/c4_shards.py 20000 1 16 2>&1 | tail -2
ncu --set full --clock-control none --import-source on -k regex:score_tma -s 1 -c 1 -o gpurun_out/prof_score_v8 python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -1 gpurun_out/ncu_score.log
