set -x
python -m pytest tests/test_gpu_decisions.py -q -x 2>&1 | tail -2
for l in build/variants/libscore_*.so paper_2512_16099_b200/libmigsched_b200.so; do echo $l; MSG_B200_LIB=$l python tools/score_bench.py 2>&1 | tail -1 | cut -c1-200; done
ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 1 -c 1 -o gpurun_out/prof_score_v6 python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -1 gpurun_out/ncu_score.log
