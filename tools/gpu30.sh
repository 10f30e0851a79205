set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>gpurun_out/bench.err | tail -1 > gpurun_out/bench_r01_v8.json; cat gpurun_out/bench_r01_v8.json | cut -c1-3000; tail -2 gpurun_out/bench.err
python bench.py --impl reference 2>&1 | tail -1 | cut -c1-400
ncu --set full --clock-control none --import-source on -k regex:score_tma -s 1 -c 1 -o gpurun_out/prof_score_v12 python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -1 gpurun_out/ncu_score.log
MSG_SHARDS=16 ncu --set full --clock-control none --import-source on -k regex:cluster_kernel -c 1 -o gpurun_out/prof_c4_s16c python tools/prof_c4.py 3000 > gpurun_out/ncu_c4.log 2>&1; tail -1 gpurun_out/ncu_c4.log
