set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3
python tools/variant_bench.py 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --set full --clock-control none --import-source on -k regex:sim_kernel -s 1 -c 1 -o gpurun_out/prof_sim python tools/prof_driver.py sim > gpurun_out/ncu_sim.log 2>&1; tail -1 gpurun_out/ncu_sim.log
ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 1 -c 1 -o gpurun_out/prof_score python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -1 gpurun_out/ncu_score.log
