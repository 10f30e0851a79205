set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -m pytest tests -m gpu -q 2>&1 | tail -25
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches.csv
ncu --set full --clock-control none --import-source on -k regex:sim_kernel -s 1 -c 1 -o gpurun_out/prof_sim python tools/prof_driver.py sim > gpurun_out/ncu_sim.log 2>&1; tail -2 gpurun_out/ncu_sim.log
ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 1 -c 1 -o gpurun_out/prof_score python tools/prof_driver.py score > gpurun_out/ncu_score.log 2>&1; tail -2 gpurun_out/ncu_score.log
ls -la gpurun_out
