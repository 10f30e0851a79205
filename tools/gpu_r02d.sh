# round-2 re-entry: full GPU suite, smoke, bench (both arms), 2-rank one-GPU bench, launch list, ncu of both kernels
mkdir -p gpurun_out/r02d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02d/smi.txt
lscpu > gpurun_out/r02d/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02d/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02d/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02d/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02d/bench.json 2> gpurun_out/r02d/bench.err; echo "bench rc=$?" >> gpurun_out/r02d/rc.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02d/bench_ref.json 2> gpurun_out/r02d/bench_ref.err; echo "ref rc=$?" >> gpurun_out/r02d/rc.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --one-gpu --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02d/bench_n2.json 2> gpurun_out/r02d/bench_n2.err; echo "n2 rc=$?" >> gpurun_out/r02d/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02d/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --c4-arrivals 2000 > gpurun_out/r02d/launches_bench.log 2>&1; echo "launches rc=$?" >> gpurun_out/r02d/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_tma_kernel -c 1 -o gpurun_out/r02d/prof_score python tools/score_bench.py > gpurun_out/r02d/ncu_score.log 2>&1; echo "ncu score rc=$?" >> gpurun_out/r02d/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -s 1 -c 1 -o gpurun_out/r02d/prof_sim python tools/prof_driver.py sim > gpurun_out/r02d/ncu_sim.log 2>&1; echo "ncu sim rc=$?" >> gpurun_out/r02d/rc.txt
cat gpurun_out/r02d/rc.txt; tail -3 gpurun_out/r02d/tests.log; tail -2 gpurun_out/r02d/smoke.log; tail -c 600 gpurun_out/r02d/bench.json; tail -c 400 gpurun_out/r02d/bench_ref.json; tail -c 400 gpurun_out/r02d/bench_n2.json; tail -3 gpurun_out/r02d/bench_n2.err
