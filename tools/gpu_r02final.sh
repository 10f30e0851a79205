# round-2 final check on HEAD: GPU suite, smoke, bench (both arms), 2-rank one-GPU bench, launch list, ncu, e2e, sanitizers
D=gpurun_out/r02final; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err; echo "bench rc=$?" >> $D/rc.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.json 2> $D/bench_ref.err; echo "ref rc=$?" >> $D/rc.txt
timeout 300 python tools/e2e_benchloop.py > $D/benchloop.log 2>&1; echo "loop rc=$?" >> $D/rc.txt
MSG_PROFILE=1 timeout 300 python tools/e2e_cold.py > $D/e2e_cold.log 2>&1; echo "cold rc=$?" >> $D/rc.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --one-gpu --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_n2.json 2> $D/bench_n2.err; echo "n2 rc=$?" >> $D/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --c4-arrivals 2000 > $D/launches_bench.log 2>&1; echo "launches rc=$?" >> $D/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -s 1 -c 1 -o $D/prof_sim python tools/prof_driver.py sim > $D/ncu_sim.log 2>&1; echo "ncu sim rc=$?" >> $D/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cluster_kernel -c 1 -o $D/prof_c4 python tools/prof_c4.py 2000 > $D/ncu_c4.log 2>&1; echo "ncu c4 rc=$?" >> $D/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 2 -o $D/prof_score_t00 python tools/prof_score_thr.py 0.0 > $D/ncu_score_t00.log 2>&1; echo "ncu score0 rc=$?" >> $D/rc.txt
rm -rf gpurun_out/sanitize; bash tools/gpu_sanitize.sh > /dev/null 2>&1; cp -r gpurun_out/sanitize $D/sanitize; echo "sanitize done" >> $D/rc.txt
cat $D/rc.txt; tail -3 $D/tests.log; tail -2 $D/smoke.log; tail -c 300 $D/bench.json; tail -c 300 $D/bench_ref.json; cat $D/benchloop.log; grep rc= $D/sanitize/summary.txt
