# round-2 closing check on HEAD: GPU suite, smoke, bench (both arms), 2-rank bench, launch list
D=gpurun_out/r02final6; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err; echo "bench rc=$?" >> $D/rc.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.json 2> $D/bench_ref.err; echo "ref rc=$?" >> $D/rc.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 2 --one-gpu --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_n2.json 2> $D/bench_n2.err; echo "n2 rc=$?" >> $D/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --c4-arrivals 2000 > $D/ncu_launch.log 2>&1; echo "launches rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -n 2 $D/tests.log; tail -n 1 $D/smoke.log
