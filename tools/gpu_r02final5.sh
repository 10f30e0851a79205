# round-2 last full check on HEAD (key-only scorer): GPU suite, smoke, bench (both arms), 2-rank bench, launch list, scorer ncu
D=gpurun_out/r02final5; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err; echo "bench rc=$?" >> $D/rc.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.json 2> $D/bench_ref.err; echo "ref rc=$?" >> $D/rc.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --one-gpu --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_n2.json 2> $D/bench_n2.err; echo "n2 rc=$?" >> $D/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --c4-arrivals 2000 > $D/ncu_launch.log 2>&1; echo "launches rc=$?" >> $D/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 1 -c 1 -o $D/prof_score_t00 python tools/prof_score_thr.py 0.0 > $D/ncu_score_t00.log 2>&1; echo "ncu t00 rc=$?" >> $D/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 1 -c 1 -o $D/prof_score_t04 python tools/prof_score_thr.py 0.4 > $D/ncu_score_t04.log 2>&1; echo "ncu t04 rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -n 2 $D/tests.log; tail -n 1 $D/smoke.log
