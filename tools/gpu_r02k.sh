# fused C4 next-event scan, flush cadence variants, reconfig-count / finish changes: full GPU suite + timings
D=gpurun_out/r02k; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 300 python tools/e2e_zc.py > $D/e2e_zc.log 2>&1; echo "zc rc=$?" >> $D/rc.txt
timeout 300 python tools/quick_bench.py > $D/qb.log 2>&1; echo "qb rc=$?" >> $D/rc.txt
timeout 300 python tools/c4_run.py 20000 0 > $D/c4_20k.log 2>&1; echo "c4 rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -3 $D/tests.log; grep "call 3" $D/e2e_zc.log; grep "zero-copy kernel" $D/e2e_zc.log | tail -12; cat $D/qb.log; cat $D/c4_20k.log
