# zero-copy inputs + warm engine: GPU suite, e2e modes, cold calls, kernel timing
D=gpurun_out/r02g; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 300 python tools/e2e_modes.py > $D/e2e_modes.log 2>&1; echo "modes rc=$?" >> $D/rc.txt
MSG_PROFILE=1 timeout 300 python tools/e2e_cold.py > $D/e2e_cold.log 2>&1; echo "cold rc=$?" >> $D/rc.txt
timeout 300 python tools/quick_bench.py > $D/qb.log 2>&1; echo "qb rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -3 $D/tests.log; cat $D/e2e_modes.log; grep -v "^\[msg\]   chunk" $D/e2e_cold.log | head -40; cat $D/qb.log
