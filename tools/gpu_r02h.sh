# progressive rows + zero copy: pipelined tests, e2e modes, kernel timing
D=gpurun_out/${TAG:-r02i}; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pipelin" > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 300 python tools/e2e_modes.py > $D/e2e_modes.log 2>&1; echo "modes rc=$?" >> $D/rc.txt
MSG_PROFILE=1 timeout 300 python tools/e2e_cold.py > $D/e2e_cold.log 2>&1; echo "cold rc=$?" >> $D/rc.txt
timeout 300 python tools/quick_bench.py > $D/qb.log 2>&1; echo "qb rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -3 $D/tests.log; cat $D/e2e_modes.log; grep -v "^\[msg\]   chunk" $D/e2e_cold.log | head -30; cat $D/qb.log
