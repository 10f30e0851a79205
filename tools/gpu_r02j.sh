D=gpurun_out/r02j; mkdir -p $D
timeout 300 python tools/e2e_zc.py > $D/e2e_zc.log 2>&1; echo "zc rc=$?" >> $D/rc.txt
timeout 300 python tools/e2e_modes.py > $D/e2e_modes.log 2>&1; echo "modes rc=$?" >> $D/rc.txt
timeout 300 python tools/quick_bench.py > $D/qb.log 2>&1; echo "qb rc=$?" >> $D/rc.txt
cat $D/rc.txt; cat $D/e2e_modes.log; cat $D/qb.log
