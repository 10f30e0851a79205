D=gpurun_out/r02l; mkdir -p $D
timeout 300 python tools/e2e_zc.py > $D/e2e_zc.log 2>&1; echo "zc rc=$?" >> $D/rc.txt
cat $D/rc.txt; grep "call 3\|call 2" $D/e2e_zc.log; grep "zero-copy kernel\|^---" $D/e2e_zc.log | grep -A1 "call 3" | grep kernel
