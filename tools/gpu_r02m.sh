D=gpurun_out/r02m; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pipelin" > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 300 python tools/e2e_zc.py > $D/e2e_zc.log 2>&1; echo "zc rc=$?" >> $D/rc.txt
bash tools/c4_phases.sh > $D/c4_phase_build.log 2>&1 && timeout 300 python tools/c4_phases.py 20000 > $D/c4_phases.log 2>&1; echo "c4ph rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -2 $D/tests.log; grep "call 3:\|call 2:" $D/e2e_zc.log; grep -B12 "call 3:" $D/e2e_zc.log | grep "zero-copy kernel\|call 3:"; cat $D/c4_phases.log
