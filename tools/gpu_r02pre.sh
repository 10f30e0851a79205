D=gpurun_out/r02pre; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 900 python tools/e2e_variant_bench.py > $D/e2e_variants.log 2>&1; echo "e2e rc=$?" >> $D/rc.txt
MSG_PROFILE=1 timeout 300 python tools/e2e_zc.py > $D/e2e_zc.log 2>&1
cat $D/rc.txt; tail -n 1 $D/tests.log; cat $D/e2e_variants.log; grep -A8 "zc + prog rows call 5" $D/e2e_zc.log
