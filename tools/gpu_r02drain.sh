# drain-phase row flushes (MSG_DRAIN_FLUSH) vs none: zero-copy parity tests, e2e A/B
D=gpurun_out/${TAG:-r02drain}; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $D/tests_parity.log 2>&1; echo "parity rc=$?" >> $D/rc.txt
timeout 600 python tools/e2e_variant_bench.py > $D/e2e_variants.log 2>&1; echo "e2e rc=$?" >> $D/rc.txt
timeout 600 python tools/e2e_variant_bench.py >> $D/e2e_variants.log 2>&1; echo "e2e2 rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/e2e_variants.log; tail -n 2 $D/tests_parity.log
