D=gpurun_out/${TAG:-r02k1}; mkdir -p $D
timeout 600 python tools/variant_bench.py > $D/variants.log 2>&1; echo "var rc=$?" >> $D/rc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decisions.py -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/variants.log; tail -2 $D/tests.log
