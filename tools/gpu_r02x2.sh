D=gpurun_out/${TAG:-r02x2}; mkdir -p $D
timeout 900 python tools/c4_variant_bench.py 20000 > $D/c4_variants.log 2>&1; echo "c4 rc=$?" >> $D/rc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "zero_copy_ragged or pipelin" > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/c4_variants.log; tail -2 $D/tests.log
