D=gpurun_out/${TAG:-r02pf}; mkdir -p $D
timeout 900 python tools/e2e_variant_bench.py > $D/e2e_variants.log 2>&1; echo "e2e var rc=$?" >> $D/rc.txt
MSG_B200_LIB=$PWD/build/variants/lib_zcpf.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "zero_copy_ragged or pipelin" > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/e2e_variants.log; tail -2 $D/tests.log
