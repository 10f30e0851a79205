D=gpurun_out/r02sc6; mkdir -p $D
timeout 600 python tools/score_variant_bench.py > $D/score_variants.log 2>&1; echo "sv rc=$?" >> $D/rc.txt
MSG_B200_LIB=$PWD/build/variants/lib_lut.so timeout 900 python -m pytest tests/test_gpu_decisions.py tests/test_gpu_oracle_suite.py -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/score_variants.log; tail -n 2 $D/tests.log
