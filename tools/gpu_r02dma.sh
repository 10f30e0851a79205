D=gpurun_out/${TAG:-r02dma}; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pipelin" > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 900 python tools/e2e_variant_bench.py > $D/e2e_variants.log 2>&1; echo "e2e var rc=$?" >> $D/rc.txt
MSG_ZC_DMA=0 timeout 300 python tools/e2e_variant_bench.py > $D/e2e_variants_nodma.log 2>&1; echo "e2e nodma rc=$?" >> $D/rc.txt
MSG_PROFILE=1 timeout 300 python tools/e2e_zc.py > $D/e2e_zc.log 2>&1; echo "zc rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -2 $D/tests.log; cat $D/e2e_variants.log $D/e2e_variants_nodma.log; grep -B12 "call 3:" $D/e2e_zc.log | grep "zero-copy kernel\|call 3:" | head -8
