D=gpurun_out/${TAG:-r02y}; mkdir -p $D
timeout 900 python tools/c4_variant_bench.py 20000 > $D/c4_variants.log 2>&1; echo "c4 rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/c4_variants.log
