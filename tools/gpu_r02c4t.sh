# C4 block engine: threads per CTA at 16 shards x held entries per thread (A/B, same box)
D=gpurun_out/${TAG:-r02c4t}; mkdir -p $D
timeout 900 python tools/c4_variant_bench.py > $D/c4_variants.log 2>&1; echo "c4 rc=$?" >> $D/rc.txt
timeout 900 python tools/c4_variant_bench.py >> $D/c4_variants.log 2>&1; echo "c4b rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/c4_variants.log
