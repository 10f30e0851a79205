D=gpurun_out/r02s; mkdir -p $D
timeout 300 python tools/e2e_benchloop.py > $D/benchloop.log 2>&1; echo "loop rc=$?" >> $D/rc.txt
timeout 600 python tools/variant_bench.py > $D/variants.log 2>&1; echo "var rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/benchloop.log $D/variants.log
