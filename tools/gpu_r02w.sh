D=gpurun_out/${TAG:-r02x}; mkdir -p $D
timeout 900 python tools/c4_variant_bench.py 20000 > $D/c4_variants.log 2>&1; echo "c4 rc=$?" >> $D/rc.txt
timeout 900 python -m pytest tests/test_gpu_cluster.py -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
bash tools/c4_phases.sh > $D/c4_phase_build.log 2>&1 && timeout 300 python tools/c4_phases.py 20000 > $D/c4_phases.log 2>&1; echo "c4ph rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/c4_variants.log; tail -2 $D/tests.log; cat $D/c4_phases.log
