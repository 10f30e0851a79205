D=gpurun_out/r02nd2; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 600 python tools/variant_bench.py > $D/variants.log 2>&1; echo "var rc=$?" >> $D/rc.txt
timeout 600 python tools/e2e_variant_bench.py > $D/e2e_variants.log 2>&1; echo "e2e rc=$?" >> $D/rc.txt
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize.py sim > $D/racecheck_sim.log 2>&1; echo "racecheck rc=$?" >> $D/rc.txt
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py sim > $D/memcheck_sim.log 2>&1; echo "memcheck rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -n 2 $D/tests.log; cat $D/variants.log $D/e2e_variants.log
