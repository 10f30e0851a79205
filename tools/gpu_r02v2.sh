# verify: racecheck fix, parallel layout fast path, zc first-block variants
D=gpurun_out/r02v2; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 50 python tools/sanitize.py sim > $D/racecheck_sim.log 2>&1; echo "racecheck sim rc=$?" >> $D/rc.txt
timeout 900 python tools/e2e_variant_bench.py > $D/e2e_variants.log 2>&1; echo "e2e var rc=$?" >> $D/rc.txt
MSG_PROFILE=1 timeout 300 python tools/e2e_zc.py > $D/e2e_zc.log 2>&1; echo "zc rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -2 $D/tests.log; tail -2 $D/racecheck_sim.log; cat $D/e2e_variants.log
