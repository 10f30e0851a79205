D=gpurun_out/${TAG:-r02sc5}; mkdir -p $D
timeout 600 python tools/score_variant_bench.py > $D/score_variants.log 2>&1; echo "sv rc=$?" >> $D/rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
for tool in memcheck racecheck synccheck initcheck; do timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize.py score > $D/${tool}_score.log 2>&1; echo "$tool score rc=$?" >> $D/rc.txt; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 2 -o $D/prof_score_t00 python tools/prof_score_thr.py 0.0 > $D/ncu_score_t00.log 2>&1; echo "ncu rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/score_variants.log; tail -n 2 $D/tests.log
