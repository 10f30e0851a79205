# key-only scorer with the table-driven start recovery; scorer sweep timed behind a queued L2 flush
D=gpurun_out/${TAG:-r02kf2}; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_decisions.py -x -q -p no:cacheprovider > $D/tests_dec.log 2>&1; echo "dec rc=$?" >> $D/rc.txt
timeout 600 python tools/score_variant_bench.py > $D/score_variants.log 2>&1; echo "sv rc=$?" >> $D/rc.txt
timeout 600 python tools/score_variant_bench.py >> $D/score_variants.log 2>&1; echo "sv2 rc=$?" >> $D/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 2 -o $D/prof_score_t00 python tools/prof_score_thr.py 0.0 > $D/ncu_score_t00.log 2>&1; echo "ncu t00 rc=$?" >> $D/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 2 -o $D/prof_score_t04 python tools/prof_score_thr.py 0.4 > $D/ncu_score_t04.log 2>&1; echo "ncu t04 rc=$?" >> $D/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err; echo "bench rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/score_variants.log; tail -n 2 $D/tests_dec.log
