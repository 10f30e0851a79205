# key-only scorer (MSG_SCORE_KF) vs the previous key form: decision tests, A/B sweep, GPU suite, ncu (score, sim)
D=gpurun_out/${TAG:-r02kf}; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_decisions.py -x -q -p no:cacheprovider > $D/tests_dec.log 2>&1; echo "dec rc=$?" >> $D/rc.txt
timeout 600 python tools/score_variant_bench.py > $D/score_variants.log 2>&1; echo "sv rc=$?" >> $D/rc.txt
timeout 600 python tools/score_variant_bench.py >> $D/score_variants.log 2>&1; echo "sv2 rc=$?" >> $D/rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 2 -o $D/prof_score_t00 python tools/prof_score_thr.py 0.0 > $D/ncu_score_t00.log 2>&1; echo "ncu t00 rc=$?" >> $D/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 2 -o $D/prof_score_t04 python tools/prof_score_thr.py 0.4 > $D/ncu_score_t04.log 2>&1; echo "ncu t04 rc=$?" >> $D/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -s 1 -c 1 -o $D/prof_sim python tools/prof_driver.py sim > $D/ncu_sim.log 2>&1; echo "ncu sim rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/score_variants.log; tail -n 2 $D/tests_dec.log $D/tests.log
