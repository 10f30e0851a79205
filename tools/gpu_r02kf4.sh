# scorer on words with idle-exact bits / draining instances: key-only (in tree) vs r02-b consumer (kf0)
D=gpurun_out/${TAG:-r02kf4}; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_decisions.py -x -q -p no:cacheprovider > $D/tests_dec.log 2>&1; echo "dec rc=$?" >> $D/rc.txt
for lib in build/variants/lib_kf0.so paper_2512_16099_b200/libmigsched_b200.so; do echo "== $lib" >> $D/score_sweep.log; MSG_B200_LIB=$lib timeout 600 python tools/score_sweep.py >> $D/score_sweep.log 2>&1; done; echo "sweep rc=$?" >> $D/rc.txt
cat $D/rc.txt $D/score_sweep.log; tail -n 2 $D/tests_dec.log
