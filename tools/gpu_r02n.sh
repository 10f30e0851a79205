D=gpurun_out/r02n; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pipelin" > $D/tests.log 2>&1; echo "tests rc=$?" >> $D/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $D/bench.json 2> $D/bench.err; echo "bench rc=$?" >> $D/rc.txt
timeout 300 python tools/e2e_zc.py > $D/e2e_zc.log 2>&1; echo "zc rc=$?" >> $D/rc.txt
cat $D/rc.txt; tail -2 $D/tests.log; grep "call 3:\|call 2:" $D/e2e_zc.log; python -c "
import json; d=json.loads(open('$D/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'])"
