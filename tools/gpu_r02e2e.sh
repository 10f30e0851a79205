D=gpurun_out/r02e2e; mkdir -p $D
timeout 300 python tools/e2e_benchloop.py > $D/loop_plain.log 2>&1
WITH_TORCH=1 timeout 300 python tools/e2e_benchloop.py > $D/loop_torch.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-configs --no-c4 --no-c1 --no-sweep > $D/bench.json 2> $D/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-configs --no-c4 --no-c1 --no-sweep > $D/bench2.json 2> $D/bench2.err
cat $D/loop_plain.log $D/loop_torch.log; for f in bench bench2; do python -c "
import json; d=json.loads(open('$D/$f.json').read().strip().splitlines()[-1]); print({k:d['e2e'][k] for k in ('ms_per_step','ms_median','ms_min','ms_max')})"; done
