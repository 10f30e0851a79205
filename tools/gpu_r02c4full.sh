D=gpurun_out/r02c4full; mkdir -p $D
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs --no-c1 --no-sweep --c4-arrivals 1000000 > $D/bench_c4full.json 2> $D/bench_c4full.err; echo "c4full rc=$?" >> $D/rc.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --one-gpu --steps 5 --warmup 3 --no-cpu-baseline --no-c4 > $D/bench_n2.json 2> $D/bench_n2.err; echo "n2 rc=$?" >> $D/rc.txt
cat $D/rc.txt; python -c "
import json
d=json.loads(open('$D/bench_c4full.json').read().strip().splitlines()[-1]); print(json.dumps(d['c4'])[:900])
d=json.loads(open('$D/bench_n2.json').read().strip().splitlines()[-1]); print(d['value'], d['weak'])"
