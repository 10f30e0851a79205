set -x
python -m pytest tests/test_gpu_decisions.py -q -x 2>&1 | tail -1
python bench.py --steps 5 --no-cpu-baseline --no-sweep --no-c4 2>gpurun_out/bench.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['configs'])[:1500]); print(d['value'])"
tail -3 gpurun_out/bench.err
