# GPU tests + bench (our arm) for host-side changes
TAG=${1:-e2e}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; tail -1 gpurun_out/${TAG}_tests.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-c4 --no-configs --no-sweep > gpurun_out/${TAG}_bench$i.json 2>/dev/null; python -c "import json;b=json.load(open('gpurun_out/${TAG}_bench$i.json'));print(b['ms_per_step'],b['e2e']['ms_per_step'],b['e2e']['value'])"; done
