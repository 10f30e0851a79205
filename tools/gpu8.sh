set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py 2>gpurun_out/bench.err | tail -1 > gpurun_out/bench_r01_v6.json; cat gpurun_out/bench_r01_v6.json; tail -3 gpurun_out/bench.err
python bench.py --impl reference 2>&1 | tail -1
timeout 900 python tools/c4_run.py 1000000 0 2>&1 | tail -2
