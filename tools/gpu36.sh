set -x
python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2>gpurun_out/bench.err | tail -1 > gpurun_out/bench_r01_v9.json; cut -c1-400 gpurun_out/bench_r01_v9.json; tail -2 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v9.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; wc -l gpurun_out/launches_v9.csv
MSG_SHARDS=16 timeout 600 python tools/c4_run.py 1000000 0 2>&1 | tail -1
