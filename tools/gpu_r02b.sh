# scorer rewrite check + sanitizer re-run + reference suites + new bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_decisions.py tests/test_gpu_oracle_suite.py tests/test_gpu_dropin.py tests/test_gpu_goldens.py -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r02b_tests.log
timeout 300 python tools/score_sweep.py > gpurun_out/r02b_sweep.log 2>&1
mkdir -p gpurun_out/sanitize2
for c in sim snapshot cluster; do timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize.py $c > gpurun_out/sanitize2/initcheck_$c.log 2>&1; echo "initcheck $c rc=$?" >> gpurun_out/sanitize2/summary.txt; done
for t in memcheck racecheck synccheck initcheck; do timeout 900 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 20 python tools/sanitize.py score > gpurun_out/sanitize2/${t}_score.log 2>&1; echo "$t score rc=$?" >> gpurun_out/sanitize2/summary.txt; done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
tail -5 gpurun_out/r02b_tests.log; cat gpurun_out/r02b_sweep.log; cat gpurun_out/sanitize2/summary.txt; tail -c 3000 gpurun_out/r02b_bench.json; tail -5 gpurun_out/r02b_bench.err
