nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/r02a_tests.log
bash tools/gpu_sanitize.sh
tail -5 gpurun_out/r02a_tests.log
cat gpurun_out/sanitize/summary.txt
