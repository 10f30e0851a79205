timeout 200 python -u tools/e2e_modes.py > gpurun_out/e2e2.log 2>&1; echo "rc=$?" >> gpurun_out/e2e2.log
cat gpurun_out/e2e2.log | tail -60
