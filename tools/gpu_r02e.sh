# round 2: compute-sanitizer over every kernel family (logs -> gpurun_out/sanitize/), then e2e host-phase profile
rm -rf gpurun_out/sanitize; bash tools/gpu_sanitize.sh
MSG_PROFILE=1 timeout 300 python tools/e2e_profile.py > gpurun_out/r02e_e2e_profile.log 2>&1
timeout 300 python tools/e2e_cold.py > gpurun_out/r02e_e2e_cold.log 2>&1
grep rc= gpurun_out/sanitize/summary.txt; tail -30 gpurun_out/r02e_e2e_profile.log; tail gpurun_out/r02e_e2e_cold.log
