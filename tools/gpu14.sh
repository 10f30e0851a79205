set -x
./tools/micro/readbw
MSG_SHARDS=16 python tools/prof_c4.py 5000
MSG_SHARDS=16 ncu --set full --clock-control none --import-source on -k regex:cluster_kernel -c 1 -o gpurun_out/prof_c4_s16 python tools/prof_c4.py 3000 > gpurun_out/ncu_c4.log 2>&1; tail -2 gpurun_out/ncu_c4.log
