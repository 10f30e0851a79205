# ncu evidence for a bench version: event-loop full capture + the bench's launch list
TAG=${1:-v}
bash tools/gpu_prof_sim.sh $TAG
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_$TAG.log 2>&1
grep -c sim_kernel gpurun_out/launches_$TAG.csv
