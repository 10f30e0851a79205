# iteration check + ncu source capture of the event loop
TAG=${1:-iter}
bash tools/gpu_iter.sh $TAG
bash tools/gpu_prof_sim.sh $TAG
