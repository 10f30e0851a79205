#!/bin/bash
# Development aid: block-engine variants (threads per CTA) as separate
# libraries under build/variants/ for A/B timing of C4 on the GPU.
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2512_16099_b200/csrc
mkdir -p build/variants
OBJS=$(ls build/csrc/*.o | grep -v engine_kernels)
for t in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
    -ccbin /usr/bin/g++ -Xcompiler -fPIC -DMSG_CLUSTER_THREADS_NARROW=$t \
    -Ipaper_2512_16099_b200/csrc -Iinclude -c paper_2512_16099_b200/csrc/engine_kernels.cu -o build/variants/ekc_$t.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ \
    -o build/variants/libcluster_$t.so build/variants/ekc_$t.o $OBJS -lpthread
  echo built build/variants/libcluster_$t.so
done
