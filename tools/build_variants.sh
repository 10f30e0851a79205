#!/bin/bash
# Development aid: build engine-kernel variants (warps/block, min blocks/SM)
# as separate libraries under build/variants/ for A/B timing on the GPU.
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2512_16099_b200/csrc
mkdir -p build/variants
OBJS=$(ls build/csrc/*.o | grep -v engine_kernels)
for v in "$@"; do
  wpb=${v%_*}; minb=${v#*_}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
    -ccbin /usr/bin/g++ -Xcompiler -fPIC -DMSG_SIM_WPB=$wpb -DMSG_SIM_MINB=$minb \
    -Ipaper_2512_16099_b200/csrc -Iinclude -c paper_2512_16099_b200/csrc/engine_kernels.cu -o build/variants/ek_$v.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ \
    -o build/variants/lib_$v.so build/variants/ek_$v.o $OBJS -lpthread
  echo built build/variants/lib_$v.so
done
