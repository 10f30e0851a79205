#!/bin/bash
# Development aid: build engine-kernel variants from alternative copies of the
# kernel sources.  Each build/hv/<name>/ holds a full copy of csrc/ (edited);
# its engine_kernels.cu is compiled and linked with the product's host
# objects into build/hv/lib_<name>.so (MSG_B200_LIB=... selects it).
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2512_16099_b200/csrc
OBJS=$(ls build/csrc/*.o | grep -v engine_kernels)
for d in build/hv/*/; do
  n=$(basename $d)
  [ -f build/hv/lib_$n.so ] && [ build/hv/lib_$n.so -nt $d/engine_core.cuh ] && continue
  ( /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
    -ccbin /usr/bin/g++ -Xcompiler -fPIC $(cat $d/FLAGS 2>/dev/null) -I$d -Iinclude -c $d/engine_kernels.cu -o $d/ek.o && \
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ \
    -o build/hv/lib_$n.so $d/ek.o $OBJS -lpthread && echo built build/hv/lib_$n.so ) &
done
wait
