#!/bin/bash
# Development aid: the product library with score.cu built with extra nvcc
# flags ($2...), as build/variants/lib_$1.so (A/B timing of the scorer).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
make -s -C paper_2512_16099_b200/csrc 2>&1 | grep -v "spill\|^ptxas" || true
mkdir -p build/variants
OBJS=$(ls build/csrc/*.o | grep -v score.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
  -ccbin /usr/bin/g++ -Xcompiler -fPIC "$@" \
  -Ipaper_2512_16099_b200/csrc -Iinclude -c paper_2512_16099_b200/csrc/score.cu -o build/variants/sc_$name.o 2>&1 | grep -v "spill\|^ptxas" || true
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ \
  -o build/variants/lib_$name.so build/variants/sc_$name.o $OBJS -lpthread
echo built build/variants/lib_$name.so
