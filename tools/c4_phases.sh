#!/bin/bash
# Development aid: the block engine with per-phase cycle counters
# (-DMSG_PHASE_PROF, cluster_core.cuh) as build/variants/libphase.so;
# tools/c4_phases.py reads them after a C4 prefix.
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2512_16099_b200/csrc
mkdir -p build/variants
OBJS=$(ls build/csrc/*.o | grep -v engine_kernels)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
  -ccbin /usr/bin/g++ -Xcompiler -fPIC -DMSG_PHASE_PROF $EXTRA \
  -Ipaper_2512_16099_b200/csrc -Iinclude -c paper_2512_16099_b200/csrc/engine_kernels.cu -o build/variants/ek_phase.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ \
  -o build/variants/libphase.so build/variants/ek_phase.o $OBJS -lpthread
echo built build/variants/libphase.so
