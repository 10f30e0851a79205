#!/bin/bash
# Development aid: build scorer variants (words per thread _ min blocks per
# SM _ chunks per item _ TMA stages _ threads) as separate libraries under build/variants/ for A/B timing on the GPU.
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2512_16099_b200/csrc
mkdir -p build/variants
OBJS=$(ls build/csrc/*.o | grep -v score.cu.o)
for v in "$@"; do
  IFS=_ read -r wpt minb item stages thr <<< "$v"; item=${item:-4}; stages=${stages:-4}; thr=${thr:-256}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
    -ccbin /usr/bin/g++ -Xcompiler -fPIC -DMSG_SCORE_WPT=$wpt -DMSG_SCORE_MINB=$minb -DMSG_SCORE_ITEM=$item -DMSG_SCORE_STAGES=$stages -DMSG_SCORE_THREADS=$thr \
    -Ipaper_2512_16099_b200/csrc -Iinclude -c paper_2512_16099_b200/csrc/score.cu -o build/variants/sc_$v.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ \
    -o build/variants/libscore_$v.so build/variants/sc_$v.o $OBJS -lpthread
  echo built build/variants/libscore_$v.so
done
