#!/bin/bash
# Development aid: build the product library of git ref $1 as
# build/variants/lib_$2.so (a worktree under /tmp), for same-box A/B timing
# with tools/variant_bench.py.
set -e
cd "$(dirname "$0")/.."
ROOT=$(pwd)
WT=/tmp/wt_$2
rm -rf $WT; git worktree prune
git worktree add -f $WT $1 >/dev/null
make -s -j8 -C $WT/paper_2512_16099_b200/csrc 2>&1 | grep -v "spill\|^ptxas" || true
mkdir -p build/variants
cp $WT/paper_2512_16099_b200/libmigsched_b200.so build/variants/lib_$2.so
git worktree remove --force $WT
echo built build/variants/lib_$2.so
