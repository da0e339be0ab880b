#!/bin/bash
# ncu captures of representative kernels (one GPU; never wrap multi-rank runs).
# usage: tools/ncu_run.sh <tag> <op> <dtype> <shapes...>   e.g. r01a tsmm d 8x8 32x32
tag=$1; op=$2; dt=$3; shift 3
for s in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${op} -s 3 -c 1 \
    -o gpurun_out/${tag}_${op}_${dt}_${s} python tools/quick_time.py --ops $op --dtypes $dt --shapes $s --reps 1 \
    > gpurun_out/${tag}_${op}_${dt}_${s}.log 2>&1
  echo "$s rc=$?"
done
