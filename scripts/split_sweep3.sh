#!/bin/bash
tag=${1:-x}; cfgs=${2:-"3 5"}
mkdir -p gpurun_out
run() { KC_LIB_PATH=$1 KC_SPLIT_ROUNDS=$2 KC_SPLIT_MIN=${4:-4096} KC_SPLIT_CACHE=1 timeout 300 python scripts/split_ab.py --config $3 2>&1 | tail -1 | tee -a gpurun_out/${tag}.txt; }
for c in $cfgs; do
  run "" 0 $c
  for v in x1 x2 x3 x4; do for sr in 0 24; do run $PWD/paper_2512_00233_b200/libkcore_b200_$v.so $sr $c; done; done
  for sr in 12 16 20 32; do run $PWD/paper_2512_00233_b200/libkcore_b200_x1.so $sr $c; done
  for sm in 1024 16384 65536; do run $PWD/paper_2512_00233_b200/libkcore_b200_x1.so 24 $c $sm; done
done
