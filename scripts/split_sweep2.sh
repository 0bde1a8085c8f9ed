#!/bin/bash
# Second sweep: the persistent kernel's own shape (w1, w2, w5, w6: split off and on), split variants w3, w4.
tag=${1:-x}; cfgs=${2:-"3 5"}
mkdir -p gpurun_out
run() { KC_LIB_PATH=$1 KC_SPLIT_ROUNDS=$2 KC_SPLIT_CACHE=1 timeout 300 python scripts/split_ab.py --config $3 2>&1 | tail -1 | tee -a gpurun_out/${tag}.txt; }
for c in $cfgs; do
  run "" 0 $c
  run $PWD/paper_2512_00233_b200/libkcore_b200_v7.so 24 $c
  run $PWD/paper_2512_00233_b200/libkcore_b200_v7.so 64 $c
  for v in w1 w2 w5 w6; do for sr in 0 24; do run $PWD/paper_2512_00233_b200/libkcore_b200_$v.so $sr $c; done; done
  for v in w3 w4; do run $PWD/paper_2512_00233_b200/libkcore_b200_$v.so 24 $c; done
done
