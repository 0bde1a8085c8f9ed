#!/bin/bash
# A/B of the per-phase-kernel variants built by scripts/split_sweep_build.sh.
tag=${1:-x}; cfgs=${2:-"3 5"}
mkdir -p gpurun_out
for c in $cfgs; do
  KC_SPLIT_ROUNDS=0 timeout 300 python scripts/split_ab.py --config $c 2>&1 | tail -1 | tee -a gpurun_out/${tag}.txt
  for v in v1 v2 v3 v4 v5 v6 v7 v8 v9 v10; do
    lib=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so
    for sc in 1 0; do
      KC_LIB_PATH=$lib KC_SPLIT_ROUNDS=${SPLIT_ROUNDS:-24} KC_SPLIT_CACHE=$sc timeout 300 python scripts/split_ab.py --config $c 2>&1 | tail -1 | tee -a gpurun_out/${tag}.txt
    done
  done
done
