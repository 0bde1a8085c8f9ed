#!/bin/bash
# scripts/split_ab.sh <tag> "<configs>" <variant>...   (under gpurun)
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
for c in $cfgs; do
  KC_SPLIT_ROUNDS=0 timeout 300 python scripts/split_ab.py --config $c 2>&1 | tail -1 | tee -a gpurun_out/${tag}.txt
  for v in "$@"; do
    if [ "$v" = "base" ]; then lib=""; else lib=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so; fi
    for sc in 1 0; do
      KC_LIB_PATH=$lib KC_SPLIT_ROUNDS=${SPLIT_ROUNDS:-24} KC_SPLIT_CACHE=$sc timeout 300 python scripts/split_ab.py --config $c 2>&1 | tail -1 | tee -a gpurun_out/${tag}.txt
    done
  done
done
