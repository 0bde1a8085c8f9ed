#!/bin/bash
# scripts/var_ab.sh <tag> "<configs>" <variant>... : solve-time A/B of built variants against the default library
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
for c in $cfgs; do
  timeout 300 python scripts/split_ab.py --config $c 2>&1 | tail -1 | tee -a gpurun_out/${tag}.txt
  for v in "$@"; do
    KC_LIB_PATH=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so timeout 300 python scripts/split_ab.py --config $c 2>&1 | tail -1 | tee -a gpurun_out/${tag}.txt
  done
done
