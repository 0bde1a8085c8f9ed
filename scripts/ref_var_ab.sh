#!/bin/bash
# reference-rule solve times (hybrid tail on, the shim's mode) of built variants against the default library
tag=$1; cfgs=$2; shift 2
for c in $cfgs; do
  echo "cfg$c base $(timeout 400 python scripts/tail_time.py --config $c 2>&1 | tail -1 | grep -o "t_solve_ms.*")" | tee -a gpurun_out/${tag}.txt
  for v in "$@"; do
    echo "cfg$c $v $(KC_LIB_PATH=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so timeout 400 python scripts/tail_time.py --config $c 2>&1 | tail -1 | grep -o "t_solve_ms.*")" | tee -a gpurun_out/${tag}.txt
  done
done
