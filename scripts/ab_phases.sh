#!/bin/bash
# A/B of library variants: plain solve time + per-round phase table per config.
# Usage (under gpurun): scripts/ab_phases.sh <tag> "<configs>" <variant>...
tag=$1; cfgs=$2; shift 2
mkdir -p gpurun_out
for c in $cfgs; do
  for v in "$@"; do
    if [ "$v" = "base" ]; then lib=""; else lib=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so; fi
    KC_LIB_PATH=$lib timeout 300 python scripts/phase_times.py --config $c > gpurun_out/${tag}_${v}_cfg$c.txt 2>&1
    echo "$v cfg$c: $(head -1 gpurun_out/${tag}_${v}_cfg$c.txt) | $(tail -1 gpurun_out/${tag}_${v}_cfg$c.txt)"
  done
done
