#!/bin/bash
# Reference-rule counter-deviation hunt across build variants (DESIGN §3.2 open
# item): default, no degree cuts (KC_SOLVE_DCUT=0), no shared-memory estimate
# cache (KC_SOLVE_CACHE_MIN=UINT_MAX).  Each variant: P processes x R solves of
# R-MAT 26 alternating hybrid_tail off/on (scripts/ref_diverge.py).
# Usage: scripts/ref_diverge_variants.sh [P] [R]
P=${1:-2}; R=${2:-500}
mkdir -p gpurun_out
for v in default nodcut nocache; do
  L=""; [ "$v" != default ] && L=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so
  for i in $(seq 1 $P); do
    KC_LIB_PATH=$L timeout 900 python scripts/ref_diverge.py --config 5 --reps $R >> gpurun_out/diverge_$v.txt 2>&1
  done
done
echo ALLDONE
