#!/bin/bash
# Reference-rule determinism sweep on R-MAT 26: fresh processes, a few solves
# each, for the default build and (optionally) a variant library.
# Usage: scripts/ref_repeat_multi.sh <processes> [variant]
n=${1:-8}; v=${2:-}
L=""; [ -n "$v" ] && L=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so
for i in $(seq 1 $n); do KC_LIB_PATH=$L timeout 200 python scripts/ref_repeat.py --config 5 --reps 6 ${ALT:+--alternate}; done
