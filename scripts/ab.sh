#!/bin/bash
# A/B timing of library variants on one config: scripts/ab.sh <config> <variant>...
cfg=$1; shift
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=""; else lib=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so; fi
  echo "== $v"; KC_LIB_PATH=$lib timeout 120 python scripts/prof_solve.py --config $cfg --reps 3 2>&1 | tail -2
done
