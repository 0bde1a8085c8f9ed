#!/bin/bash
# A/B sweep printing one "variant config t_solve_ms" line per run (3 reps, last shown).
# Usage: scripts/ab_table.sh "<configs>" <variant>...
cfgs=$1; shift
for c in $cfgs; do
  for v in "$@"; do
    if [ "$v" = "base" ]; then lib=""; else lib=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so; fi
    t=$(KC_LIB_PATH=$lib timeout 150 python scripts/prof_solve.py --config $c --reps 3 2>&1 | tail -1 | sed -n "s/.*'t_solve_ms': \([0-9.]*\).*/\1/p")
    echo "$v cfg$c $t"
  done
done
