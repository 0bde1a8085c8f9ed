#!/bin/bash
# ncu evidence for the north-star counters: per config, one
# --set full capture of the solver kernel (2nd solve) and of the estimate
# gather probe, after the same command ran clean without ncu.
#   scripts/ncu_evidence.sh <tag> "<configs>"
tag=$1; cfgs=${2:-"3 5"}
mkdir -p gpurun_out
for c in $cfgs; do
  cmd="python scripts/prof_solve.py --config $c --reps 2 --probe 1"
  $cmd > gpurun_out/${tag}_cfg${c}_plain.log 2>&1 || { echo "plain run failed cfg$c"; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"count_rounds_kernel|est_gather_probe" -s 1 -c 2 \
      -o gpurun_out/${tag}_cfg${c} $cmd > gpurun_out/${tag}_cfg${c}_ncu.log 2>&1
  echo "cfg$c ncu exit $?"
done
