#!/bin/bash
# Longer stress on the final build: digest-checked back-to-back solves, both layouts.
mkdir -p gpurun_out
for spec in "3 1000 2" "1 2000 2" "2 300 2" "4 300 2" "5 300 2" "3 300 0" "4 100 0"; do
  set -- $spec
  timeout 1500 python scripts/stress_counting.py --config $1 --solves $2 --rule $3 > gpurun_out/r02_stress_final_cfg$1_rule$3.txt 2>&1
  echo "exit $?" >> gpurun_out/r02_stress_final_cfg$1_rule$3.txt
  tail -n 2 gpurun_out/r02_stress_final_cfg$1_rule$3.txt
done
