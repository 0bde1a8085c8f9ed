#!/bin/bash
# pageable one-shot e2e: non-temporal host copy on/off
mkdir -p gpurun_out; grep -m1 "model name" /proc/cpuinfo; grep -m1 -o "avx2" /proc/cpuinfo
for c in 3 5; do for nt in 0 1; do
  echo "cfg$c KC_STAGE_NT=$nt"; KC_STAGE_NT=$nt timeout 600 python scripts/one_shot.py --config $c --reps 4 2>&1 | tail -3
done; done 2>&1 | tee gpurun_out/${1:-x}_stage_nt.txt
