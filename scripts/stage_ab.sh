#!/bin/bash
# pageable one-shot e2e against the staging thread count
mkdir -p gpurun_out; nproc; 
for c in 3 5; do for t in 4 8 12 16 24; do
  echo "cfg$c threads $t"; KC_STAGE_THREADS=$t timeout 600 python scripts/one_shot.py --config $c --reps 4 2>&1 | tail -2
done; done 2>&1 | tee gpurun_out/${1:-x}_stage.txt
