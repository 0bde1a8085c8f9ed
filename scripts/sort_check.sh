#!/bin/bash
# Layout tests + one-shot e2e A/B (unsorted vs fused relabel-and-sort) + prep times.
tag=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_degree_cut.py -m gpu -x -q > gpurun_out/${tag}_layout.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_layout.log
tail -5 gpurun_out/${tag}_layout.log
for c in 3 5; do
  timeout 300 python scripts/split_ab.py --config $c --reps 3 2>&1 | tail -1 | tee -a gpurun_out/${tag}_solve.txt
done
CFGS="${CFGS:-3 5}" VARIANTS="base osort" bash scripts/e2e_ab.sh 2>&1 | tee gpurun_out/${tag}_e2e.txt
for c in 3 5; do
for v in base osort; do if [ $v = base ]; then L=""; else L=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so; fi
KC_LIB_PATH=$L timeout 600 python scripts/one_shot.py --config $c --reps 3 2>&1 | tail -2 | sed "s/^/$v cfg$c /" | tee -a gpurun_out/${tag}_oneshot.txt
done; done
