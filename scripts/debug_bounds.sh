#!/bin/bash
# The GPU suite under the device bounds-check build (KC_DEBUG_BOUNDS=1:
# every queue / list / long-scan-queue / histogram / per-vertex write
# index checked, __trap on violation) — compute-sanitizer is closed on this
# pool.  Build here: python -m paper_2512_00233_b200.build --variant bounds -DKC_DEBUG_BOUNDS=1
# Run (GPU): scripts/debug_bounds.sh <tag>
tag=${1:-bounds}
mkdir -p gpurun_out
KC_LIB_PATH=$PWD/paper_2512_00233_b200/libkcore_b200_bounds.so timeout 1200 \
  python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log
for c in 3 4 5; do
  KC_LIB_PATH=$PWD/paper_2512_00233_b200/libkcore_b200_bounds.so timeout 600 \
    python scripts/stress_counting.py --config $c --solves 3 >> gpurun_out/${tag}_configs.log 2>&1
  echo "cfg$c exit $?" >> gpurun_out/${tag}_configs.log
done
tail -2 gpurun_out/${tag}_pytest_gpu.log; grep -c KC_BOUNDS gpurun_out/${tag}_pytest_gpu.log gpurun_out/${tag}_configs.log
