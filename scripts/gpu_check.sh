#!/bin/bash
# One GPU call: C++ drop-in tests, the GPU suite, and per-round phase times.
#   gpurun -- bash scripts/gpu_check.sh <tag> [configs...]
tag=${1:-x}; shift
cfgs=${@:-3}
mkdir -p gpurun_out
./tests/cpp/test_shim > gpurun_out/${tag}_shim.txt 2>&1; echo "shim rc=$?" >> gpurun_out/${tag}_shim.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log
for c in $cfgs; do
  timeout 300 python scripts/phase_times.py --config $c > gpurun_out/${tag}_phases_cfg$c.txt 2>&1
done
tail -2 gpurun_out/${tag}_shim.txt gpurun_out/${tag}_pytest_gpu.log
