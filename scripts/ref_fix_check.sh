mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fix_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/fix_pytest_gpu.log
for c in 1 2 3 4 5; do timeout 400 python scripts/tail_time.py --config $c > gpurun_out/fix_refrule_cfg$c.txt 2>&1; done
for i in 1 2 3; do timeout 900 python scripts/ref_diverge.py --config 5 --reps 500 >> gpurun_out/diverge_fixed.txt 2>&1; done
echo ALLDONE
