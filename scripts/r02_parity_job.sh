bash scripts/debug_bounds.sh r02_bounds
for c in 4 5; do timeout 900 python scripts/stress_counting.py --config $c --solves 200 > gpurun_out/r02_stress_counting_cfg$c.txt 2>&1; echo "exit $?" >> gpurun_out/r02_stress_counting_cfg$c.txt; done
timeout 900 python scripts/stress_counting.py --config 5 --solves 50 --rule 0 > gpurun_out/r02_stress_reference_cfg5.txt 2>&1; echo "exit $?" >> gpurun_out/r02_stress_reference_cfg5.txt
tail -3 gpurun_out/r02_stress_*.txt
