#!/bin/bash
# Round evidence across the five configs (run under gpurun from the repo root):
# bench line per config (CPU baseline on 1-3), reference-rule timings, phase
# times.  Usage: scripts/sweep.sh <tag>
tag=${1:-s}
mkdir -p gpurun_out
for c in 1 2 3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_${tag}_cfg$c.json 2> gpurun_out/bench_${tag}_cfg$c.err
done
for c in 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${tag}_cfg$c.json 2> gpurun_out/bench_${tag}_cfg$c.err
done
for c in 1 2 3; do
  timeout 300 python scripts/tail_time.py --config $c > gpurun_out/refrule_${tag}_cfg$c.txt 2>&1
done
for c in 2 3; do
  timeout 300 python scripts/phase_times.py --config $c > gpurun_out/phases_${tag}_cfg$c.txt 2>&1
done
echo done
