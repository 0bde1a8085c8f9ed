#!/bin/bash
# Round evidence on one GPU (run under gpurun from the repo root):
#   bench line (no profiler), launch list (ncu, per-launch durations),
#   one full ncu capture of the counting solver kernel, phase times.
# Usage: scripts/profile_round.sh <tag> [config]
tag=${1:-r01}; cfg=${2:-3}
mkdir -p gpurun_out
timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/bench_${tag}_cfg${cfg}.json 2> gpurun_out/bench_${tag}_cfg${cfg}.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${tag}_cfg${cfg}.csv \
  python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:count_rounds -c 1 \
  -o gpurun_out/ncu_${tag}_cfg${cfg} -f python scripts/prof_solve.py --config $cfg --reps 1 > /dev/null 2>&1
timeout 120 python scripts/phase_times.py --config $cfg > gpurun_out/phases_${tag}_cfg${cfg}.txt 2>&1
echo done
