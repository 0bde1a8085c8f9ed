#!/bin/bash
# One ncu --set full capture of the counting solver's kernel on a config
# (after a plain run of the same command exited 0).  scripts/ncu_full.sh <tag> <config>
tag=$1; cfg=${2:-3}
mkdir -p gpurun_out
cmd="python scripts/prof_solve.py --config $cfg --reps 2"
$cmd > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:count_rounds_kernel -s 1 -c 1 \
    -o gpurun_out/${tag} $cmd > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu exit $?"
