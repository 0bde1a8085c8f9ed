#!/bin/bash
# Builds the single-flag variants of scripts/var_ab.sh tuning runs (3 at a time).
b() { name=$1; shift; python -m paper_2512_00233_b200.build --variant $name "$@" > /tmp/build_$name.log 2>&1 && echo "built $name: $*" || echo "FAILED $name"; }
b t1 -DKC_FLAT_EVAL=0 &
b t2 -DKC_SPEC_BINS=128 &
b t3 -DKC_LIST_MIN_DEG=32 &
wait
b t4 -DKC_LIST_MIN_DEG=128 &
b t5 -DKC_GMAX_WARP=8 -DKC_GMAX_BIG=4 &
b t6 -DKC_GMAX_WARP=32 -DKC_GMAX_BIG=16 &
wait
b t7 -DKC_EST_CACHE=0 &
b t8 -DKC_L2_PREFETCH=0 &
b t9 -DKC_FLAT_NOTIFY=1 &
wait
