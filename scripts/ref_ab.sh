# REFERENCE-rule A/B (rounds with and without the hybrid tail) of variant libraries vs the default build.
# Usage: VARIANTS="x base" scripts/ref_ab.sh
for c in 3 5 4 1 2; do for v in ${VARIANTS:-sold base}; do if [ $v = base ]; then L=""; else L=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so; fi
echo "== $v cfg$c"; KC_LIB_PATH=$L timeout 300 python scripts/tail_time.py --config $c 2>&1 | tail -2; done; done
