for c in ${CFGS:-3 4 5 1 2}; do for v in ${VARIANTS:-base osort}; do if [ $v = base ]; then L=""; else L=$PWD/paper_2512_00233_b200/libkcore_b200_$v.so; fi
KC_LIB_PATH=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('$v cfg$c', 'e2e_ms', e['ms_per_step'], e['device_ms'], 'solve', d['ms_per_step'])"
done; done
