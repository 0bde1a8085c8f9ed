#!/bin/bash
# Launch list (ncu gpu__time_duration) of one kc_fastk_run on a config; summarised per kernel.
tag=${1:-x}; cfg=${2:-3}; lib=${3:+$(realpath $3)}
mkdir -p gpurun_out
KC_LIB_PATH=$lib timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${tag}_launches_cfg${cfg}.csv python scripts/one_shot.py --config $cfg --reps 1 > gpurun_out/${tag}_launches_cfg${cfg}.log 2>&1
python - <<PY
import csv, collections, re
rows = list(csv.reader(l for l in open("gpurun_out/${tag}_launches_cfg${cfg}.csv") if l.startswith('"')))
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    v = float(r[vi].replace(",", "")); u = r[ui]
    v = v / 1e3 if u in ("ns", "nsecond") else v if u in ("us", "usecond") else v * 1e3 if u in ("ms", "msecond") else v
    k = re.sub(r"\(.*", "", r[ki])[:110]
    a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += v
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{t:12.1f} us  x{c:<5d} {k}")
PY
