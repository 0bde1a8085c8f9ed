#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root): GPU suite, smoke, bench
# lines (default = cfg3 + cfg5 inside the same line, then every config), the reference arm,
# reference-rule timings, phase profiles, launch list of the default bench.  Outputs under
# gpurun_out/<tag>_*; copy what is to be judged into profiles/.
tag=${1:-r02}
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log
./tests/cpp/test_shim > gpurun_out/${tag}_test_shim.txt 2>&1; echo "shim rc=$?" >> gpurun_out/${tag}_test_shim.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench_default.json 2> gpurun_out/${tag}_bench_default.err
for c in 1 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --also '' > gpurun_out/${tag}_bench_cfg$c.json 2> gpurun_out/${tag}_bench_cfg$c.err; done
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --also '' > gpurun_out/${tag}_bench_cfg5.json 2> gpurun_out/${tag}_bench_cfg5.err
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_reference_default.json 2> gpurun_out/${tag}_bench_reference_default.err
for c in 1 2 3 4 5; do timeout 400 python scripts/tail_time.py --config $c > gpurun_out/${tag}_refrule_cfg$c.txt 2>&1; done
for c in 1 2 3 4 5; do timeout 300 python scripts/phase_times.py --config $c > gpurun_out/${tag}_phases_cfg$c.txt 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file gpurun_out/${tag}_launches_bench_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --also '' > gpurun_out/${tag}_launches_bench_default.log 2>&1
echo ALLDONE
