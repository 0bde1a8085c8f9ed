set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/n_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/n_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/n_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/n_bench_default.json 2> gpurun_out/n_bench_default.err
for c in 1 2 3 4 5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/n_bench_cfg$c.json 2> gpurun_out/n_bench_cfg$c.err; done
timeout 600 python bench.py --impl reference --config 3 --steps 2 --warmup 1 > gpurun_out/n_bench_reference_cfg3.json 2> gpurun_out/n_bench_reference_cfg3.err
timeout 600 python bench.py --impl reference > gpurun_out/n_bench_reference_default.json 2> gpurun_out/n_bench_reference_default.err
for c in 1 2 3 4 5; do timeout 400 python scripts/tail_time.py --config $c > gpurun_out/n_refrule_cfg$c.txt 2>&1; done
bash scripts/profile_round.sh r01n 3 > gpurun_out/n_profile.log 2>&1
echo ALLDONE
