mkdir -p gpurun_out
for c in 3 5 1 2 4; do
  timeout 300 python scripts/phase_times.py --config $c > gpurun_out/p1_pull_cfg$c.txt 2>&1
  timeout 300 python scripts/phase_times.py --config $c --debug-flags 8 > gpurun_out/p1_push_cfg$c.txt 2>&1
  echo "cfg$c pull: $(head -1 gpurun_out/p1_pull_cfg$c.txt) | push: $(head -1 gpurun_out/p1_push_cfg$c.txt)"
done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
