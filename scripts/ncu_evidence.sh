#!/bin/bash
# ncu evidence for the north-star counters: per config, one
# --set full capture of every solver kernel of one solve (the persistent
# kernel and the per-phase kernels) and of the estimate gather probe, after
# the same command ran clean without ncu; summarised per config.
#   scripts/ncu_evidence.sh <tag> "<configs>"
tag=$1; cfgs=${2:-"3 5"}
mkdir -p gpurun_out
for c in $cfgs; do
  cmd="python scripts/prof_solve.py --config $c --reps 1 --probe 1"
  $cmd > gpurun_out/${tag}_cfg${c}_plain.log 2>&1 || { echo "plain run failed cfg$c"; continue; }
  timeout 2400 ncu --set full --clock-control none \
      -k regex:"count_rounds_kernel|count_phase_kernel|est_gather_probe" -c 80 -f \
      -o gpurun_out/${tag}_cfg${c} $cmd > gpurun_out/${tag}_cfg${c}_ncu.log 2>&1
  echo "cfg$c ncu exit $?"
  nnz=$(python -c "import re,sys; print(re.search(r'over (\d+) entries', open('gpurun_out/${tag}_cfg${c}_plain.log').read()).group(1))")
  python scripts/ncu_evidence_summary.py gpurun_out/${tag}_cfg${c}.ncu-rep $nnz > gpurun_out/${tag}_ncu_evidence_cfg${c}.json 2> gpurun_out/${tag}_ncu_evidence_cfg${c}.err
  # per-launch table (kernel, duration, DRAM bytes, warps active, registers) as text; the report
  # itself (tens of kernels x full set) is too large to bring back
  ncu -i gpurun_out/${tag}_cfg${c}.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__block_size,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum > gpurun_out/${tag}_ncu_launches_cfg${c}.csv 2>/dev/null
  rm -f gpurun_out/${tag}_cfg${c}.ncu-rep
done
