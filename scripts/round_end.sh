#!/bin/bash
# Everything the round's evidence needs, on the final build, in one GPU call.
bash scripts/r02_parity_job.sh > gpurun_out/r02_parity_job.txt 2>&1
bash scripts/final_evidence.sh r02 > gpurun_out/r02_final_evidence.txt 2>&1
bash scripts/ncu_evidence.sh r02f "3 2 5" > gpurun_out/r02_ncu_evidence.txt 2>&1
tail -3 gpurun_out/r02_parity_job.txt gpurun_out/r02_final_evidence.txt gpurun_out/r02_ncu_evidence.txt
