#!/bin/bash
# ncu --set full + SASS source page of the forward tensor-core column kernel (ModUp launch)
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt_col_tc -s 5 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_tc.log 2>&1
ncu -i gpurun_out/prof_tc.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_tc_src.csv 2>/dev/null
