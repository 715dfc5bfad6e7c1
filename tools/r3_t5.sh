#!/bin/bash
# ncu --set full of the BC kernels
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bconv" -s 2 -c 2 -o gpurun_out/prof_bc $CMD > gpurun_out/ncu_bc.log 2>&1
ncu -i gpurun_out/prof_bc.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_bc_src.csv 2>/dev/null
