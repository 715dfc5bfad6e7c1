#!/bin/bash
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${1:-ks_row} -s 1 -c 1 -o gpurun_out/prof_k $CMD > gpurun_out/ncu_k.log 2>&1
ncu -i gpurun_out/prof_k.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_k_src.csv 2>/dev/null
