#!/bin/bash
CMD="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ntt_col_tc2" -s 2 -c 2 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_full.log 2>&1
