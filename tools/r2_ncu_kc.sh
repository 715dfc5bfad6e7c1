#!/bin/bash
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kc_row -s 1 -c 1 -o gpurun_out/prof_kc $CMD > gpurun_out/ncu_full.log 2>&1
