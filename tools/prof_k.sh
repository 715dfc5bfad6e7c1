#!/bin/bash
# ncu --set full of one launch of kernels matching $1 (skip $2 launches) in a C3 step
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-0} -c ${3:-1} \
  -o gpurun_out/prof_k python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_k.log 2>&1
