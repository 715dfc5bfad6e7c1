#!/bin/bash
# ncu --set full of one launch of every kernel of a C3 step (the second step; 1 GPU).
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ntt_row|ntt_col|ks_row|md_row|bconv" \
  -s 10 -c 10 -o gpurun_out/prof_all $CMD > gpurun_out/ncu_all.log 2>&1
