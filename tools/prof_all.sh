#!/bin/bash
# ncu --set full of one launch of every kernel of a C3 step (run under gpurun, 1 GPU)
ncu --set full --clock-control none --import-source on -k regex:"ntt_row|ntt_col|ks_row|md_row" -s 7 -c 7 \
  -o gpurun_out/prof_all python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_all.log 2>&1
