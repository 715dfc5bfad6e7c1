#!/bin/bash
export CKB200_KC=0
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ks_row|md_row|ntt_row" -s 3 -c 4 -o gpurun_out/prof_rows $CMD > gpurun_out/ncu_full.log 2>&1
