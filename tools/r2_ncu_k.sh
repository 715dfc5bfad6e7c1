#!/bin/bash
# usage: r2_ncu_k.sh CONFIG KERNEL_REGEX SKIP  -> gpurun_out/prof_k.ncu-rep (one launch, --set full)
c=$1; A="--config $c"; [ $c = C3 ] && A="--no-e2e"
CMD="python bench.py $A --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${3:-1} -c 1 -o gpurun_out/prof_k $CMD > gpurun_out/ncu_full.log 2>&1
