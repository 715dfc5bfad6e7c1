#!/bin/bash
# One-step launch list + ncu --set full of the BC tensor-core kernels (run under gpurun).
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bconv_tc -s 2 -c 2 -o gpurun_out/prof_bctc \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
