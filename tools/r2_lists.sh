#!/bin/bash
export CKB200_KC=0
for c in C4 C5 C3M; do
python bench.py --config $c --steps 1 --warmup 1 > gpurun_out/plain_$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 > gpurun_out/ncu_list_$c.log 2>&1
done
