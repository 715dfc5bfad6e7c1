#!/bin/bash
# small-batch efficiency of the fused key-switch (the API's one-ciphertext calls): ms per step and launch lists
rm -f gpurun_out/sweep.log
for b in 1 2 4 8 16 64; do
  timeout 300 python bench.py --no-cpu --no-e2e --batch $b 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('batch=$b', round(d['ms_per_step'],4), 'ms', round(d['value'],1), d['unit'])
" >> gpurun_out/sweep.log
done
cp gpurun_out/sweep.log gpurun_out/r4_small_sweep.log
for b in 1 4; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/r4_launches_b$b.csv python bench.py --steps 1 --warmup 2 --no-cpu --no-e2e --batch $b > gpurun_out/r4_ncu_b$b.log 2>&1
done
