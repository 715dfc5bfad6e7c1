#!/bin/bash
# usage: r2_list.sh CONFIG  -> gpurun_out/launches_CONFIG.csv (one-step launch list)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed
c=$1; A="--config $c"; [ $c = C3 ] && A="--no-e2e"
python bench.py $A --steps 1 --warmup 2 --no-cpu > gpurun_out/plain_$c.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$c.csv \
  python bench.py $A --steps 1 --warmup 2 --no-cpu > gpurun_out/ncu_list_$c.log 2>&1
