#!/bin/bash
# every config's bench line (with CPU baseline + clocks) and its one-step ncu launch list
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 600 python bench.py > gpurun_out/line_C3.json 2>gpurun_out/line_C3.err
for c in C1 C2 C3M C4 C5; do
  timeout 600 python bench.py --config $c > gpurun_out/line_$c.json 2>gpurun_out/line_$c.err
done
for c in C3 C1 C2 C3M C4 C5; do
  A="--config $c"; [ $c = C3 ] && A="--no-e2e"
  python bench.py $A --steps 1 --warmup 2 --no-cpu > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py $A --steps 1 --warmup 2 --no-cpu > gpurun_out/ncu_list_$c.log 2>&1
done
