#!/bin/bash
# Final measurement pass (run under gpurun): one-step ncu launch lists of every config ->
# profiles/r02_traffic.json (DRAM bytes per unit, fma-heavy use) -> every config's bench line
# (with CPU baseline, clocks, e2e for C3) -> the reference arm.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed
for c in C3 C1 C2 C3M C4 C5; do
  A="--config $c"; [ $c = C3 ] && A="--no-e2e"
  python bench.py $A --steps 1 --warmup 2 --no-cpu > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py $A --steps 1 --warmup 2 --no-cpu > gpurun_out/ncu_list_$c.log 2>&1
done
python tools/traffic_json.py profiles/r02_traffic.json C3:gpurun_out/launches_C3.csv:10:64 \
  C1:gpurun_out/launches_C1.csv:10:1 C2:gpurun_out/launches_C2.csv:4:384 C3M:gpurun_out/launches_C3M.csv:12:64 \
  C4:gpurun_out/launches_C4.csv:25:1 C5:gpurun_out/launches_C5.csv:10:32 > gpurun_out/traffic_json.log 2>&1
cp profiles/r02_traffic.json gpurun_out/r02_traffic.json
timeout 900 python bench.py > gpurun_out/line_C3.json 2>gpurun_out/line_C3.err
for c in C1 C2 C3M C4 C5; do
  timeout 900 python bench.py --config $c > gpurun_out/line_$c.json 2>gpurun_out/line_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/line_reference.json 2>gpurun_out/line_reference.err
