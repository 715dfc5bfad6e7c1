#!/bin/bash
# partial key-tile L2 prefetch sweep in ks_row (CKB200_KPF = eighths of the tile)
for v in 0 1 2 4 8; do
  CKB200_KPF=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:ks_row -s 1 -c 1 --csv --log-file gpurun_out/kpf_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
  echo "kpf=$v $(grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/kpf_$v.csv | tail -1) $(grep -o '"dram__bytes_read.sum","[A-Za-z]*","[0-9.,]*"' gpurun_out/kpf_$v.csv | tail -1)"
done
