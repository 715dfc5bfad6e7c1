#!/bin/bash
rm -f gpurun_out/sweep.log
L=paper_2112_06396_b200
M=gpu__time_duration.sum
for lib in libckks_b200.so abl_KSNTT.so abl_KSRED.so; do
  CKB200_LIB=$L/$lib ncu --metrics $M --clock-control none -k regex:ks_row -s 1 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e 2>/dev/null | grep ks_row | tail -1 >> gpurun_out/sweep.log
done
