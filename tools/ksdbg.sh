for d in 0 1 2 4 7 3; do
  CKB200_KSDBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ks_row -s 1 -c 1 --csv --log-file gpurun_out/ksdbg_$d.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
done
