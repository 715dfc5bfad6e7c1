for v in 0 1; do
  CKB200_KSWS=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ks_row -s 1 -c 1 --csv --log-file gpurun_out/ksws_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
  echo "ws=$v $(grep ks_row gpurun_out/ksws_$v.csv | awk -F'","' '{print $NF}')"
done
CKB200_KSWS=1 ncu --set full --clock-control none --import-source on -k regex:ks_row -s 1 -c 1 -o gpurun_out/prof_ws python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
