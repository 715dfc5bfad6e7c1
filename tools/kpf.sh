for v in 1 0; do
  echo "kpf=$v $(CKB200_KPF=$v python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"])')"
  CKB200_KPF=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:ks_row -s 1 -c 1 --csv --log-file gpurun_out/kpf_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
  grep ks_row gpurun_out/kpf_$v.csv | awk -F'","' '{print $(NF-2), $NF}'
done
