#!/bin/bash
# GPU tests + A/B of CKB200_NTTTC modes (1 = fwd+inv on tensor cores, 2 = fwd only, 0 = butterflies)
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for i in 1 2; do
  for v in 1 2 0; do
    CKB200_NTTTC=$v timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NTTTC=$v', round(d['value'],1), round(d['ms_per_step'],3))" >> gpurun_out/ab.log
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_list.log 2>&1
