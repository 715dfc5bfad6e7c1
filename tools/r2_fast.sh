#!/bin/bash
# parity of the full configs + C3 bench + one-step launch list (run under gpurun)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_relin.py -q -x --timeout 600 -k "full_config or relin or c4" > gpurun_out/pytest_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_f.log
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_list.log 2>&1
