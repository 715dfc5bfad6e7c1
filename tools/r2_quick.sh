#!/bin/bash
# core GPU parity subset + C3 bench + one-step launch list (run under gpurun)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_levels.py tests/test_gpu_relin.py tests/test_gpu_batch.py tests/test_gpu_extremes.py -q -x --timeout 600 > gpurun_out/pytest_q.log 2>&1; echo rc=$? >> gpurun_out/pytest_q.log
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --config C3M > gpurun_out/bench_c3m.log 2>&1
timeout 300 python bench.py --config C5 > gpurun_out/bench_c5.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_list.log 2>&1
