#!/bin/bash
# gpu tests + C3 / C3M bench lines (device-resident only); run under gpurun
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --config C3M > gpurun_out/bench_c3m.log 2>&1
