#!/bin/bash
# parity of the full configs + ncu --set full of the BC kernels
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_relin.py -q -x --timeout 600 -k "full_config or relin or c4" > gpurun_out/pytest_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_f.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bconv" -s 2 -c 2 -o gpurun_out/prof_bc $CMD > gpurun_out/ncu_bc.log 2>&1
