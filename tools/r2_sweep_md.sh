#!/bin/bash
rm -f gpurun_out/sweep.log gpurun_out/pytest_f.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_relin.py -q -x --timeout 600 -k "full_config or relin or c4" > gpurun_out/pytest_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_f.log
bash tools/sweep_env.sh CKB200_MD_G "1 2 4 8 16"
