#!/bin/bash
rm -f gpurun_out/sweep.log gpurun_out/pytest_f.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_relin.py -q -x --timeout 600 -k "full_config or relin or c4 or c2" > gpurun_out/pytest_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_f.log
bash tools/sweep_env.sh CKB200_TCPP "0 1"
bash tools/sweep_env.sh CKB200_TCPP "0 1" --config C2
