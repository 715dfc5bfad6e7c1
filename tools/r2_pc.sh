#!/bin/bash
rm -f gpurun_out/sweep.log gpurun_out/pytest_f.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_levels.py tests/test_gpu_relin.py -q -x --timeout 600 > gpurun_out/pytest_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_f.log
bash tools/sweep_env.sh CKB200_BSGS_FUSED "1" --config C4
bash tools/sweep_env.sh CKB200_BSGS_FUSED "1"
