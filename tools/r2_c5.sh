#!/bin/bash
rm -f gpurun_out/sweep.log gpurun_out/pytest_f.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extremes.py tests/test_gpu_levels.py tests/test_gpu_shard.py -q -x --timeout 900 -k "C5 or c5 or large or extreme" > gpurun_out/pytest_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_f.log
bash tools/sweep_env.sh CKB200_MD_G "4" --config C5
bash tools/sweep_env.sh CKB200_MD_G "4"
