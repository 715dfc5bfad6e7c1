#!/bin/bash
# full GPU suite + quick device-resident lines
rm -f gpurun_out/sweep.log
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
bash tools/sweep_env.sh CKB200_MD_G "4"
bash tools/sweep_env.sh CKB200_MD_G "4" --config C4
bash tools/sweep_env.sh CKB200_MD_G "4" --config C2
