#!/bin/bash
rm -f gpurun_out/sweep.log
L=paper_2112_06396_b200
bash tools/sweep_env.sh CKB200_LIB "$L/libckks_b200.so $L/abl_LOAD.so $L/abl_STORE.so $L/abl_TWIST.so $L/abl_ALL.so" --config C2
