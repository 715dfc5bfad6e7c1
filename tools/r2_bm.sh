#!/bin/bash
rm -f gpurun_out/sweep.log
L=paper_2112_06396_b200
bash tools/sweep_env.sh CKB200_LIB "$L/libckks_b200.so $L/bm_NSG_1.so $L/bm_MINB_3.so $L/bm_MINB_4.so $L/libckks_b200.so" --config C4
