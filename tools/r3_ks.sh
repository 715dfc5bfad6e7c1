#!/bin/bash
rm -f gpurun_out/sweep.log
L=paper_2112_06396_b200
for i in 1 2; do
bash tools/sweep_env.sh CKB200_LIB "$L/libckks_b200.so $(ls $L/v_*.so | tr '\n' ' ')"
done
