#!/bin/bash
rm -f gpurun_out/sweep.log
L=paper_2112_06396_b200
for i in 1 2; do
bash tools/sweep_env.sh CKB200_LIB "$L/libckks_b200.so $L/ks_e1r2.so $L/ks_e1r3.so $L/ks_e1r1.so $L/ks_e1r2m4.so $L/ks_e05r2.so $L/ks_e1r0.so"
done
