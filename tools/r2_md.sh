#!/bin/bash
rm -f gpurun_out/sweep.log gpurun_out/pytest_f.log
L=paper_2112_06396_b200
for lib in md_t1.so md_t1e1.so; do
CKB200_LIB=$L/$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_relin.py -q -x --timeout 600 -k "C3_rot or C5_rot0 or C1_rot or new_mult or relin" >> gpurun_out/pytest_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_f.log
done
for i in 1 2; do
bash tools/sweep_env.sh CKB200_LIB "$L/libckks_b200.so $L/md_t1.so $L/md_t1e1.so $L/md_t1e1m6.so $L/md_t0e1.so"
done
