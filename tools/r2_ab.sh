#!/bin/bash
# A/B two library builds, alternating, 2 rounds
rm -f gpurun_out/sweep.log
L=paper_2112_06396_b200
for i in 1 2; do
  bash tools/sweep_env.sh CKB200_LIB "$L/libckks_b200.so $L/$1" "${@:2}"
done
