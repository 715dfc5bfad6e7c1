#!/bin/bash
# A/B two library builds, alternating, 3 rounds (device-resident C3 unless extra args)
rm -f gpurun_out/sweep.log
L=paper_2112_06396_b200
for i in 1 2 3; do
  bash tools/sweep_env.sh CKB200_LIB "$L/libckks_b200.so $L/$1" "${@:2}"
done
