#!/bin/bash
rm -f gpurun_out/sweep.log
L=paper_2112_06396_b200
for pp in 0 1; do
  export CKB200_TCPP=$pp
  echo "TCPP=$pp" >> gpurun_out/sweep.log
  bash tools/sweep_env.sh CKB200_LIB "$L/libckks_b200.so $L/abl_TWIST.so $L/abl_RED.so $L/abl_MMA.so" --config C2
done
