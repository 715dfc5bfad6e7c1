#!/bin/bash
rm -f gpurun_out/sweep.log
for e in 0 2; do export CKB200_KEY_EARLY=$e; echo "EARLY=$e" >> gpurun_out/sweep.log; bash tools/sweep_env.sh CKB200_KEY_LATE "2 4 6 8"; done
