#!/bin/bash
# A/B: default lib vs $1 (CKB200_LIB), C3 device-resident bench, 2 runs each (run under gpurun)
ALT=${1:-paper_2112_06396_b200/libckks_exact.so}
for i in 1 2; do
  timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['value'], d['ms_per_step'])" >> gpurun_out/ab.log
  CKB200_LIB=$ALT timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('alt', d['value'], d['ms_per_step'])" >> gpurun_out/ab.log
done
