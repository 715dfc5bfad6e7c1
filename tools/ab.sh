#!/bin/bash
# A/B: default lib vs each .so given (CKB200_LIB), C3 device-resident bench, 2 rounds (run under gpurun)
# extra bench args via $BENCH_ARGS
for i in 1 2; do
  for lib in default "$@"; do
    if [ "$lib" = default ]; then env=""; else env="CKB200_LIB=$lib"; fi
    env $env timeout 300 python bench.py --no-cpu --no-e2e $BENCH_ARGS 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['ms_per_step'],3))" >> gpurun_out/ab.log
  done
done
