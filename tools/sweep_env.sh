#!/bin/bash
# usage: sweep_env.sh VAR "v1 v2 ..." [bench args]  -> ms/step and value per setting (device-resident C3 unless args)
VAR=$1; VALS=$2; shift 2
for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --no-cpu --no-e2e "$@" 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('$VAR=$v', round(d['ms_per_step'],3), 'ms', round(d['value'],1), d['unit'])
" >> gpurun_out/sweep.log
done
