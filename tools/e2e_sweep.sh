#!/bin/bash
# e2e host-pipeline sweep (chunk size x buffer count); run under gpurun
for cfg in "8 2" "8 4" "4 6" "16 3"; do
  set -- $cfg
  timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 --e2e-chunk $1 --e2e-nbuf $2 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); e=d['e2e']; print('chunk',$1,'nbuf',$2,'e2e',round(e['value'],1),'compressed',round(e['compressed_keys']['value'],1), e['matches_device_outputs'], e['compressed_keys']['matches_device_outputs'])"
done
