#!/bin/bash
# e2e host-pipeline sweep (compressed-key chunk size x buffer count); run under gpurun
for cfg in "8 4" "16 3" "16 4" "32 2" "4 6" "8 2"; do
  set -- $cfg
  timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 --e2e-chunk-compressed $1 --e2e-nbuf $2 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); e=d['e2e']; x=e.get('expanded_keys') or {}; print('chunk',$1,'nbuf',$2,'e2e(compressed)',round(e['value'],1),'expanded',round(x.get('value',0),1), e['matches_device_outputs'])"
done
