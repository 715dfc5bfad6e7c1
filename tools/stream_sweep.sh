for cfg in "1 0" "2 0" "2 8" "3 0" "4 0" "2 16"; do
  set -- $cfg
  echo "streams=$1 chunk=$2 $(CKB200_STREAMS=$1 CKB200_CHUNK=$2 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"])')"
done
