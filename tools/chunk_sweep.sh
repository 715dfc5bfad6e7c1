for c in 1 2 4 8 16 0; do
  echo "chunk=$c $(CKB200_CHUNK=$c python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"])')"
done
