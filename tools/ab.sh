# A/B: python tools/ab.sh ENVVAR  -> 3 alternating bench runs per arm
for i in 1 2 3; do
  python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('A', d['value'], d['p90_batch1_ms'])"
  env $1=1 python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B', d['value'], d['p90_batch1_ms'])"
done
