for i in 1 2; do
for m in 0 1 2; do
  MTG_STEP_FUSION=$m python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mode $m', d['value'], d['p90_batch1_ms'])"
done; done
