for i in 1 2; do for p in f32 int8; do
  python bench.py --steps 5 --warmup 3 --precision $p --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$p', round(d['value'],1), round(d['p90_batch1_ms'],2))"
done; done
