# A/B an environment switch: bash tools/ab_env.sh VAR VALUE precision
for i in 1 2 3; do
  python bench.py --steps 5 --warmup 3 --precision $3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('A', round(d['value'],1), round(d['p90_batch1_ms'],2))"
  env $1=$2 python bench.py --steps 5 --warmup 3 --precision $3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B($1=$2)', round(d['value'],1), round(d['p90_batch1_ms'],2))"
done
