for cfg in "148 160" "296 160" "296 96" "444 64"; do
  set -- $cfg
  for p in f32 int8; do
  MTG_SPLIT_CTAS=$1 MTG_SPLIT_KB=$2 python bench.py --steps 5 --warmup 3 --precision $p --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ctas=$1 kb=$2 $p', round(d['value'],1), round(d['p90_batch1_ms'],2))"
  done
done
