# A/B two library builds on one box: bash tools/ab_lib.sh LIB_B [precision]
P=${2:-int8}
for i in 1 2 3; do
  python bench.py --steps 5 --warmup 3 --precision $P --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('A(tree)', d['value'], d['p90_batch1_ms'])"
  MTG_LIB_PATH=$1 python bench.py --steps 5 --warmup 3 --precision $P --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B($1)', d['value'], d['p90_batch1_ms'])"
done
