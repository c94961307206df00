# A/B the e2e (public API, host buffers) number of two library builds: bash tools/ab_e2e.sh LIB_B precision
P=${2:-int8}
for i in 1 2 3; do
  python bench.py --steps 5 --warmup 3 --precision $P --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('A(tree)', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  MTG_LIB_PATH=$1 python bench.py --steps 5 --warmup 3 --precision $P --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
