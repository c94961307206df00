# bench A/B over library builds: bash tools/ab_libs.sh <prec> lib1 lib2 ... ("" = in-tree)
P=$1; shift
for i in 1 2; do
for lib in "$@"; do
  r=$(MTG_LIB_PATH=$lib python bench.py --steps 5 --warmup 3 --precision $P --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['p90_batch1_ms'],2))")
  echo "$P lib=${lib:-new} $r"
done; done
