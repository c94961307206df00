for i in 1 2; do
for p in bf16 int8 f32; do
for lib in "" "build_ab/libminimt_gpu_head.so"; do
  r=$(MTG_LIB_PATH=$lib python bench.py --steps 5 --warmup 3 --precision $p --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['p90_batch1_ms'],2))")
  echo "$p lib=${lib:-new} $r"
done; done; done
