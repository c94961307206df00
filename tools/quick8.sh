python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for p in int8 f32; do
for v in 1 0; do
MTG_LOGITS_PERSISTENT=$v python bench.py --steps 5 --warmup 3 --precision $p --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$p persistent=$v', d['value'], d['p90_batch1_ms'], d['kernels']['logits_gemm']['ms'])"
done; done
