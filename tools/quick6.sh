python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for p in int8 f32; do
python bench.py --steps 5 --warmup 3 --precision $p --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$p', d['value'], d['ms_per_step'], d['p90_batch1_ms'])"
MTG_NO_SPLIT_K=1 python bench.py --steps 5 --warmup 3 --precision $p --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$p nosplit', d['value'], d['ms_per_step'], d['p90_batch1_ms'])"
done
python tools/diag_step.py f32 | grep -E "gemm|total"
