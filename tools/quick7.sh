python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for p in int8 f32; do
python bench.py --steps 5 --warmup 3 --precision $p --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$p', d['value'], d['ms_per_step'], d['p90_batch1_ms'])"
done
python tools/diag_step.py int8 | sed -n '/encoder/,$p'
