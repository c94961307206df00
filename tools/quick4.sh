set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline > gpurun_out/q_bench_int8.json 2> gpurun_out/q_bench_int8.err
python -c "import json; d=json.load(open('gpurun_out/q_bench_int8.json')); print(d['value'], d['ms_per_step'], d['p90_batch1_ms'], d['kernels'])"
python tools/diag_step.py int8
