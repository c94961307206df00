python bench.py --steps 5 --warmup 3 --precision f32 --no-cpu-baseline > gpurun_out/q_bench_f32.json 2> gpurun_out/q_bench_f32.err
python -c "import json; d=json.load(open('gpurun_out/q_bench_f32.json')); print(d['value'], d['ms_per_step'], d['p90_batch1_ms'], d['kernels'])"
python tools/diag_step.py f32
