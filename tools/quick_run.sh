# Quick GPU check: parity tests, int8 bench, warm-cache launch list.
set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline > gpurun_out/q_bench_int8.json 2> gpurun_out/q_bench_int8.err
python bench.py --steps 5 --warmup 3 --precision f32 --no-cpu-baseline > gpurun_out/q_bench_f32.json 2> gpurun_out/q_bench_f32.err
cat gpurun_out/q_bench_f32.json
cat gpurun_out/q_bench_int8.json
python tools/profile_step.py int8 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv --log-file gpurun_out/q_launches_int8_warm.csv python tools/profile_step.py int8 > gpurun_out/q_ncu.log 2>&1
python tools/launches.py gpurun_out/q_launches_int8_warm.csv | head -20
