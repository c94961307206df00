set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline > gpurun_out/q_bench_int8.json 2> gpurun_out/q_bench_int8.err
python -c "import json; d=json.load(open('gpurun_out/q_bench_int8.json')); print(d['value'], d['ms_per_step'], d['kernels'])"
python tools/profile_step.py int8 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv --log-file gpurun_out/q_launches_int8_warm.csv python tools/profile_step.py int8 > gpurun_out/q_ncu.log 2>&1
python tools/launches.py gpurun_out/q_launches_int8_warm.csv > gpurun_out/q_launches.txt; head -12 gpurun_out/q_launches.txt
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base mangled -k regex:ILi0ELi256ELi1E -s 20 -c 1 -o gpurun_out/r01_logits_fused_int8 python tools/profile_step.py int8 > gpurun_out/ncu_c.log 2>&1
