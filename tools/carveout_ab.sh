set -x
python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline > gpurun_out/ab_on.json 2>&1
MTG_MIXED_CARVEOUT=1 python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline > gpurun_out/ab_off.json 2>&1
python -c "
import json
for f in ['ab_on','ab_off']:
    d=json.loads(open('gpurun_out/'+f+'.json').read().strip().splitlines()[-1]); print(f, d['value'], d['ms_per_step'], d['p90_batch1_ms'])
"
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/profile_step.py int8 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv --log-file gpurun_out/q_launches_int8_warm.csv python tools/profile_step.py int8 > gpurun_out/q_ncu.log 2>&1
python tools/launches.py gpurun_out/q_launches_int8_warm.csv > gpurun_out/q_launches.txt; head -14 gpurun_out/q_launches.txt
