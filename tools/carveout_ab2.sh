python tools/profile_step.py int8 > /dev/null 2>&1
MTG_MAX_CARVEOUT=1 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv --log-file gpurun_out/ab_launches_max.csv python tools/profile_step.py int8 > /dev/null 2>&1
python tools/launches.py gpurun_out/ab_launches_max.csv > gpurun_out/ab_launches_max.txt
