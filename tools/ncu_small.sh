python tools/profile_step.py int8 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none --cache-control none --profile-from-start off -k regex:step_begin -s 20 -c 1 -o gpurun_out/r01_step_begin python tools/profile_step.py int8 > gpurun_out/ncu_i.log 2>&1
ncu --set full --import-source on --clock-control none --cache-control none --profile-from-start off -k regex:layernorm_reg -s 100 -c 1 -o gpurun_out/r01_layernorm python tools/profile_step.py int8 > gpurun_out/ncu_j.log 2>&1
