# Full ncu captures of the fused output projection and the softmax/top-k merge.
set -x
python tools/profile_step.py int8 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base mangled -k regex:ILi0ELi256ELi1E -s 20 -c 1 -o gpurun_out/r01_logits_fused_int8 python tools/profile_step.py int8 > gpurun_out/ncu_c.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:softmax_topk -s 20 -c 1 -o gpurun_out/r01_softmax_topk_int8 python tools/profile_step.py int8 > gpurun_out/ncu_d.log 2>&1
ls -la gpurun_out
python tools/profile_step.py int8 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv --log-file gpurun_out/q_launches_int8_warm.csv python tools/profile_step.py int8 > gpurun_out/q_ncu.log 2>&1
python tools/launches.py gpurun_out/q_launches_int8_warm.csv | head -8
