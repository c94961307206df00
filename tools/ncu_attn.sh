set -x
python tools/profile_step.py int8 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:dec_cross -s 40 -c 1 -o gpurun_out/r01_cross_attn_int8 python tools/profile_step.py int8 > gpurun_out/ncu_f.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:dec_self -s 80 -c 1 -o gpurun_out/r01_self_attn_int8 python tools/profile_step.py int8 > gpurun_out/ncu_g.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base mangled -k regex:ILi0ELi32ELi0E -s 200 -c 1 -o gpurun_out/r01_small_gemm_int8 python tools/profile_step.py int8 > gpurun_out/ncu_h.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:beam_select -s 20 -c 1 -o gpurun_out/r01_beam_select_int8 python tools/profile_step.py int8 > gpurun_out/ncu_e.log 2>&1
