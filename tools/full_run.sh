# Round-end style measurement run (tests, smoke, bench arms, launch lists, ncu captures).
set -x
nproc; lscpu | grep -E "Model name|Thread|Socket"
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 --precision f32 > gpurun_out/bench_f32.json
python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline > gpurun_out/bench_int8.json
python bench.py --steps 5 --warmup 3 --precision bf16 --no-cpu-baseline > gpurun_out/bench_bf16.json
python bench.py --impl reference --steps 2 --warmup 1 --precision f32 > gpurun_out/bench_ref_f32.json
cat gpurun_out/bench_*.json
python tools/diag_step.py f32 > gpurun_out/diag_f32.txt 2>&1
python tools/diag_step.py int8 > gpurun_out/diag_int8.txt 2>&1
# ncu cannot profile kernels inside graphs with conditional (while) nodes:
# the profiled runs drive the same step graphs from the host (MTG_DEVICE_LOOP=0).
export MTG_DEVICE_LOOP=0
for p in int8 f32; do
python tools/profile_step.py $p > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$p.csv python tools/profile_step.py $p > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:logits_tc -s 20 -c 1 -o gpurun_out/logits_f32 python tools/profile_step.py f32 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base mangled -k regex:ILi0ELi256ELi1E -s 20 -c 1 -o gpurun_out/logits_int8 python tools/profile_step.py int8 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:dec_self -s 40 -c 1 -o gpurun_out/self_attn_int8 python tools/profile_step.py int8 > /dev/null 2>&1
ls -la gpurun_out
