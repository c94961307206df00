set -x
nproc; lscpu | grep -E "Model name|Thread|Socket" 
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 --precision f32 > gpurun_out/bench_f32.json
python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline > gpurun_out/bench_int8.json
python bench.py --steps 5 --warmup 3 --precision bf16 --no-cpu-baseline > gpurun_out/bench_bf16.json
python bench.py --impl reference --steps 2 --warmup 1 --precision f32 > gpurun_out/bench_ref_f32.json
cat gpurun_out/bench_*.json
python tools/profile_step.py int8 > gpurun_out/prof_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_int8.csv python tools/profile_step.py int8 > gpurun_out/ncu_l8.log 2>&1
python tools/profile_step.py f32 > gpurun_out/prof_plain32.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_f32.csv python tools/profile_step.py f32 > gpurun_out/ncu_l32.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_tc -s 107 -c 1 -o gpurun_out/r01_logits_gemm_int8 python tools/profile_step.py int8 > gpurun_out/ncu_a.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:topk -s 20 -c 1 -o gpurun_out/r01_topk_int8 python tools/profile_step.py int8 > gpurun_out/ncu_b.log 2>&1
ls -la gpurun_out
