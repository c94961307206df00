# Round-2 measurement run: tests, smoke, bench arms, in-graph timelines,
# launch lists, ncu captures; outputs under gpurun_out/r02_*, summaries copied
# into profiles/r02/ (tools/ncu_summary.py, tools/launches.py). The per-phase
# timelines need build_ab/libminimt_gpu_phases.so (tools/build_phases.sh).
# Three gpurun calls (each call's gpurun_out/ must stay under 64 MiB):
#   bash tools/full_run_r02.sh a   tests, smoke, bench arms, timelines, launch lists
#   bash tools/full_run_r02.sh b   ncu captures of the two output projections
#   bash tools/full_run_r02.sh c   the remaining ncu captures
set -x
O=gpurun_out
if [ "$1" = "a" ]; then
nproc; lscpu | grep -E "Model name|Thread|Socket"
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 --precision f32 > $O/r02_bench_f32.json
python bench.py --steps 5 --warmup 3 --precision int8 --no-cpu-baseline > $O/r02_bench_int8.json
python bench.py --steps 5 --warmup 3 --precision bf16 --no-cpu-baseline > $O/r02_bench_bf16.json
python bench.py --impl reference --steps 2 --warmup 1 --precision f32 > $O/r02_bench_ref_f32.json
cat $O/r02_bench_*.json
for p in f32 int8 bf16; do
  MTG_TRACE=1 python tools/step_trace.py $p 64 > $O/r02_trace_${p}_b64.txt 2>&1
  MTG_LIB_PATH=build_ab/libminimt_gpu_phases.so MTG_TRACE=2 python tools/step_trace.py $p 64 > $O/r02_trace_phases_${p}_b64.txt 2>&1
  MTG_TRACE=1 python tools/b1_trace.py $p > $O/r02_trace_${p}_b1.txt 2>&1
done
fi
# ncu cannot profile kernels inside graphs with conditional (while) nodes:
# the profiled runs drive the same step graphs from the host (MTG_DEVICE_LOOP=0).
export MTG_DEVICE_LOOP=0
if [ "$1" = "a" ]; then
for p in int8 f32; do
  for n in 64 1; do
    python tools/profile_step.py $p $n > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/r02_launches_${p}_b$n.csv python tools/profile_step.py $p $n > /dev/null 2>&1
  done
done
fi
[ "$1" = "a" ] && { ls -la $O; exit 0; }
NCU="ncu --set full --import-source on --clock-control none --profile-from-start off"
if [ "$1" = "b" ]; then
$NCU -k regex:logits_tc2 -s 20 -c 1 -o $O/r02_logits_f32_pair python tools/profile_step.py f32 > /dev/null 2>&1
$NCU --kernel-name-base mangled -k regex:ILi0ELi256ELi1E -s 20 -c 1 -o $O/r02_logits_int8 python tools/profile_step.py int8 > /dev/null 2>&1
ls -la $O; exit 0; fi
# part c: the remaining captures
$NCU -k regex:gemm_tc_kernel -s 88 -c 1 -o $O/r02_gemm_qkv_f32 python tools/profile_step.py f32 > /dev/null 2>&1
$NCU -k regex:dec_self -s 40 -c 1 -o $O/r02_self_attn_f32 python tools/profile_step.py f32 > /dev/null 2>&1
$NCU -k regex:attn_cross_sent -s 40 -c 1 -o $O/r02_cross_attn_f32 python tools/profile_step.py f32 > /dev/null 2>&1
$NCU --kernel-name-base mangled -k regex:gemv_kernelILi0ELb1E -s 4 -c 1 -o $O/r02_b1_gemv_logits_int8 python tools/profile_step.py int8 1 > /dev/null 2>&1
$NCU --kernel-name-base mangled -k regex:gemv_kernelILi2ELb1E -s 4 -c 1 -o $O/r02_b1_gemv_logits_f32 python tools/profile_step.py f32 1 > /dev/null 2>&1
$NCU -k regex:attn_small -s 8 -c 1 -o $O/r02_b1_self_attn_int8 python tools/profile_step.py int8 1 > /dev/null 2>&1
$NCU -k regex:topk_select -s 20 -c 1 -o $O/r02_tail_f32 python tools/profile_step.py f32 > /dev/null 2>&1
ls -la $O
