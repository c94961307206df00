# Decoder GEMM tiling sweep at batch 64 from the in-graph timeline
# (tools/step_trace.py): per config, each GEMM's duration and the step time.
#   bash tools/dec_gemm_sweep.sh <f32|int8|bf16> "ENV=.. ENV=.." ...
P=$1; shift
for cfg in "" "$@"; do
  out=$(env $cfg MTG_TRACE=1 timeout 300 python tools/step_trace.py $P 64 2>&1)
  echo "[$cfg] $(echo "$out" | grep -E '^ +(2|4|6|8|10|11) gemm' | awk '{printf "%s=%s ", $3, $NF}') $(echo "$out" | grep 'step ' | awk '{print "step", $2}')"
done
