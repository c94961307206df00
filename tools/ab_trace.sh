# Step-trace A/B: bash tools/ab_trace.sh <prec> <n> "ENV=.. ENV=.." ...  (MTG_LIB_PATH=... selects another build)
P=$1; N=$2; shift 2
for cfg in "" "$@"; do
  echo "== [$cfg]"; env $cfg MTG_TRACE=1 timeout 300 python tools/step_trace.py $P $N 2>&1 | tail -n +3
done
