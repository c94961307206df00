# Decoder GEMM tile-width sweep (MTG_DEC_BN_MAP="NxK:bn"): bash tools/ab_decbn_map.sh precision
P=${1:-f32}
for m in "" "2048x512:64" "2048x512:128" "1536x512:64" "512x512:64"; do
  echo "MAP=$m $(MTG_DEC_BN_MAP=$m python bench.py --steps 5 --warmup 3 --precision $P --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['p90_batch1_ms'],2))")"
done
