for bn in 0 32 64 128 256; do
  echo "== MTG_ENC_BN=$bn"; MTG_ENC_BN=$bn python tools/enc_probe.py 2>&1 | tail -2
done
