# GEMM launch floor vs work, graph mode (PDL on, then off)
for pdl in 0 1; do
  echo "== HP_NO_PDL=$pdl"
  for s in "2048 1280 64" "2048 1280 1280" "2048 1280 5120" "2048 3840 1280" "2048 10240 1280 0 3" "8192 640 640" "256 1280 64"; do
    HP_NO_PDL=$pdl python tools/prof_gemm.py $s 2>&1 | tail -1
  done
done
