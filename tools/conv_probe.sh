for s in "2 128 128 320 320 1" "2 64 64 640 640 1" "2 32 32 1280 1280 1" "2 64 64 320 640 1" "2 32 32 2560 1280 1" "2 128 128 640 320 1" "2 128 128 320 320 2" "2 64 64 640 640 2"; do
  for bn in 0 256 128; do timeout 60 python tools/prof_gemm.py conv $s $bn | tail -1; done
done
