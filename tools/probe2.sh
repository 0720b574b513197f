for e in 0 1; do
 for s in "8192 1920 640 160" "8192 2048 2560 128" "2048 1280 1280" "8192 640 640 160" "4096 4096 4096 256" "2048 10240 1280 256 3"; do
  if [ $e = 1 ]; then HP_GEMM_RASTER_N=1 python tools/prof_gemm.py $s | tail -1; else python tools/prof_gemm.py $s | tail -1; fi
 done
 for s in "2 32 32 2560 1280 1" "2 64 64 640 640 1"; do
  if [ $e = 1 ]; then HP_GEMM_RASTER_N=1 python tools/prof_gemm.py conv $s | tail -1; else python tools/prof_gemm.py conv $s | tail -1; fi
 done
done
