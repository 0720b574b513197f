for s in "2048 1280 1280 0 0 20" "2048 3840 1280 0 0 20" "2048 10240 1280 256 3 20" "8192 640 640 0 0 20" "8192 1920 640 0 0 20"; do
  echo "-- $s"; python tools/prof_gemm.py $s | tail -1; (cd _ab/head && python tools/prof_gemm.py $s | tail -1)
done
python tools/prof_gemm.py 2048 1280 1280 0 0 20 graph stats | tail -1
python tools/prof_gemm.py 2048 3840 1280 0 0 20 graph fold | tail -1
python tools/prof_gemm.py 2048 10240 1280 256 3 20 graph fold | tail -1
python tools/prof_gemm.py 8192 1920 640 0 0 20 graph fold | tail -1
