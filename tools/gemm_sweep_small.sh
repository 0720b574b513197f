for M in 1024 2048; do
 for bn in 0 64 128 160 256 320; do python tools/prof_gemm.py $M 1280 1280 $bn 0 50; done
 for K in 64 320 640 2560 5120; do python tools/prof_gemm.py $M 1280 $K 0 0 50; done
 python tools/prof_gemm.py $M 3840 1280 0 0 50
done
