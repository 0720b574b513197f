timeout 300 python -m pytest tests/test_denoiser_kernels_gpu.py -x -q 2>&1 | tail -2
for s in "8192 640 640 320" "8192 640 640 160" "8192 640 2560 320" "8192 640 2560 160" "32768 320 640 320" "32768 320 640 160" "8192 1920 640 320" "8192 1920 640 160"; do python tools/prof_gemm.py $s | tail -1; done
for s in "2 128 128 320 320 1 320" "2 128 128 320 320 1 160" "2 64 64 640 640 1 320" "2 64 64 640 640 1 160" "2 128 128 640 320 1 320"; do python tools/prof_gemm.py conv $s | tail -1; done
python tools/time_unet.py | grep forward
