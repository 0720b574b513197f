timeout 300 python -m pytest tests/test_denoiser_kernels_gpu.py -x -q 2>&1 | tail -3
for s in "2048 1280 1280" "2048 3840 1280" "2048 10240 1280 256 3" "8192 640 640" "8192 1920 640" "8192 5120 640 256 3" "4096 4096 4096"; do
  timeout 60 python tools/prof_gemm.py $s | tail -1
done
python tools/time_unet.py | grep forward
