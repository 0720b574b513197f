timeout 300 python -m pytest tests/test_denoiser_kernels_gpu.py -x -q -k attention 2>&1 | tail -2
for a in "4096 10 20" "1024 20 50" "4096 10 50 77" "1024 20 50 77"; do python tools/prof_attn.py $a; done
python tools/time_unet.py | grep forward
