timeout 300 python -m pytest tests/test_denoiser_kernels_gpu.py -x -q -k attention 2>&1 | tail -2
for v in 1 0; do echo "== HP_ATTN_SOLO=$v"; for a in "4096 10 20" "1024 20 50"; do HP_ATTN_SOLO=$v python tools/prof_attn.py $a; done; done
python tools/time_unet.py | grep forward
