for v in "" var_deg3 var_deg3half; do echo "== ${v:-current}"; for a in "4096 10 20" "1024 20 50"; do HP_LIB_VARIANT=$v python tools/prof_attn.py $a; done; done
HP_LIB_VARIANT=var_deg3 timeout 120 python -m pytest tests/test_denoiser_kernels_gpu.py -q -k attention 2>&1 | tail -1
HP_LIB_VARIANT=var_deg3half timeout 120 python -m pytest tests/test_denoiser_kernels_gpu.py -q -k attention 2>&1 | tail -1
