# one ncu --set full capture per dominant kernel (run only after the same commands exited 0 without ncu)
set -x
ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 3 -c 1 -o gpurun_out/full_gemm_geglu python tools/prof_gemm.py 2048 10240 1280 256 3 3 eager
ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 3 -c 1 -o gpurun_out/full_gemm_oproj python tools/prof_gemm.py 2048 1280 1280 0 0 3 eager
ncu --set full --clock-control none --import-source on -k regex:gemm_splitk -s 3 -c 1 -o gpurun_out/full_gemm_splitk python tools/prof_gemm.py conv 2 32 32 1280 1280 1 0 3
ncu --set full --clock-control none --import-source on -k regex:attn -s 2 -c 1 -o gpurun_out/full_attn_s1024 python tools/prof_attn.py 1024 20 3
ncu --set full --clock-control none --import-source on -k regex:attn -s 2 -c 1 -o gpurun_out/full_attn_s4096 python tools/prof_attn.py 4096 10 3
