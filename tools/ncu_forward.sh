# ncu launch lists (device time + DRAM bytes per kernel) of one eager SDXL forward,
# B=2 (CFG batch) and B=1 (one branch); run after `python tools/prof_forward.py 2` exited 0.
# Usage: bash tools/ncu_forward.sh <tag>
tag=${1:-r2}
K='regex:^(gemm|attn|gn_|ln_|timestep|embed|add_rows|concat|conv_small|copy_cols|upsample|silu|cast|gated|patchify|softmax|quick)'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/prof_forward.py 2 > gpurun_out/pf_plain.log 2>&1 &&
python tools/prof_forward.py 2 b1 > gpurun_out/pf_plain_b1.log 2>&1 &&
ncu --metrics $M --clock-control none --kernel-name-base function -k "$K" -c 1400 --csv \
    --log-file gpurun_out/launches_fwd_$tag.csv python tools/prof_forward.py 2 > gpurun_out/ncu_fwd.log 2>&1 &&
ncu --metrics $M --clock-control none --kernel-name-base function -k "$K" -c 1400 --csv \
    --log-file gpurun_out/launches_fwd_b1_$tag.csv python tools/prof_forward.py 2 b1 > gpurun_out/ncu_fwd_b1.log 2>&1
echo ncu_forward=$?
