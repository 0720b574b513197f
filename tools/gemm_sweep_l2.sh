# level-2 / level-1 GEMM shapes of the SDXL forward (B=2 and B=1) over block_n
for s in "8192 640 640" "4096 640 640" "8192 1920 640" "4096 1920 640" "8192 640 2560" "4096 640 2560" "8192 5120 640" "32768 320 640" "16384 320 640" "2048 3840 1280" "1024 3840 1280"; do
  for bn in 0 64 128 160 256 320; do python tools/prof_gemm.py $s $bn 0 30 2>/dev/null | grep graph; done
done
