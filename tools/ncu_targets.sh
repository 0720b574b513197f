# one ncu --set full capture per dominant kernel; each command runs plain first and is
# profiled only if that run exited 0. Usage: bash tools/ncu_targets.sh <tag>
tag=${1:-r2}
run() {   # run <name> <kernel regex> <skip> <command...>
  local name=$1 k=$2 s=$3; shift 3
  "$@" > gpurun_out/plain_$name.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o gpurun_out/${tag}_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name: $?"
}
run gemm_geglu gemm_pair 3 python tools/prof_gemm.py 2048 10240 1280 256 3 3 eager
run gemm_oproj gemm_pair 3 python tools/prof_gemm.py 2048 1280 1280 0 0 3 eager
run gemm_splitk gemm_splitk 3 python tools/prof_gemm.py conv 2 32 32 1280 1280 1 0 3
run attn_s1024 attn_stream 2 python tools/prof_attn.py 1024 20 3
run attn_s4096 attn_stream 2 python tools/prof_attn.py 4096 10 3
run attn_sd3 attn_stream 2 python tools/prof_attn.py 4429 24 3
run attn_cross attn_single 2 python tools/prof_attn.py 1024 20 3 77
run gn_parts gn_parts 0 python tools/gn_parts_time.py
