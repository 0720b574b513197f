for v in attn_v3 attn_v5; do echo "== $v"; for a in "4096 10 20" "1024 20 50" "4096 10 50 77" "1024 20 50 77"; do HP_LIB_VARIANT=$v python tools/prof_attn.py $a; done; done
