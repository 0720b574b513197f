for v in "" var_nomask "" var_nomask; do echo "== ${v:-current}"; for a in "4096 10 20" "1024 20 50"; do HP_LIB_VARIANT=$v python tools/prof_attn.py $a; done; done
