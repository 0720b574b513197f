for v in "" var_lean "" var_lean; do echo "== ${v:-current}"; HP_LIB_VARIANT=$v python tools/time_unet.py | grep forward; done
