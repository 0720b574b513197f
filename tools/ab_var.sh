for v in "" var_noact "" var_noact; do echo "== ${v:-current}"; HP_LIB_VARIANT=$v python tools/time_unet.py | grep forward; done
