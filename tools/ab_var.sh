for v in "" var_noqgelu var_oldattn; do echo "== ${v:-current}"; HP_LIB_VARIANT=$v python tools/time_unet.py | grep forward; done
