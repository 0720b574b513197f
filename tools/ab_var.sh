# A/B: in-tree lib vs lib/$VAR.so (HP_LIB_VARIANT) on the U-Net / SD3 forward
VAR=${VAR:-var_base}
for v in "" $VAR "" $VAR; do
  echo "== ${v:-current}"
  HP_LIB_VARIANT=$v python tools/time_unet.py | grep forward
done
