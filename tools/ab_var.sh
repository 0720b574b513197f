# A/B: in-tree lib vs lib/$VAR.so (HP_LIB_VARIANT) on the U-Net / SD3 forward and GroupNorm shapes
VAR=${VAR:-var_gn}
for v in "" $VAR "" $VAR; do
  echo "== ${v:-current}"
  HP_LIB_VARIANT=$v python tools/time_unet.py | grep forward
  HP_LIB_VARIANT=$v timeout 120 python tools/gn_probe.py
done

