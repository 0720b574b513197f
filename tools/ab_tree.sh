# A/B of two source trees: this checkout vs the committed base in _ab/base (git worktree, own built lib)
for t in . _ab/base . _ab/base; do
  echo "== $t"
  (cd $t && python tools/time_unet.py | grep forward && timeout 120 python tools/gn_probe.py | grep GN)
done
