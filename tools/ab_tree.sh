# A/B of two source trees: this checkout vs the committed base in _ab/base (git worktree, own built lib)
for t in . _ab/base . _ab/base; do
  echo "== $t"
  (cd $t && python tools/time_unet.py | grep forward)
done
for t in . _ab/base; do echo "== VAE $t"; (cd $t && python tools/time_vae.py 2>&1 | tail -1); done
