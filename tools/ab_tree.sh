# A/B of two source trees: this checkout vs the committed base in _ab/base (git worktree, own built lib)
for t in . _ab/base . _ab/base; do
  echo "== $t"
  (cd $t && python tools/time_unet.py | grep forward && for a in "4096 10 20" "1024 20 50" "333 10 50"; do python tools/prof_attn.py $a; done)
done
