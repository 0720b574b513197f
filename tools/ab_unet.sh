# A/B the U-Net forward: this tree vs _ab/head (a git worktree of another commit)
for i in 1 2; do
  echo "== new"; python tools/time_unet.py 2>&1 | grep forward
  echo "== head"; (cd _ab/head && python tools/time_unet.py 2>&1 | grep forward)
done
