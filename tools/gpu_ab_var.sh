# same-box A/B of library variants under ab/ (plus the in-tree build) on C2: tools/gpu_ab_var.sh v1 v2 ...
cd $GRAFT_REPO_ROOT
for round in 1 2; do
  python tools/ab_c2.py $GRAFT_REPO_ROOT
  for v in "$@"; do python tools/ab_c2.py $GRAFT_REPO_ROOT/ab/$v; done
done
