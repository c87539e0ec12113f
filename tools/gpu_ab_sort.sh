cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in "" ab/lsdsort; do
  for a in "c1 256" "c1 1024" "c1 2000" "c2 4096"; do echo -n "${v:-tree} "; RTK_PKG_ROOT=$GRAFT_REPO_ROOT/$v python tools/ab_env.py $a; done
done; done
