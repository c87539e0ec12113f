cd $GRAFT_REPO_ROOT
for rep in 1 2; do for a in "c3 4096" "c3b 4096" "c3 1024"; do
  for v in "" ab/lh2; do echo -n "${v:-tree} "; RTK_PKG_ROOT=${v:+$GRAFT_REPO_ROOT/$v} timeout 120 python tools/ab_env.py $a; done
done; done
