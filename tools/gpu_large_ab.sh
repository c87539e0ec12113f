# large-k rows variant ring shape: 1 x 32 KB (tree) vs 2 x 16 KB, 4 x 8 KB, 3 x 8 KB
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for a in "c3 4096" "c3b 4096" "c3 1024"; do
  for v in "" ab/l22 ab/l41 ab/l31; do echo -n "${v:-tree} "; RTK_PKG_ROOT=${v:+$GRAFT_REPO_ROOT/$v} timeout 120 python tools/ab_env.py $a; done
done; done
