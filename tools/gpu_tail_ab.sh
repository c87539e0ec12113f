# call-tail store variants (rtk_rows.cu rebuilt with RTK_TAIL_MODE=1/2 under ab/)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for a in "tiny 1" "c1 256" "c3 50" "c3 4096"; do
  for v in "" ab/t1 ab/t2; do echo -n "${v:-tree} "; RTK_PKG_ROOT=${v:+$GRAFT_REPO_ROOT/$v} timeout 120 python tools/ab_env.py $a; done
done; done
