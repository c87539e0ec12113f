cd $GRAFT_REPO_ROOT
for rep in 1 2; do for a in "c3 50" "c3 4096" "c3b 50" "c3b 4096"; do
  for v in "" ab/s0; do echo -n "${v:-tree} "; RTK_PKG_ROOT=${v:+$GRAFT_REPO_ROOT/$v} timeout 120 python tools/ab_env.py $a; done
done; done
RTK_ROWS_TRACE=1 python tools/prof_marks.py c3 50 2>&1 | grep -A3 "rows trace" | tail -3
