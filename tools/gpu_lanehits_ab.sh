# per-lane candidate appends in k_rows_fused's small-k stream (tree) vs warp-aggregated (ab/lh0)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for a in "c3 50" "c3b 50" "c3 512" "tiny 1"; do
  for v in "" ab/lh0; do echo -n "${v:-tree} "; RTK_PKG_ROOT=${v:+$GRAFT_REPO_ROOT/$v} timeout 120 python tools/ab_env.py $a; done
done; done
RTK_ROWS_TRACE=1 python tools/prof_marks.py c3 50 2>&1 | grep -A3 "rows trace" | tail -2
timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 2>&1 | tail -2
