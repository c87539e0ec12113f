cd $GRAFT_REPO_ROOT
for k in 50 4096; do RTK_ROWS_TRACE=1 python tools/prof_marks.py c3 $k 2>&1 | grep -A8 "rows trace" | head -24; done
