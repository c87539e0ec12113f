# one-shot L2 prefetch at the row's start (RTK_ROWS_PF0 chunks of 32 KB beyond the ring)
cd $GRAFT_REPO_ROOT
python tools/c3_ab.py "" "RTK_ROWS_PF0=2" "RTK_ROWS_PF0=4" "RTK_ROWS_PF0=6" "RTK_ROWS_PF0=9" "RTK_ROWS_PF0=13" "" "RTK_ROWS_PF0=4" 
DT=bf16 python tools/c3_ab.py "" "RTK_ROWS_PF0=2" "RTK_ROWS_PF0=4" "RTK_ROWS_PF0=7"
for a in "tiny 1" "c1 256" "c2 1048576" "c4 65536 2"; do python tools/ab_env.py $a; done
RTK_ROWS_TRACE=1 RTK_ROWS_PF0=4 python tools/prof_marks.py c3 50 2>&1 | grep -A3 "rows trace" | tail -3
timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 2>&1 | tail -2
