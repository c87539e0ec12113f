# where the fixed per-call cost goes: kernel span (trace) vs event-to-event, with/without the mapped completion word
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
RTK_ROWS_TRACE=1 python tools/prof_marks.py tiny 1 2>&1 | grep -A3 "rows trace" | tail -4
for v in "RTK_X=0" "RTK_NO_SIGNAL=1"; do for a in "tiny 1" "c1 256" "c3 50"; do env $v python tools/ab_env.py $a; done; done
ncu --metrics gpu__time_duration.sum,sm__ctas_launched.sum --clock-control none -c 6 --csv python tools/ab_env.py tiny 1 2>/dev/null | grep -v "^==" | cut -c1-60,200-400 | tail -8
