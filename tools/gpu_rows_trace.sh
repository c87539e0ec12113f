# per-CTA phase trace of k_rows_fused (start, threshold, stream, select, sort[, gather]) on the C3 logits, f32 and bf16
cd $GRAFT_REPO_ROOT
for k in 50 4096; do RTK_ROWS_TRACE=1 python tools/prof_marks.py c3 $k 2>&1 | grep -A3 "rows trace" | tail -3; done
for k in 50 4096; do BF16=1 RTK_ROWS_TRACE=1 python tools/prof_marks.py c3 $k 2>&1 | grep -A3 "rows trace" | tail -3; done
