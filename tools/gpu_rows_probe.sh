# C3 small-k rows kernel: per-phase trace and L2-prefetch distance sweep; the GPU tests after the sanitizer file
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sharded.py -q --timeout=300 2>&1 | tail -2
for k in 50 4096; do RTK_ROWS_TRACE=1 python tools/prof_marks.py c3 $k 2>&1 | grep -A8 "rows trace" | head -12; done
python tools/c3_ab.py "" "RTK_ROWS_PF=1" "RTK_ROWS_PF=2" "RTK_ROWS_PF=4" "RTK_ROWS_PF=8"
