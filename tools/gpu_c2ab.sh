cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/c2_ab.py "" "RTK_SPARSE_MAX=0" "RTK_SPARSE_MAX=4" "RTK_SPARSE_MAX=16" "RTK_PREFETCH_MB=0" "RTK_PREFETCH_MB=64" "RTK_PDL_COMPACT=1" > gpurun_out/c2ab.log 2>&1
cat gpurun_out/c2ab.log
