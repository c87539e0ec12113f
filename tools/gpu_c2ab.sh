cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/c2_ab.py "" "RTK_SPARSE_SEL=1" "RTK_AHEAD=1" "RTK_AHEAD=1 RTK_SPARSE_MAX=512" "RTK_AHEAD=1 RTK_SPARSE_MAX=32" > gpurun_out/c2ab.log 2>&1
cat gpurun_out/c2ab.log
