cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KS=256,1048576 timeout 1200 python tools/c2_ab.py "" "RTK_PDL_COMPACT=0" "RTK_DYN=12" "RTK_DYN=12 RTK_PDL_COMPACT=0" "RTK_DYN=24" "RTK_DYN=0 RTK_PDL_COMPACT=0" "" "RTK_PDL_COMPACT=0" "RTK_DYN=12" "RTK_DYN=12 RTK_PDL_COMPACT=0" "RTK_DYN=24" "RTK_DYN=0 RTK_PDL_COMPACT=0" > gpurun_out/c2ab.log 2>&1; cat gpurun_out/c2ab.log
