cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B=1 RTK_GRAPH_DUMP=gpurun_out/graph_b1.dot python tools/c3_ab.py "" > gpurun_out/g.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_b1.csv env B=1 KS=50 python tools/c3_ab.py "" >> gpurun_out/g.log 2>&1
cat gpurun_out/g.log
