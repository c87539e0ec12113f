cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KS=1048576 RTK_GRAPH_DUMP=gpurun_out/graph_c2.dot python tools/c2_ab.py "" > gpurun_out/g.log 2>&1
cat gpurun_out/g.log
grep -o 'label="[^"]*"' gpurun_out/graph_c2.dot | head -40
