cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
RTK_GRAPH_DUMP=gpurun_out/g_tiny.dot python tools/ab_env.py tiny 1
RTK_GRAPH_DUMP=gpurun_out/g_c3.dot python tools/ab_env.py c3 50
RTK_GRAPH_EVENTS=0 python tools/ab_env.py tiny 1
RTK_GRAPH_EVENTS=0 python tools/ab_env.py c3 50
