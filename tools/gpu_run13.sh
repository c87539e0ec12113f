RTK_PROFILE=1 timeout 300 python tools/prof_topk.py 28 1048576 3 2>&1 | tail -3
RTK_PROFILE=1 timeout 300 python tools/prof_topk.py 20 256 3 2>&1 | tail -3
