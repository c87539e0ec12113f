RTK_PROFILE=1 timeout 300 python tools/prof_topk.py 28 1048576 4 2>&1 | tail -3
RTK_PROFILE=1 timeout 300 python tools/prof_topk.py 28 256 4 2>&1 | tail -2
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_sample_select|k_seg_plan|k_seg_hist" -c 3 -o gpurun_out/ss10 python tools/prof_topk.py 28 1048576 1 > gpurun_out/ncu10.log 2>&1
tail -1 gpurun_out/ncu10.log
