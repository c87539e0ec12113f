timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -4
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_sort_groups|k_seg_hist|k_seg_scatter|k_seg_plan|k_radix_pass|k_sample" -c 7 -o gpurun_out/finish6 python tools/prof_topk.py 28 1048576 1 > gpurun_out/ncu6.log 2>&1
tail -2 gpurun_out/ncu6.log
