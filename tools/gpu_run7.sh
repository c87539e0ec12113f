timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "randomized_suite and uint32-1-2-1048579" 2>&1 | grep -E "Error|assert|mismatch|rtk_" | head -20
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_sort_groups" -c 1 -o gpurun_out/sort7 python tools/prof_topk.py 28 1048576 1 > gpurun_out/ncu7.log 2>&1
tail -1 gpurun_out/ncu7.log
