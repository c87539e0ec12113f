#!/bin/bash
# k_row_cluster: parity tests + C1 A/B against the general path (RTK_NO_RCLUSTER=1) + phase trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_row_cluster.py tests/test_gpu_parity.py -k "row_cluster or c1 or randomized or sorted or ties" -x -q --timeout=300 --timeout-method=thread > gpurun_out/rc_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rc_tests.log
{ timeout 120 python tools/ab_env.py tiny 1
for k in 1 256 512; do
  timeout 120 python tools/ab_env.py c1 $k
  RTK_NO_RCLUSTER=1 timeout 120 python tools/ab_env.py c1 $k
done
for k in 1 256 512; do RTK_ROWS_TRACE=1 python tools/prof_marks.py c1 $k 2>&1 | grep -A1 "rows trace" | tail -2; done
} > gpurun_out/rc_ab.log 2>&1
tail -3 gpurun_out/rc_tests.log; grep -E "^E |FAILED" gpurun_out/rc_tests.log | head; cat gpurun_out/rc_ab.log
