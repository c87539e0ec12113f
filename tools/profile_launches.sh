mkdir -p gpurun_out
ncu --replay-mode application --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_launches_app.csv python tools/prof_topk.py 28 1048576 3 > gpurun_out/prof_launches_app.log 2>&1
echo "app-replay rc=$?"
RTK_MSD_Q=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_launches_q1.csv python tools/prof_topk.py 28 1048576 3 > /dev/null 2>&1
echo "q1 rc=$?"
