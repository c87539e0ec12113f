cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
MODE=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launch_c4a.csv python tools/prof_marks.py c4 > /dev/null 2>&1; echo rc=$?
MODE=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launch_c4s.csv python tools/prof_marks.py c4 > /dev/null 2>&1; echo rc=$?
