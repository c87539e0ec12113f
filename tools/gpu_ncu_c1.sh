cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sample_select|k_compact|k_sort_groups" -s 6 -c 3 \
    -o /tmp/ncu/c1 -f python tools/prof_marks.py c1 256 > /tmp/ncu/c1.log 2>&1; echo rc=$?
python tools/ncu_summary.py /tmp/ncu/c1.ncu-rep 30 > gpurun_out/ncu_c1_full.txt 2>&1
ncu -i /tmp/ncu/c1.ncu-rep --page details --csv > gpurun_out/ncu_c1_details.csv 2>&1
