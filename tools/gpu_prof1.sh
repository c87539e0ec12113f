# per-phase marks of the bench workloads + ncu launch lists (C1, C2 k=256/2^20, C3 vocab LSD/MSD)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; O=gpurun_out/marks.txt; : > $O
for a in "c1 256" "c2 256" "c2 1048576" "c3 50" "c3 4096" "c3 128256"; do
  echo "== $a" >> $O; RTK_PROFILE=1 timeout 120 python tools/prof_marks.py $a 2>&1 | grep -E "rtk profile|rtk dbg|stats|rtk ctl" >> $O
done
echo "== c3 128256 RTK_LSD=off" >> $O; RTK_LSD=off RTK_PROFILE=1 timeout 120 python tools/prof_marks.py c3 128256 2>&1 | grep -E "rtk profile|stats|rtk ctl" >> $O
for m in 0 2; do echo "== c4 mode $m" >> $O; MODE=$m RTK_PROFILE=1 timeout 120 python tools/prof_marks.py c4 2>&1 | grep -E "rtk profile|stats|rtk ctl" >> $O; done
for a in "c1 256" "c2 256" "c2 1048576" "c3 128256"; do
  f=$(echo $a | tr ' ' _)
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launch_$f.csv python tools/prof_marks.py $a > /dev/null 2>&1; echo "ncu $a rc=$?"
done
