# full ncu captures (source-level) of the kernels under work; text summaries in gpurun_out/ (the
# .ncu-rep files stay on the box unless KEEP is set: gpurun returns at most 64 MiB)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/ncu
cap() {  # name, kernel regex, skip, count, workload args...
  local name=$1 rx=$2 s=$3 c=$4; shift 4
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $s -c $c \
    -o /tmp/ncu/$name -f python tools/prof_marks.py "$@" > /tmp/ncu/$name.log 2>&1; echo "$name rc=$?"
  python tools/ncu_summary.py /tmp/ncu/$name.ncu-rep 25 > gpurun_out/ncu_$name.txt 2>&1
  case " $KEEP " in *" $name "*) cp /tmp/ncu/$name.ncu-rep gpurun_out/ ;; esac
}
cap lsd_mid "k_lsd_pass" 1 1 c3 128256
cap rows50 "k_rows_fused" 1 1 c3 50
cap c2_finish "k_sort_groups|k_sample_select" 2 2 c2 1048576
cap compact "k_compact" 1 1 c2 1048576
cap c1 "." 5 5 c1 256
