# ncu full captures (source-level) of the finishing kernels on the C2 k=2^20 workload
mkdir -p gpurun_out
RTK_PROFILE=1 python tools/prof_topk.py 28 1048576 2 2>&1 | grep ctl | tail -1
for K in k_msd_cluster k_sort_groups k_compact; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
     -o gpurun_out/ncu_$K -f python tools/prof_topk.py 28 1048576 2 > gpurun_out/ncu_$K.log 2>&1
  echo "$K rc=$?"
done
