# Profiles for the round: launch list of the bench-equivalent call and one full capture of the
# streaming kernel (k_compact) plus the finishing kernels. Run under gpurun (1 GPU).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_launches.csv python tools/prof_topk.py 28 1048576 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_compact" -s 1 -c 1 \
    -o gpurun_out/prof_compact python tools/prof_topk.py 28 1048576 2 > gpurun_out/prof_compact.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_sort_groups|k_seg_hist|k_seg_scatter|k_sample_select" \
    -s 4 -c 4 -o gpurun_out/prof_finish python tools/prof_topk.py 28 1048576 2 > gpurun_out/prof_finish.log 2>&1
python -c "
import torch, paper_2501_14336_b200 as rtk
x=torch.randn(256,128256,device='cuda')
for _ in range(3): rtk.batch_topk_dense(x, 50)
" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_batch_launches.csv python -c "
import torch, paper_2501_14336_b200 as rtk
x=torch.randn(256,128256,device='cuda')
for kb in (50, 4096): rtk.batch_topk_dense(x, kb)
" > /dev/null 2>&1
