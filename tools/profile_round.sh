# Profiles for the round (1 GPU): launch list of the bench-equivalent calls (C2 k=2^20, C3 batch)
# and full captures of the streaming kernel (k_compact) and the sort kernel. Run under gpurun.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_launches.csv python tools/prof_topk.py 28 1048576 3 > /dev/null 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_compact" -s 2 -c 1 \
    -o gpurun_out/prof_compact -f python tools/prof_topk.py 28 1048576 3 > gpurun_out/prof_compact.log 2>&1
echo "compact rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_sort_groups|k_sample_select" -s 2 -c 2 \
    -o gpurun_out/prof_finish -f python tools/prof_topk.py 28 1048576 3 > gpurun_out/prof_finish.log 2>&1
echo "finish rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_batch_launches.csv python -c "
import torch, paper_2501_14336_b200 as rtk
x=torch.randn(256,128256,device='cuda')
for kb in (50, 4096, 128256): rtk.batch_topk_dense(x, kb)
torch.cuda.synchronize()
" > /dev/null 2>&1
echo "batch rc=$?"
