# Round-end evidence (1 GPU): full bench line (+ reference arm), ncu launch lists of the bench
# configs, and full captures of the top kernels. Run under gpurun; outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_launches.csv env RTK_MSD_Q=1 python tools/prof_topk.py 28 1048576 3 > /dev/null 2>&1; echo "launches rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_batch_launches.csv python -c "
import torch, paper_2501_14336_b200 as rtk
x=torch.randn(256,128256,device='cuda')
for kb in (50, 4096, 128256): rtk.batch_topk_dense(x, kb)
torch.cuda.synchronize()
" > /dev/null 2>&1; echo "batch rc=$?"
cat > /tmp/c4a.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
from paper_2501_14336_b200 import rtk as R
g = torch.Generator(device="cuda"); g.manual_seed(1)
xa = (128.6 + 0.1 * torch.rand(1 << 26, device="cuda", generator=g)).float()
for m in (0, 1, 2):
    pol = R.ScalePolicy(mode=R.ScaleMode(m), trigger_fraction=0.5, seed=31)
    for i in range(2): rtk.scaled_topk(xa, 1 << 16, policy=pol)
torch.cuda.synchronize()
PY
MODE=2 RTK_MSD_Q=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_c4_launches.csv python /tmp/c4a.py > /dev/null 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:"k_compact" -s 2 -c 1 \
    -o gpurun_out/prof_compact -f python tools/prof_topk.py 28 1048576 3 > gpurun_out/prof_compact.log 2>&1; echo "compact rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_msd_cluster|k_sort_groups|k_sample_select" -s 3 -c 3 \
    -o gpurun_out/prof_finish -f env RTK_MSD_Q=1 python tools/prof_topk.py 28 1048576 3 > gpurun_out/prof_finish.log 2>&1; echo "finish rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_rows_fused" -s 1 -c 2 \
    -o gpurun_out/prof_rows -f python -c "
import torch, paper_2501_14336_b200 as rtk
x=torch.randn(256,128256,device='cuda')
for kb in (50, 50, 4096, 4096): rtk.batch_topk_dense(x, kb)
torch.cuda.synchronize()
" > gpurun_out/prof_rows.log 2>&1; echo "rows rc=$?"
# dense bf16 rows (k = vocab): the one-sweep LSD kernels
cat > /tmp/lsd.py <<'PY'
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
x = torch.randn(256, 128256, device="cuda").to(torch.bfloat16)
for _ in range(2): rtk.batch_topk_dense(x, 128256)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_lsd_launches.csv python /tmp/lsd.py > /dev/null 2>&1; echo "lsd launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_lsd_pass" -s 2 -c 1 \
    -o gpurun_out/prof_lsd -f python /tmp/lsd.py > gpurun_out/prof_lsd.log 2>&1; echo "lsd rc=$?"
