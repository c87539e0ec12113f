cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/d.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, paper_2501_14336_b200 as rtk
x = torch.randn(256, 128256, device="cuda")
for _ in range(2): rtk.batch_topk_dense(x, 128256)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:"k_lsd_pass" -s 5 -c 1 -o gpurun_out/prof_lsd32 -f python /tmp/d.py > gpurun_out/prof_lsd32.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/prof_lsd32.ncu-rep --page details --section WarpStateStats --section SchedulerStats --section Occupancy > gpurun_out/lsd32_details.txt 2>&1
