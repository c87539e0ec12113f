cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/d.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, paper_2501_14336_b200 as rtk
x = torch.randn(256, 128256, device="cuda")
for _ in range(2): rtk.batch_topk_dense(x, 128256)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lsd_launches.csv python /tmp/d.py > /dev/null 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_lsd_pass" -s 2 -c 1 -o gpurun_out/prof_lsd -f python /tmp/d.py > gpurun_out/prof_lsd.log 2>&1; echo "full rc=$?"
