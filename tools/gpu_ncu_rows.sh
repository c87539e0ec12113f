cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/r.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = torch.randn(256, 128256, device="cuda", generator=g)
k = int(os.environ.get("K", "50"))
for _ in range(3): rtk.batch_topk_dense(L, k)
torch.cuda.synchronize()
PY
K=50 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rows_fused -s 2 -c 1 -f -o gpurun_out/ncu_rows50 python /tmp/r.py > gpurun_out/ncu_rows50.log 2>&1
K=50 RTK_NO_FUSED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_compact -s 2 -c 1 -f -o gpurun_out/ncu_c3compact python /tmp/r.py > gpurun_out/ncu_c3compact.log 2>&1
tail -3 gpurun_out/ncu_rows50.log gpurun_out/ncu_c3compact.log
