cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/r.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = torch.randn(256, 128256, device="cuda", generator=g)
for _ in range(3): rtk.batch_topk_dense(L, 128256)
torch.cuda.synchronize()
PY
RTK_GRAPHS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sort_groups -s 2 -c 1 -f -o gpurun_out/ncu_vsort python /tmp/r.py > gpurun_out/ncu_vsort.log 2>&1
RTK_GRAPHS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_msd_cluster -s 2 -c 1 -f -o gpurun_out/ncu_vmsd python /tmp/r.py > gpurun_out/ncu_vmsd.log 2>&1
tail -2 gpurun_out/ncu_vsort.log; tail -2 gpurun_out/ncu_vmsd.log
