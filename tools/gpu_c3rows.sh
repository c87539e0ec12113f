cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/r.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
for B in [int(x) for x in os.environ.get("BS", "74,148,256,296").split(",")]:
    L = torch.randn(B, 128256, device="cuda", generator=g)
    k = int(os.environ.get("K", "50"))
    for _ in range(4): rtk.batch_topk_dense(L, k)
    torch.cuda.synchronize()
    print("B", B, flush=True)
PY
RTK_PROFILE=1 python /tmp/r.py 2>&1 | grep -E "^B |profile" | awk '/^B/{print; next} {last=$0} /rows_fused/{l=$0} END{}' > /dev/null
RTK_PROFILE=1 python /tmp/r.py 2>&1 | grep -E "^B |profile" | grep -oE "^B .*|rows_fused=[0-9.]+us" | paste -sd' ' | sed 's/ B /\nB /g'
