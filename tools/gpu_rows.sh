cd $GRAFT_REPO_ROOT
cat > /tmp/r.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = torch.randn(256, 128256, device="cuda", generator=g)
for k in (128256,):
    for _ in range(3): rtk.batch_topk_dense(L, k)
    torch.cuda.synchronize()
    print("k", k, flush=True)
PY
RTK_PROFILE=1 python /tmp/r.py 2>&1 | grep -E "^k |profile|ctl|msd/rows" | tail -4 | cut -c1-250
