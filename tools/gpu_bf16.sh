cd $GRAFT_REPO_ROOT
cat > /tmp/b.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = torch.randn(256, 128256, device="cuda", generator=g).to(torch.bfloat16)
for k in (50, 4096):
    for _ in range(4): rtk.batch_topk_dense(L, k)
    torch.cuda.synchronize()
    print("k", k, rtk.last_stats(), flush=True)
PY
RTK_PROFILE=1 python /tmp/b.py 2>&1 | grep -E "^k |profile|ctl|dbg" | tail -12 | cut -c1-260
python -m pytest tests -q -x -m gpu 2>&1 | tail -2
