cd $GRAFT_REPO_ROOT
cat > /tmp/m.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.rand(1 << 28, device="cuda", generator=g)
for _ in range(4): rtk.topk(x, 1 << 20)
torch.cuda.synchronize()
PY
for b in 14; do echo "== bits $b"; RTK_MSD_BITS=$b RTK_PROFILE=1 python /tmp/m.py 2>&1 | grep -E "profile|dbg|ctl" | tail -4 | cut -c1-260; done
