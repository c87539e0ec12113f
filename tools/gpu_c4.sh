cd $GRAFT_REPO_ROOT
cat > /tmp/c4.py <<'PY'
import sys, os, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
from paper_2501_14336_b200 import rtk as R
g = torch.Generator(device="cuda"); g.manual_seed(1)
xa = (128.6 + 0.1 * torch.rand(1 << 26, device="cuda", generator=g)).float()
pol = R.ScalePolicy(mode=R.ScaleMode(0), trigger_fraction=0.5, seed=31)
for i in range(3): rtk.scaled_topk(xa, 1 << 16, policy=pol)
torch.cuda.synchronize()
PY
RTK_PROFILE=1 python /tmp/c4.py 2>&1 | tee gpurun_out/c4.log | grep -E "profile|ctl|dbg" | tail -8 | cut -c1-300
