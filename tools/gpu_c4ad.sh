cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/c4a.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
from paper_2501_14336_b200 import rtk as R
g = torch.Generator(device="cuda"); g.manual_seed(1)
xa = (128.6 + 0.1 * torch.rand(1 << 26, device="cuda", generator=g)).float()
pol = R.ScalePolicy(mode=R.ScaleMode(int(os.environ.get("MODE", "2"))), trigger_fraction=0.5, seed=31)
for i in range(4): rtk.scaled_topk(xa, 1 << 16, policy=pol)
torch.cuda.synchronize()
PY
MODE=2 RTK_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python /tmp/c4a.py 2>/dev/null | grep -E "k_|\"ID\"" | awk -F'","' '{print $5, $NF}' | tail -14
MODE=2 RTK_GRAPHS=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_first_digit -s 1 -c 1 -f -o gpurun_out/ncu_fdh python /tmp/c4a.py > /dev/null 2>&1
