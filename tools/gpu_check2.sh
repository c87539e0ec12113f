cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/c4.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, paper_2501_14336_b200 as rtk
from paper_2501_14336_b200 import rtk as R
g = torch.Generator(device="cuda"); g.manual_seed(1)
xa = (128.6 + 0.1 * torch.rand(1 << 26, device="cuda", generator=g)).float()
pol = R.ScalePolicy(mode=R.ScaleMode(0), trigger_fraction=0.5, seed=31)
for _ in range(3): rtk.scaled_topk(xa, 1 << 16, policy=pol)
torch.cuda.synchronize()
PY
RTK_MSD_Q=1 ncu --set full --clock-control none --import-source on -k regex:"k_compact" -s 1 -c 1 -o gpurun_out/prof_c4compact -f python /tmp/c4.py > gpurun_out/prof_c4c.log 2>&1; echo "rc=$?"
