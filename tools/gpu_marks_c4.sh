cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
RTK_PROFILE=1 python - > gpurun_out/marks4.log 2>&1 <<'PY'
import torch, paper_2501_14336_b200 as rtk
from paper_2501_14336_b200 import rtk as R
g = torch.Generator(device="cuda"); g.manual_seed(1)
xa = (128.6 + 0.1 * torch.rand(1 << 26, device="cuda", generator=g)).float()
for m in (0, 1):
    pol = R.ScalePolicy(mode=R.ScaleMode(m), trigger_fraction=0.5, seed=31)
    for _ in range(3): rtk.scaled_topk(xa, 1 << 16, policy=pol)
    torch.cuda.synchronize(); print("mode", m, rtk.last_stats(), flush=True)
PY
grep -E '^mode|profile|ctl|phases' gpurun_out/marks4.log | tail -12
