# quick C2 k=2^20 run with profile marks + diagnostics
RTK_PROFILE=1 python - 2>&1 <<'PY' | tail -12
import torch, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.rand(1 << 28, device="cuda", generator=g)
for _ in range(3): rtk.topk(x, 1<<20)
torch.cuda.synchronize()
print(rtk.last_stats())
PY
