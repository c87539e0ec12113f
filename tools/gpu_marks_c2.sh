cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
RTK_PROFILE=1 python - > gpurun_out/marks2.log 2>&1 <<'PY'
import torch, time, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.rand(1 << 28, device="cuda", generator=g)
for k in (256, 512, 1<<20):
    for _ in range(3): rtk.topk(x, k)
    torch.cuda.synchronize()
    print("k", k, rtk.last_stats(), flush=True)
PY
grep -E '^k |profile' gpurun_out/marks2.log | tail -12
