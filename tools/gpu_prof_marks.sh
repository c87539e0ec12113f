# Per-stage GPU/host times of the pipeline (RTK_PROFILE=1 marks), C2 and C3 shapes
mkdir -p gpurun_out
RTK_PROFILE=1 python - > gpurun_out/marks.log 2>&1 <<'PY'
import torch, time, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.rand(1 << 28, device="cuda", generator=g)
for k in (256, 1<<14, 1<<20):
    for _ in range(3): rtk.topk(x, k)
    torch.cuda.synchronize()
    t=time.perf_counter(); rtk.topk(x,k); torch.cuda.synchronize(); print("k",k,"host wall us",(time.perf_counter()-t)*1e6, rtk.last_stats(), flush=True)
L = torch.randn(256, 128256, device="cuda", generator=g)
for k in (50, 4096, 128256):
    for _ in range(3): rtk.batch_topk_dense(L, k)
    torch.cuda.synchronize()
    t=time.perf_counter(); rtk.batch_topk_dense(L,k); torch.cuda.synchronize(); print("batch k",k,"host wall us",(time.perf_counter()-t)*1e6, rtk.last_stats(), flush=True)
PY
cat gpurun_out/marks.log | tail -40
