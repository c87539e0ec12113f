cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/t.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch
from paper_2501_14336_b200 import rtk as R
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = torch.randn(256, 128256, device="cuda", generator=g)
if os.environ.get("DT") == "bf16": L = L.to(torch.bfloat16)
for k in [int(v) for v in os.environ.get("KS", "50,4096").split(",")]:
    for _ in range(2): R.batch_topk_dense(L, k)
    torch.cuda.synchronize(); print("k", k, flush=True)
PY
RTK_GRAPHS=0 RTK_ROWS_TRACE=1 python /tmp/t.py > gpurun_out/trace.log 2>&1
DT=bf16 RTK_GRAPHS=0 RTK_ROWS_TRACE=1 python /tmp/t.py > gpurun_out/trace_bf16.log 2>&1
echo f32; grep -A2 'rows trace' gpurun_out/trace.log | tail -6
echo bf16; grep -A2 'rows trace' gpurun_out/trace_bf16.log | tail -6
