cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cat > /tmp/t.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch
from paper_2501_14336_b200 import rtk as R
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = torch.randn(256, 128256, device="cuda", generator=g)
for k in [int(v) for v in os.environ.get("KS", "50,4096").split(",")]:
    for _ in range(3): R.batch_topk_dense(L, k)
    torch.cuda.synchronize(); print("k", k, flush=True)
PY
RTK_GRAPHS=0 RTK_ROWS_TRACE=1 python /tmp/t.py > gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log | tail -24
