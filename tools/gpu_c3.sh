cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/r.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2501_14336_b200 as rtk
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = torch.randn(256, 128256, device="cuda", generator=g)
ks = [int(x) for x in os.environ.get("KS", "50,4096").split(",")]
for k in ks:
    for _ in range(4): rtk.batch_topk_dense(L, k)
    torch.cuda.synchronize()
    print("k", k, flush=True)
PY
for v in ${VARIANTS:-""}; do
  echo "== $v"
  env $v RTK_PROFILE=1 python /tmp/r.py 2>&1 | grep -E "^k |profile|msd/rows" | cut -c1-300
done > gpurun_out/c3.log 2>&1
cat gpurun_out/c3.log
