cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or randomized or two_value or 16bit or dense" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log | grep -v '^\s*$' | tail -3
KS=128256 DT=f32,bf16 timeout 600 python tools/c3_ab.py "" "RTK_LSD=all" > gpurun_out/c3ab.log 2>&1; cat gpurun_out/c3ab.log
cat > /tmp/d.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, paper_2501_14336_b200 as rtk
x = torch.randn(256, 128256, device="cuda")
for _ in range(2): rtk.batch_topk_dense(x, 128256)
torch.cuda.synchronize()
PY
RTK_LSD=all ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lsd_launches.csv python /tmp/d.py > /dev/null 2>&1; echo "launch rc=$?"
grep lsd gpurun_out/lsd_launches.csv | tail -5 | awk -F'","' '{print substr($5,1,40), $NF}'
