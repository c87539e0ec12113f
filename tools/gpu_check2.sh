cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log | grep -v '^\s*$' | tail -3
KS=50,4096 DT=f32,bf16 timeout 300 python tools/c3_ab.py "" "" > gpurun_out/c3ab.log 2>&1; cat gpurun_out/c3ab.log
