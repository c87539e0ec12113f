# GPU parity suite (+ optional pytest args in $PYARGS); outputs in gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q --timeout=300 --timeout-method=thread ${PYARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|error" gpurun_out/pytest_gpu.log | tail -30
