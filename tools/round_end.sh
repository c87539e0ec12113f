# Round-end evidence: GPU parity suite, smoke, then tools/profile_round2.sh (bench line, reference
# arm, ncu launch lists and full captures). Run under gpurun; outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
bash tools/profile_round2.sh
