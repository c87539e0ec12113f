cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py -q -s --timeout=1400 > gpurun_out/san.log 2>&1; echo "san rc=$?"; grep -E "passed|failed|RACECHECK|ERROR SUMMARY|Race|hazard" gpurun_out/san.log | head -20
python tools/ab_env.py c4 65536 0; python tools/ab_env.py c4 65536 1; python tools/ab_env.py c4 65536 2
