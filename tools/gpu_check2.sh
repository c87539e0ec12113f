cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "c1 or c2_full or select_finish or randomized or narrow or special or scaled or dupl or host" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/c2_ab.py "" "RTK_NO_SELECT_FINISH=1" > gpurun_out/c2ab.log 2>&1; cat gpurun_out/c2ab.log
bash tools/gpu_marks_c2.sh > /dev/null; grep -B3 '^k 256' gpurun_out/marks2.log
