# long seeded fuzz run on the working tree (tools/fuzz_explore.py), bounded by FUZZ_SECONDS
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
FUZZ_SECONDS=${FUZZ_SECONDS:-1200} timeout $((${FUZZ_SECONDS:-1200} + 300)) python tools/fuzz_explore.py ${SEED0:-500000} 100000 > gpurun_out/fuzz_long.log 2>&1; echo "fuzz rc=$?"
tail -5 gpurun_out/fuzz_long.log
