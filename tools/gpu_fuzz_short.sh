# 6-minute fuzz run on the working tree (tools/gpu_fuzz_long.sh with FUZZ_SECONDS=360, seeds from 700000)
cd $GRAFT_REPO_ROOT; FUZZ_SECONDS=360 SEED0=700000 bash tools/gpu_fuzz_long.sh
