# the working tree: GPU suite + the fixed-cost and headline workloads (tools/ab_env.py)
cd $GRAFT_REPO_ROOT
for a in "tiny 1" "c1 256" "c3 50" "c3 4096" "c2 1048576" "c4 65536 0" "c4 65536 2"; do python tools/ab_env.py $a; done
timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 2>&1 | tail -2
for a in "tiny 1" "c1 256" "c3 50"; do python tools/ab_env.py $a; done
