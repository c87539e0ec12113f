# completion signalling A/B: system fence + spin on the mapped word (default) vs event wait (RTK_SIGNAL=event)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in "RTK_X=0" "RTK_SIGNAL=event"; do for a in "tiny 1" "c1 256" "c3 50" "c3 4096" "c2 1048576" "c4 65536 2"; do env $v python tools/ab_env.py $a; done; done; done
RTK_SIGNAL=event timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 2>&1 | tail -2
