cd $GRAFT_REPO_ROOT
for r in 1 2; do python tools/ab_env.py tiny 1; python tools/ab_env.py tinynf 1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv python tools/ab_env.py tinynf 1 2>/dev/null | grep -v "^==" | cut -c1-50,200-300 | tail -4
