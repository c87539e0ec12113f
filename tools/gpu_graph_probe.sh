# fixed per-call cost: graph replay vs plain launches for the one-kernel calls (C1, C3 small k)
cd $GRAFT_REPO_ROOT
python tools/launch_floor.py
for v in "" "RTK_GRAPHS=0"; do for a in "tiny 1" "c1 256" "c3 50" "c3 4096"; do env $v python tools/ab_env.py $a; done; done
