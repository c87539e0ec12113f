cd $GRAFT_REPO_ROOT
python tools/ab_c2.py $GRAFT_REPO_ROOT/ab_old; python tools/ab_c2.py $GRAFT_REPO_ROOT
python tools/ab_c2.py $GRAFT_REPO_ROOT/ab_old; python tools/ab_c2.py $GRAFT_REPO_ROOT
