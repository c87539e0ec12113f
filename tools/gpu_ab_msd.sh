cd $GRAFT_REPO_ROOT
for r in 1 2 3; do for v in "" ab/sortold; do for a in "c2 1048576" "c4 65536"; do echo -n "${v:-tree} "; RTK_PKG_ROOT=$GRAFT_REPO_ROOT/$v python tools/ab_env.py $a; done; done; done
