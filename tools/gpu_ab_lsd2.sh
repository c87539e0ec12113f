cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in "" ab/i8m4 ab/i8m6 ab/i16m4; do for a in "c3 128256" "c3b 128256"; do echo -n "${v:-tree} "; RTK_PKG_ROOT=$GRAFT_REPO_ROOT/$v python tools/ab_env.py $a; done; done; done
