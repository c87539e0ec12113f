cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in "" ab/lsdold; do for a in "c3 128256" "c3b 128256"; do echo -n "${v:-tree} "; RTK_PKG_ROOT=$GRAFT_REPO_ROOT/$v python tools/ab_env.py $a; done; done; done
timeout 600 python -m pytest tests -m gpu -q -k "lsd or vocab or dense or c3_headline or 16bit" --timeout=600 2>&1 | tail -2
